"""Per-kernel summary of an ncu --set full report (time, DRAM bytes, throughput, occupancy, pipes).

usage: python tools/ncu_summary.py REPORT.ncu-rep [--json OUT]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("time_ms", "gpu__time_duration.sum", 1e-6),
    ("dram_read_B", "dram__bytes_read.sum", 1),
    ("dram_write_B", "dram__bytes_write.sum", 1),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),   # (B200 --set full name)
    ("dram_pct_alt", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("smem_dyn_B", "launch__shared_mem_per_block_dynamic", 1),
    ("grid", "launch__grid_size", 1),
    ("inst", "smsp__inst_executed.sum", 1),
    ("lsu_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("alu_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("adu_pct", "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active", 1),
    ("smem_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("l2_bytes", "lts__t_bytes.sum", 1),
]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, m, scale in KEYS:   # (a metric absent from the report is skipped, not read as 0)
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    continue
                u = units[hdr.index(m)]
                if m == "gpu__time_duration.sum":
                    x = x * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1, "nsecond": 1e-6}.get(u, 1e-6)
                elif u.lower().startswith("gbyte"):
                    x *= 1e9
                elif u.lower().startswith("mbyte"):
                    x *= 1e6
                elif u.lower().startswith("kbyte"):
                    x *= 1e3
                d[k] = x
        if "dram_pct" not in d and "dram_pct_alt" in d:
            d["dram_pct"] = d["dram_pct_alt"]
        res.append(d)
    return res


def main():
    rep = sys.argv[1]
    res = load(rep)
    for d in res:
        dram = d.get("dram_read_B", 0) + d.get("dram_write_B", 0)
        gbs = dram / (d["time_ms"] / 1e3) / 1e9 if d.get("time_ms") else 0
        print(f"{d['kernel'][:60]:60s} {d.get('time_ms', 0):8.3f} ms  dram {dram / 1e6:9.1f} MB  {gbs:7.0f} GB/s "
              f"dram% {d['dram_pct'] if 'dram_pct' in d else float('nan'):5.1f} sm% {d.get('sm_pct', 0):5.1f} warps% {d.get('warps_active_pct', 0):5.1f} "
              f"lsu% {d.get('lsu_pct', 0):5.1f} alu% {d.get('alu_pct', 0):5.1f} adu% {d.get('adu_pct', 0):5.1f} "
              f"regs {d.get('regs', 0):.0f} conflicts {d.get('smem_conflicts', 0):.3g}")
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


main()
