"""Per-launch DRAM traffic of every kernel class from an ncu CSV log of one bench run
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file X.csv`)
-> profiles/ncu_traffic.json (bench.py reads it for roofline.traffic).

usage: python tools/ncu_traffic_csv.py X.csv [OUT.json]
"""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_traffic import CLASS  # noqa: E402

EXTRA = {"k_hash_gather": "kh1_hash_gather", "k_hash_runs": "kh2_hash_runs", "k_emit_runs": "kh5_emit_runs",
         "k_dense_tiles": "k2d_dense_scan", "k_dense_clear": "k0_dense_clear", "k_msd_scatter_p": "k4m_msd_scatter"}


def main():
    src = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_traffic.json")
    rows = [r for r in csv.reader(l for l in open(src) if l.startswith('"'))]
    hdr = rows[0]
    iid, iname, imet, iunit, ival = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        v = float(r[ival].replace(",", ""))
        unit = r[iunit].lower()
        if r[imet] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
        elif unit.startswith("kbyte"):
            v *= 1e3
        elif unit.startswith("mbyte"):
            v *= 1e6
        elif unit.startswith("gbyte"):
            v *= 1e9
        per[(r[iid], r[iname])][r[imet]] = v
    agg = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "time_ms": 0.0})
    for (_, name), m in per.items():
        base = name.split("(")[0].split("::")[-1].split("<")[0].strip()
        cls = EXTRA.get(base) or CLASS.get(base) or base
        a = agg[cls]
        a["launches"] += 1
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a["time_ms"] += m.get("gpu__time_duration.sum", 0.0)
    res = {k: {"dram_bytes_per_launch": v["dram_bytes"] / v["launches"], "launches": v["launches"],
               "ncu_time_ms_per_launch": v["time_ms"] / v["launches"], "source": os.path.basename(src)}
           for k, v in sorted(agg.items())}
    json.dump(res, open(out, "w"), indent=1)
    for k, v in sorted(res.items(), key=lambda kv: -kv[1]["ncu_time_ms_per_launch"] * kv[1]["launches"])[:15]:
        print(f"{k:24s} launches {v['launches']:3d}  {v['ncu_time_ms_per_launch']:.3f} ms  {v['dram_bytes_per_launch'] / 1e6:9.1f} MB")


if __name__ == "__main__":
    main()
