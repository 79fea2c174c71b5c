"""Per-launch DRAM traffic of every kernel class from an `ncu --set full` report of one tokenize+sort
step -> profiles/ncu_traffic.json (bench.py reads it for roofline.traffic).

usage: python tools/ncu_traffic.py REPORT.ncu-rep [OUT.json]
"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import load  # noqa: E402

# ncu kernel name -> bench kernel class (wsort_kernel_stats names)
CLASS = {
    "k_ingest": "k1_ingest", "k_dense_lensum": "k2_dense_lensum", "k_bucket_offsets": "k2_bucket_offsets",
    "k_dense_reduce": "k2d_dense_scan", "k_dense_scan": "k2d_dense_scan", "k_dense_compact": "k2d_dense_scan",
    "k_emit_dense": "k5d_emit_dense", "k_lscatter": "k3c_chunk_scatter", "k_msd_count": "k4m_msd_count",
    "k_msd_plan": "k4m_msd_plan", "k_msd_scatter": "k4m_msd_scatter", "k_msd_fin": "k4m_msd_finish",
    "k_msd_warp_sort": "k4m_msd_finish", "k_msd_copy": "k4m_msd_finish", "k_emit": "k5_emit",
    "k_msd_fin_split": "k4m_msd_fin_split", "k_msd_fin_emit": "k4m_msd_fin_emit",
    "k_msd_count0": "k4m_msd_count0", "k_msd_scatter0": "k4m_msd_scatter0",
}


def main():
    rep = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_traffic.json")
    agg = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "time_ms": 0.0})
    for d in load(rep):
        name = d["kernel"].split("(")[0].split("::")[-1]
        cls = CLASS.get(name)
        if cls is None:
            continue
        a = agg[cls]
        a["launches"] += 1
        a["dram_bytes"] += d.get("dram_read_B", 0) + d.get("dram_write_B", 0)
        a["time_ms"] += d.get("time_ms", 0)
    res = {k: {"dram_bytes_per_launch": v["dram_bytes"] / v["launches"], "launches": v["launches"],
               "ncu_time_ms_per_launch": v["time_ms"] / v["launches"], "source": os.path.basename(rep)}
           for k, v in agg.items()}
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)
    for k, v in sorted(res.items()):
        print(f"{k:22s} {v['dram_bytes_per_launch'] / 1e6:9.1f} MB/launch  x{v['launches']}")


if __name__ == "__main__":
    main()
