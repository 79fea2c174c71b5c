"""Per-kernel instruction counts by CUDA source line from an ncu report (source page, cuda+sass).

usage: python tools/ncu_lines.py REPORT.ncu-rep [TOP]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
res = {}
fn = path = hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        iI = hdr.index("Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or not r[0].strip().isdigit():
        continue
    d = res.setdefault(fn, collections.defaultdict(lambda: [0.0, 0.0]))
    try:
        e = d[(path, int(r[0]), r[1].strip()[:80])]
        e[0] += float(r[iI] or 0)
        e[1] += float(r[iS] or 0)
    except ValueError:
        pass
for fn, d in res.items():
    ti = sum(v[0] for v in d.values()) or 1
    ts = sum(v[1] for v in d.values()) or 1
    print(f"== {fn[:70]}  inst={ti:.3g}")
    for k, v in sorted(d.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {100 * v[0] / ti:5.1f}% inst {100 * v[1] / ts:5.1f}% stall  {k[0]}:{k[1]:4d}  {k[2]}")
