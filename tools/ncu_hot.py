"""Summarise an ncu report: top CUDA source lines by warp-stall samples / instructions, per kernel.

usage: python tools/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [TOP]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fn, path, hdr = None, None, None
    agg = collections.defaultdict(lambda: collections.defaultdict(lambda: [0.0, 0.0, ""]))
    cur_line = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1]
            continue
        if r[0] == "Function Name":
            fn = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            iS = hdr.index("Warp Stall Sampling (All Samples)")
            iI = hdr.index("Instructions Executed")
            continue
        if hdr is None or fn is None or not re.search(kre, fn):
            continue
        if r[0]:
            cur_line = (path.rsplit("/", 1)[-1], r[0], r[1].strip()[:100])
        try:
            s = float(r[iS] or 0)
            i = float(r[iI] or 0)
        except (ValueError, IndexError):
            continue
        a = agg[fn][cur_line]
        a[0] += s
        a[1] += i
    for fn, d in agg.items():
        ts = sum(v[0] for v in d.values()) or 1
        ti = sum(v[1] for v in d.values()) or 1
        print(f"== {fn}  samples={ts:.0f} warp-inst={ti:.3g}")
        for k, v in sorted(d.items(), key=lambda kv: -kv[1][0])[:top]:
            print(f"{100*v[0]/ts:5.1f}% stall {100*v[1]/ti:5.1f}% inst  {k[0]}:{k[1]:>4} {k[2]}")


main()
