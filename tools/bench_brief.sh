#!/bin/bash
# one-line summary of a bench JSON line: ms/step, Gwords/s, roofline frac, per-kernel ms
python - "$1" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(f"ms/step {d['ms_per_step']:.3f}  Gwords/s {d['value']/1e9:.2f}  input GB/s {d['input_gbs']:.1f}  roofline {d['roofline']['kernel']} {d['roofline']['achieved']:.0f} GB/s frac {d['roofline']['frac']:.3f}")
for k, v in d["kernels"].items():
    print(f"   {k:22s} {v['ms_per_step']:7.3f} ms  x{v['launches_per_step']:<4.0f} {v['gbs'] or 0:7.0f} GB/s")
if "e2e" in d: print("   e2e", round(d["e2e"]["value"]/1e9, 3), "Gwords/s")
if "cpu_baseline" in d: print("   cpu", round(d["cpu_baseline"]["value"]/1e6, 2), "Mwords/s")
print("   clocks", d.get("clocks"))
PY
