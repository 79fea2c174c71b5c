#!/bin/bash
# one bench line for a given config (default 5 = the 1 GiB slice of config 5 via gen n) — experiments
python - "$@" <<'PY'
import sys, os, json, time
sys.path.insert(0, os.getcwd())
import gen
from paper_1411_5283_b200 import WSort
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = (1 << 30) if cfg == 5 else None
text, W = gen.generate(cfg, n=n)
with WSort(0) as ws:
    ws.load_text(text); ws.tokenize(); ws.sort("auto")
    ws.set_profiling(True); ws.reset_kernel_stats()
    import torch
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5):
        ws.tokenize(); ws.sort("auto")
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    print(f"config {cfg}: {W} words, {dt*1e3:.2f} ms/step (host clock), {W/dt/1e9:.2f} G words/s")
    for k, v in sorted(ws.kernel_stats().items(), key=lambda kv: -kv[1]["ms"]):
        print(f"   {k:22s} {v['ms']/5:8.3f} ms x{v['launches']/5:.0f}")
PY
