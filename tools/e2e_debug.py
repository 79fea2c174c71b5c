"""Host timestamps of the pipelined e2e loop (which call blocks) — experiments."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

cfg = gen.CONFIGS[4]
host = torch.empty(cfg.n, dtype=torch.uint8, pin_memory=True)
gen.generate(4, out=host.numpy())
mode = sys.argv[1] if len(sys.argv) > 1 else "own"
if mode == "own":
    ctx = [WSort(0), WSort(0)]
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    ctx = [WSort(0, stream=s[0].cuda_stream), WSort(0, stream=s[1].cuda_stream)]
else:
    s2 = torch.cuda.Stream()
    ctx = [WSort(0), WSort(0, stream=s2.cuda_stream)]
for c in ctx:
    c.load_text(host)
    c.tokenize()
    c.sort()
words_len = ctx[0].sizes().words_len
outs = [torch.empty(words_len + 64, dtype=torch.uint8, pin_memory=True).numpy() for _ in range(2)]
torch.cuda.synchronize()
t0 = time.perf_counter()
log = []
ctx[0].load_text(host)
K = 6
for i in range(K):
    cur, nxt = ctx[i % 2], ctx[(i + 1) % 2]
    cur.tokenize(); log.append(("tok", i, time.perf_counter() - t0))
    if i + 1 < K:
        nxt.load_text(host); log.append(("load", i + 1, time.perf_counter() - t0))
    cur.sort(); log.append(("sort", i, time.perf_counter() - t0))
    cur.fetch_async(outs[i % 2]); log.append(("fetch", i, time.perf_counter() - t0))
for c in ctx:
    c.sync()
tt = time.perf_counter() - t0
for e in log:
    print(f"{e[0]:6s} {e[1]} {e[2]*1e3:8.2f} ms")
print(mode, f"total {tt*1e3:.1f} ms, per step {tt/K*1e3:.1f} ms")
