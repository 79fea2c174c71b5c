"""Device time of wsort_tokenize and wsort_sort (CUDA events on the context stream) vs their kernels'
summed event times: the difference is host-side bubbles (syncs, uploads, launches). Experiments."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

text, _ = gen.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
dev = torch.device("cuda:0")
s = torch.cuda.Stream(dev)
with torch.cuda.stream(s), WSort(0, stream=s.cuda_stream) as ws:
    ws.load_text(text)
    for _ in range(3):
        ws.tokenize()
        ws.sort("auto")
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tt = ts = 0.0
    ht = hs = 0.0
    for _ in range(5):
        e[0].record(s)
        t0 = time.perf_counter()
        ws.tokenize()
        t1 = time.perf_counter()
        e[1].record(s)
        ws.sort("auto")
        t2 = time.perf_counter()
        e[2].record(s)
        torch.cuda.synchronize()
        tt += e[0].elapsed_time(e[1])
        ts += e[1].elapsed_time(e[2])
        ht += t1 - t0
        hs += t2 - t1
    print(f"tokenize device {tt / 5:.3f} ms host {ht / 5 * 1e3:.3f} ms | sort device {ts / 5:.3f} ms host {hs / 5 * 1e3:.3f} ms")
