"""Experiments: device throughput with 1 vs 2 texts in flight (two contexts on two streams, one host thread
each; ctypes releases the GIL inside libwsort calls)."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

text, _ = gen.generate(4)
dev = torch.device("cuda:0")
d_text = torch.from_numpy(text).to(dev)
K = 20


def run(nctx):
    streams = [torch.cuda.Stream(dev) for _ in range(nctx)]
    ctxs = [WSort(0, stream=s.cuda_stream) for s in streams]
    for c in ctxs:
        c.load_text(d_text)
        for _ in range(3):
            c.tokenize()
            c.sort("auto")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for s in streams[1:]:
        s.wait_event(e0)

    def work(c, n):
        for _ in range(n):
            c.tokenize()
            c.sort("auto")

    ths = [threading.Thread(target=work, args=(c, K // nctx)) for c in ctxs]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for s in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(s)
        streams[0].wait_event(ev)
    e1.record(streams[0])
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    print(f"{nctx} context(s): {ms:.3f} ms per text, {len(text) / ms / 1e6:.1f} GB/s input")
    for c in ctxs:
        c.close()


run(1)
run(2)
run(1)
run(2)
