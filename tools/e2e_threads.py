"""Experiments: end-to-end throughput (pinned host text in, host words out) with T host threads, each
driving its own context and stream (load_text -> tokenize -> sort -> fetch_async -> sync), vs the bench's
single-thread 3-context pipeline."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

cfg = gen.CONFIGS[4]
host = torch.empty(cfg.n, dtype=torch.uint8, pin_memory=True)
gen.generate(4, out=host.numpy())
K = 30


def run(T):
    streams = [torch.cuda.Stream(0) for _ in range(T)]
    ctxs = [WSort(0, stream=s.cuda_stream) for s in streams]
    ws0 = ctxs[0]
    ws0.load_text(host)
    n = ws0.tokenize()
    ws0.sort("auto")
    wl = int(ws0.sizes().words_len)
    outs = [torch.empty(wl + 64, dtype=torch.uint8, pin_memory=True).numpy() for _ in range(T)]
    for c, o in zip(ctxs, outs):
        c.load_text(host)
        c.tokenize()
        c.sort("auto")
        c.fetch_async(o)
        c.sync()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for s in streams[1:]:
        s.wait_event(e0)

    def work(i):
        c, o = ctxs[i], outs[i]
        for _ in range(K // T):
            c.load_text(host)
            c.tokenize()
            c.sort("auto")
            c.fetch_async(o)
            c.sync()

    ths = [threading.Thread(target=work, args=(i,)) for i in range(T)]
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
    ms = e0.elapsed_time(e1) / (K // T * T)
    print(f"{T} threads: {ms:.2f} ms per text end to end, {n / ms / 1e6:.2f} G words/s", flush=True)
    for c in ctxs:
        c.close()


for T in (1, 2, 3, 4):
    run(T)
