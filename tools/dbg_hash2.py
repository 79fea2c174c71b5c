"""Hash path diagnostics (experiments): distinct long words per length vs the oracle, first mismatch."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import gen, oracle, build_native
build_native.build_wsort()
from paper_1411_5283_b200 import WSort
for cfg, n in ((1, None), (2, None), (3, 8 << 20)):
    text, _ = gen.generate(cfg, n=n)
    ref = oracle.sort(text, oracle.MERGE)
    ws = WSort(0)
    ws.load_text(text)
    ws.tokenize()
    info = ws.ingest_info()
    ws.sort("auto")
    w, off = ws.fetch()
    w = w.tobytes()
    words = ref.words.split(b"\n")[:-1]
    dist = {}
    for L in range(6, ref.max_len + 1):
        b = words[ref.off[L]:ref.off[L + 1]]
        dist[L] = len(set(b))
    print("cfg", cfg, "info", info, "oracle distinct 6..24:", sum(v for L, v in dist.items() if L <= 24),
          "25..:", sum(v for L, v in dist.items() if L > 24), "equal:", w == ref.words, "off equal:", off == ref.off, flush=True)
    if w != ref.words:
        g = w.split(b"\n")
        i = next(i for i in range(min(len(g), len(words))) if g[i] != words[i])
        L = len(words[i])
        print("  first diff word", i, "L", L, "gpu", g[i][:40], "ref", words[i][:40], "bucket start", ref.off[L])
    ws.close()
