import sys, numpy as np
sys.path.insert(0, '/root/repo')
import gen, oracle
from paper_1411_5283_b200 import WSort
text, _ = gen.generate(4)
for mb in [int(x) for x in sys.argv[1:]]:
    t = text[: mb << 20]
    with WSort(0) as ws:
        ws.load_text(t)
        n = ws.tokenize()
        try:
            ws.sort("dense_msd")
            w, off = ws.fetch()
            print(mb, "ok", n, flush=True)
        except Exception as e:
            print(mb, "FAIL", e, flush=True)
