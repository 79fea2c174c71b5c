import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
print("import", flush=True)
from paper_1411_5283_b200 import WSort
texts = {"tiny": b"hello world abcdefg", "longs": b" ".join([b"abcdefgh"] * 5000), "mixed": b"the quick brown foxes jumped overthelazy dogs " * 2000}
with WSort(0) as ws:
    print("created", flush=True)
    for name, t in texts.items():
        t0 = time.time()
        ws.load_text(t)
        print(name, "loaded", flush=True)
        try:
            n = ws.tokenize()
            print(name, "tokenized", n, flush=True)
            ws.sort("dense_msd")
            w, off = ws.fetch()
            print(name, "ok", n, len(w), time.time() - t0, flush=True)
        except Exception as e:
            print(name, "ERR", e, flush=True)
