"""Experiments: k1_ingest mean launch time on config 4 for the library at WSORT_LIB (or the in-tree one),
for each WSORT_INGEST_DEBUG value given (0 = the real kernel; other values skip parts: outputs unused)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

cfg = int(os.environ.get("CFG", "4"))
text, _ = gen.generate(cfg)
tag = os.environ.get("WSORT_LIB", "in-tree")
for d in (sys.argv[1:] or ["0"]):
    os.environ["WSORT_INGEST_DEBUG"] = d
    ws = WSort(0)
    ws.load_text(text)
    for _ in range(3):
        try:
            ws.tokenize()
        except Exception:
            pass
    ws.reset_kernel_stats()
    ws.set_profiling(True)
    for _ in range(10):
        try:
            ws.tokenize()
        except Exception:
            pass
    st = ws.kernel_stats()
    print(f"{tag} debug {d}: k1_ingest {st['k1_ingest']['ms'] / st['k1_ingest']['launches']:.4f} ms", flush=True)
    ws.close()
