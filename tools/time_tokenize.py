"""Time wsort_tokenize (K1 ingest) alone on a config, per-kernel CUDA-event stats (experiments)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
text, _ = gen.generate(cfg)
with WSort(0) as ws:
    ws.load_text(text)
    for _ in range(3):
        ws.tokenize()
    ws.set_profiling(True)
    ws.reset_kernel_stats()
    for _ in range(10):
        ws.tokenize()
    for k, v in ws.kernel_stats().items():
        print(os.environ.get("WSORT_INGEST_DEBUG", "0"), k, v)
