"""One tokenize + sort with per-launch CUDA events, printed in stream order with the gaps (experiments)."""
import os
import sys

os.environ["WSORT_DEBUG_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
text, _ = gen.generate(cfg, n=(1 << 30) if cfg == 5 else None)   # config 5: its 1 GiB slice
with WSort(0) as ws:
    ws.load_text(text)
    for _ in range(2):
        ws.tokenize()
        ws.sort("auto")
    ws.set_profiling(True)
    ws.tokenize()
    ws.sort("auto")
    ws.kernel_stats()
