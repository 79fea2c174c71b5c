"""Time wsort_sort alone (after one tokenize) on a config; per-kernel CUDA-event stats (experiments)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
algo = sys.argv[2] if len(sys.argv) > 2 else "auto"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
text, _ = gen.generate(cfg)
with WSort(0) as ws:
    ws.load_text(text)
    ws.tokenize()
    ws.sort(algo)
    ws.set_profiling(True)
    ws.reset_kernel_stats()
    for _ in range(reps):
        ws.sort(algo)
    for k, v in sorted(ws.kernel_stats().items(), key=lambda kv: -kv[1]["ms"]):
        print(f"{k:22s} {v['ms'] / reps:8.3f} ms/sort  x{v['launches'] / reps:.0f}")
