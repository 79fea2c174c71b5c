"""Print the MSD queue counters (WSORT_DEBUG_MSD) for the split-job parity cases (experiments)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["WSORT_DEBUG_MSD"] = "1"
from test_gpu_parity import SPLIT  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

with WSort(0) as ws:
    for name, text in SPLIT.items():
        print("==", name, flush=True)
        ws.load_text(text)
        ws.tokenize()
        ws.sort("dense_msd")
        ws.fetch()
