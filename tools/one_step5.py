"""One tokenize + sort of the 1 GiB slice of config 5 (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

text, _ = gen.generate(5, n=1 << 30)
with WSort(0) as ws:
    ws.load_text(text)
    ws.tokenize()
    ws.sort("auto")
