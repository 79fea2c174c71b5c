"""Exactly one tokenize + sort of a config on cuda:0 (for ncu captures of every kernel of one step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402

text, _ = gen.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
with WSort(0) as ws:
    ws.load_text(text)
    ws.tokenize()
    ws.sort(sys.argv[2] if len(sys.argv) > 2 else "auto")
    ws.fetch()
