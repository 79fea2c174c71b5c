"""Hash-mode ingest diagnostics (experiments): table fill, distinct words, overflow flag, K1 time."""
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import gen, build_native
build_native.build_wsort()
from paper_1411_5283_b200 import WSort
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
text, _ = gen.generate(cfg, n=(int(sys.argv[2]) if len(sys.argv) > 2 else None))
ws = WSort(0)
ws.load_text(text)
ws.set_profiling(True)
for i in range(3):
    ws.tokenize()
st = ws.kernel_stats()
print({k: (v["launches"], round(v["ms"] / max(v["launches"], 1), 3)) for k, v in st.items()})
print("ingest info", ws.ingest_info())
