# K1 cost breakdown by category (timing experiments only: WSORT_INGEST_DEBUG skips parts of k_ingest;
# the outputs are then wrong and unused). Prints k1_ingest ms per step for each setting.
for d in 0 1 16 17 8 2 25; do
  WSORT_INGEST_DEBUG=$d python - <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, gen, build_native
build_native.build_wsort()
from paper_1411_5283_b200 import WSort
text, _ = gen.generate(4)
ws = WSort(0)
ws.load_text(text)
for _ in range(3):
    ws.tokenize()
ws.reset_kernel_stats(); ws.set_profiling(True)
for _ in range(10):
    try:
        ws.tokenize()
    except Exception:
        pass
st = ws.kernel_stats()
print("debug", os.environ["WSORT_INGEST_DEBUG"], "k1_ingest ms", st["k1_ingest"]["ms"] / st["k1_ingest"]["launches"], flush=True)
PY
done
