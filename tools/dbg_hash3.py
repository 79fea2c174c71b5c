import os, sys
sys.path.insert(0, os.getcwd())
import gen, build_native
build_native.build_wsort()
from paper_1411_5283_b200 import WSort
text, _ = gen.generate(1)
ws = WSort(0); ws.load_text(text); ws.tokenize(); ws.sort("auto"); ws.fetch(); ws.close()
