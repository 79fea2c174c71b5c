"""Stress workload: small texts through every sort path of libwsort, `WSORT_STRESS_REPS` times each (default
1) on one context, every output compared byte for byte with the oracle (compute-sanitizer is not available on
the GPU pool: intermittent races show up as a MISMATCH over many repetitions instead).

    python tools/stress_run.py <size> [algo ...]

size: c1 | c2 | mid (8 MiB of config 3: several CTAs per kernel, level-0 chunk path) | edge (hand-made
texts: empty, no letters, all 256 byte values, 66/67/255-letter words, one bucket).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
import oracle  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402


def texts(size):
    if size == "c1":
        return [("c1", gen.generate(1)[0])]
    if size == "c2":
        return [("c2", gen.generate(2)[0])]
    if size == "mid":
        return [("c3-8MiB", gen.generate(3, n=8 << 20)[0]), ("c5-4MiB", gen.generate(5, n=4 << 20)[0])]
    rng = np.random.default_rng(7)
    out = [("empty", np.zeros(0, np.uint8)), ("no-letters", np.frombuffer(b"1234 5678 !!\n", np.uint8)),
           ("all-bytes", rng.integers(0, 256, 65536, dtype=np.uint8)),
           ("long-words", np.frombuffer(b" ".join([b"a" * 66, b"b" * 67, b"Zq" * 127 + b"x", b"c" * 6, b"dd", b"e" * 48] * 40), np.uint8)),
           ("one-bucket", np.frombuffer(b" ".join(bytes(rng.integers(97, 123, 9, dtype=np.uint8)) for _ in range(30000)), np.uint8))]
    return out


def main():
    size = sys.argv[1]
    algos = sys.argv[2:] or ["auto", "auto_count", "lsd_radix", "oets_merge", "msd_radix", "msd_oets", "ragged"]
    bad = 0
    with WSort(0) as ws:
        for name, text in texts(size):
            ref = oracle.sort(text, oracle.MERGE, want_src=True)
            for algo in algos * int(os.environ.get("WSORT_STRESS_REPS", "1")):
                ws.set_ingest("count" if algo == "auto_count" else "auto")
                ws.load_text(text)
                n = ws.tokenize()
                src = algo in ("lsd_radix", "ragged")
                ws.sort("auto" if algo == "auto_count" else algo, src_off=src)
                got = ws.fetch(src_off=src)
                ok = n == ref.n_words and got[1] == ref.off and got[0].tobytes() == ref.words
                if src:
                    ok = ok and bool((got[2] == ref.src_off).all())
                print(f"{name:12s} {algo:11s} words={n:9d} {'ok' if ok else 'MISMATCH'}", flush=True)
                bad += not ok
        ws.set_ingest("auto")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
