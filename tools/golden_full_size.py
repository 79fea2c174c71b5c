"""Write tests/golden/full_size_sha256.json: the SHA-256 of the ORACLE's output for the full-size
workloads (BASELINE.json configs[3] = c4 1 GiB, a 1 GiB slice of configs[4], and configs[4] = c5 8 GiB
in full), plus their bucket offsets.

Calls only gen/ (input bytes) and oracle/ (the method): the whole output is the concatenation, over
consecutive length ranges, of oracle.sort_lengths (the per-length sub-arrays of PAPER.md:58 sorted in the
paper-mpi shape), which tests/test_oracle.py pins against oracle.sort and against a
regex + sorted() library routine. The GPU tests (tests/test_gpu_fullsize.py) hash the CUDA path's output
and compare. Run on a host with ~48 GB of RAM (c5 in full: the 8 GiB text + the largest length group).

    python tools/golden_full_size.py [c4 c5_slice c5_full]
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import build_native  # noqa: E402

build_native.build_gen()
build_native.build_oracle()
import gen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full_size_sha256.json")
CASES = {"c4": (4, None), "c5_slice": (5, 1 << 30), "c5_full": (5, None)}
MAX_GROUP_WORDS = 400_000_000


def golden(cfg: int, n, threads: int):
    t0 = time.time()
    text, ntok = gen.generate(cfg, n=n)
    hist, off, lmax = oracle.histogram(text)
    groups, cur, cur_w = [], None, 0
    for L in range(1, lmax + 1):
        h = int(hist[L])
        if cur is not None and cur_w + h > MAX_GROUP_WORDS:
            groups.append(cur)
            cur = None
        if cur is None:
            cur, cur_w = [L, L], 0
        cur[1] = L
        cur_w += h
    if cur is not None:
        groups.append(cur)
    sha = hashlib.sha256()
    words_len = 0
    for a, b in groups:
        part = oracle.sort_lengths(text, a, b, threads, as_array=True)
        sha.update(memoryview(part))
        words_len += part.size
        del part
    c = gen.CONFIGS[cfg]
    return {"config": cfg, "workload": c.name, "n": len(text), "seed": c.seed, "gen_tokens": ntok,
            "n_words": int(off[256]), "words_len": words_len, "max_len": int(lmax),
            "off": [int(x) for x in off[: lmax + 2]], "sha256": sha.hexdigest(),
            "length_groups": groups, "seconds": round(time.time() - t0, 1)}


def main():
    names = sys.argv[1:] or list(CASES)
    data = json.load(open(OUT)) if os.path.exists(OUT) else {
        "_about": "SHA-256 of the oracle's sorted output (words, \"w\\n\" per word) and the bucket offsets of the "
                  "full-size workloads; written by tools/golden_full_size.py (gen/ + oracle/ only). "
                  "Citation: PAPER.md:58 (the whole result of the method), PAPER.md:54 (dataset shapes, scaled "
                  "by BASELINE.json configs)."}
    threads = os.cpu_count() or 1
    for name in names:
        cfg, n = CASES[name]
        d = golden(cfg, n, threads)
        data[name] = d
        print(name, {k: v for k, v in d.items() if k != "off"}, flush=True)
        json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
