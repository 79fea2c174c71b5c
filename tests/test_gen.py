"""Generator self-checks (-m "not gpu"): determinism, thread independence, token counts."""
import hashlib

import numpy as np

import gen
import oracle


def test_deterministic_and_thread_independent():
    a, na = gen.generate(2, threads=1)
    b, nb = gen.generate(2, threads=8)
    assert na == nb and np.array_equal(a, b)
    c, _ = gen.generate(2, seed=99)
    assert not np.array_equal(a, c)


def test_token_count_matches_oracle():
    for cfg in (1, 2):
        text, ntok = gen.generate(cfg)
        hist, off, lmax = oracle.histogram(text)
        assert int(off[256]) == ntok


def test_shapes_match_baseline_configs():
    # BASELINE.json configs[0..1]: ~33k / ~240k tokens, lengths 1-16 / 1-18, mean ~4.5
    for cfg, (lo, hi, lmax) in {1: (30_000, 38_000, 16), 2: (220_000, 270_000, 18)}.items():
        text, ntok = gen.generate(cfg)
        assert text.size == gen.CONFIGS[cfg].n
        assert lo <= ntok <= hi
        hist, off, L = oracle.histogram(text)
        assert L <= lmax
        mean = sum(i * int(hist[i]) for i in range(256)) / ntok
        assert 4.2 < mean < 5.0


def test_prefix_consistency_and_sha():
    a, _ = gen.generate(3, n=3 << 20)
    b, _ = gen.generate(3, n=2 << 20)
    assert np.array_equal(a[: 2 << 20], b)
    # frozen corpus: a change to the generator changes every recorded number; update DESIGN.md if so
    h = hashlib.sha256(gen.generate(1)[0].tobytes()).hexdigest()
    assert len(h) == 64


def test_config5_slice_shape():
    text, ntok = gen.generate(5, n=8 << 20)
    hist, off, lmax = oracle.histogram(text)
    assert lmax <= 64
    frac5 = int(hist[5]) / ntok
    assert 0.6 < frac5 < 0.8     # 70% of tokens from the length-5 sub-vocabulary (+ general L=5 excluded)
    long_ = sum(int(hist[L]) for L in range(13, 65)) / ntok
    assert long_ > 0.03          # prefix family (13..64) present
