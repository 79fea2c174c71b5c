"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar: bit-exact words, bucket offsets and src_off (all integer/byte work).
Sizes: hand-written edge cases, random texts spanning many 8 KiB tokenizer steps / CTA chunks /
radix tiles with ragged tails, BASELINE configs 1-3 in full. The full-size workloads (config 4, the
bench workload in its launch configuration, and config 5) are in tests/test_gpu_fullsize.py.
"""
import glob
import json
import os
import random

import numpy as np
import pytest

import gen
import oracle
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

ALGOS = ["lsd_radix", "oets_merge", "msd_radix", "msd_oets", "dense_msd", "auto_count", "ragged"]
# keys-only algorithms: without src_off (with it they fall back to the stable LSD path)
KEYS_ONLY = {"msd_radix", "msd_oets", "dense_msd", "auto_count"}
# "auto_count": AUTO after a counting ingest (wsort_set_ingest COUNT: the table of distinct long words)


@pytest.fixture(scope="module")
def ws():
    import build_native

    build_native.build_wsort()
    from paper_1411_5283_b200 import WSort

    w = WSort(0)
    yield w
    w.close()


def gpu_sort(ws, text, algo="lsd_radix", src=True):
    ws.set_ingest("count" if algo == "auto_count" else "auto")
    ws.load_text(text)
    ws.tokenize()
    ws.sort("auto" if algo == "auto_count" else algo, src_off=src)
    ws.set_ingest("auto")
    if src:
        w, off, so = ws.fetch(src_off=True)
        return w.tobytes(), off, so
    w, off = ws.fetch()
    return w.tobytes(), off, None


def check(ws, text, algo="lsd_radix"):
    ref = oracle.sort(text, oracle.MERGE, want_src=True)
    keys_only = algo in KEYS_ONLY
    words, off, src = gpu_sort(ws, text, algo, src=not keys_only)
    assert off == ref.off
    if words != ref.words:
        a, b = words.split(b"\n"), ref.words.split(b"\n")
        i = next((i for i in range(min(len(a), len(b))) if a[i] != b[i]), min(len(a), len(b)))
        pytest.fail(f"first differing word #{i} of {len(b)}: gpu={a[i][:80] if i < len(a) else None!r} "
                    f"oracle={b[i][:80] if i < len(b) else None!r}")
    if not keys_only:
        assert np.array_equal(src, ref.src_off)
    return ref


GOLD = [json.load(open(p)) for p in sorted(glob.glob(os.path.join(GOLDEN, "*.json")))]
GOLD = [g for g in GOLD if "text_latin1" in g]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("fx", GOLD, ids=[g["name"] for g in GOLD])
def test_golden(ws, fx, algo):
    text = fx["text_latin1"].encode("latin-1")
    words, off, src = gpu_sort(ws, text, algo, src=algo not in KEYS_ONLY)
    assert words == b"".join(w.encode() + b"\n" for w in fx["words"])
    assert off == fx["off"]
    if algo not in KEYS_ONLY:
        assert src.tolist() == fx["src_off"]


def _edge_cases():
    S = 8192
    cases = {
        "empty": b"",
        "separators_only": b" \n\t.,;!?0123456789\x00\xff" * 1000,
        "one_letter": b"Q",
        "max_len_255": b"ab " + b"x" * 255 + b" c",
        "max_len_255_at_end": b"zz " + b"Y" * 255,
        "giant_duplicate_run": b"a " * 600_000,
        "duplicate_word_run": b"hello " * 300_000,
        "all_one_word_no_sep": b"w" * 200,
        "straddle_step": b" " * (S - 3) + b"abcdef" + b" " * (S - 1) + b"q" + b"r" * 7 + b" z",
        "step_multiple_exact": (b"abc de " * (2 * S // 7 + 1))[: 2 * S],
        "ends_mid_word": (b"lorem ipsum dolor " * 2000) + b"sitame",
        "high_bytes": bytes(range(256)) * 300,
        "prefix_12_ties": b" ".join(b"abcdefghijkl" + bytes([97 + (i * 7) % 26, 97 + i % 26]) for i in range(5000)),
        "long_words_13_64": b" ".join(bytes([97 + (i * j) % 26 for j in range(13 + i % 52)]) for i in range(3000)),
        "long_words_65_255": b" ".join(bytes([97 + (i * j * 3) % 26 for j in range(65 + i % 191)]) for i in range(600)),
        "mixed_case_dups": b"Apple APPLE apple aPPle " * 5000,
        "reverse_sorted_distinct": b" ".join(
            bytes([97 + (i // 676) % 26, 97 + (i // 26) % 26, 97 + i % 26]) for i in reversed(range(17576))),
        # dense tables (L <= 5): every L=1/L=2 entry, first/last entries, cache overflow (many distinct
        # L=5 words go to the global fallback), hot words hit in every CTA
        "dense_all_l1_l2": b" ".join([bytes([97 + i]) for i in range(26)] +
                                     [bytes([97 + i // 26, 97 + i % 26]) for i in range(676)]) * 3,
        "dense_extremes": b"a aa aaa aaaa aaaaa z zz zzz zzzz zzzzz ZZZZZ Aaaaa " * 777,
        "dense_l5_distinct": b" ".join(bytes([97 + (i * 7919 // 26 ** j) % 26 for j in range(5)])
                                       for i in range(120_000)),
        "dense_hot_l4_l5": b"that with those their there " * 60_000,
        # staged classes: L = 6 (class 1), 7..12 (2), ..., 43..48 (class 8), enough to fill many chunks
        "staged_l6_many": b" ".join(bytes([97 + (i * 31 // 26 ** j) % 26 for j in range(6)]) for i in range(150_000)),
        "staged_classes_6_48": b" ".join(bytes([97 + (i * j + j * j) % 26 for j in range(6 + i % 43)])
                                         for i in range(40_000)),
        "staged_l48_dups": (b"q" * 47 + b"r ") * 5000 + (b"q" * 48 + b" ") * 3000,
        # key-width classes 9..11 (49..66 letters, config 5's longest words) and the first unstaged length
        "staged_classes_9_11": b" ".join(bytes([97 + (i * j + 3 * j) % 26 for j in range(49 + i % 18)])
                                         for i in range(6_000)) + b" " + b"z" * 66 + b" " + b"a" * 66,
        "unstaged_67": b"ab " * 1000 + b"m" * 67 + b" x",
        # small-text path: one bucket of 12 000 distinct 7-letter words (more than one tile, more distinct
        # keys than a finishing table holds: the whole-bucket job re-enters the MSD as a level-0 segment)
        "small_bucket_overflows": b" ".join(bytes([97 + (i * 7919 // 26 ** j) % 26 for j in range(7)])
                                            for i in range(12_000)),
        # small-text path, wide keys: whole buckets of 3000 distinct 19- / 40-letter words (more than one
        # tile, more distinct keys than a finishing table holds): the finishing CTA partitions the whole
        # bucket itself, by digit 0 (first two letters, which vary here), into sub-jobs
        "small_wide_bucket_partitioned": b" ".join(
            bytes([97 + (i * 7919 + (i * i >> j % 11) * (j + 1)) % 26 for j in range(19 if i % 2 else 40)])
            for i in range(6_000)),
    }
    # a word crossing every 8 KiB boundary of a multi-step text (CTA chunk boundaries too)
    t = bytearray(b"." * (S * 40))
    for k in range(1, 40):
        pos = k * S - 5 + (k % 9)
        t[pos: pos + 10 + (k % 5)] = b"m" * (10 + (k % 5))
    cases["cross_every_step"] = bytes(t)
    return cases


EDGE = _edge_cases()


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("name", list(EDGE))
def test_edge_cases(ws, name, algo):
    check(ws, EDGE[name], algo)


@pytest.mark.parametrize("name", list(EDGE))
def test_edge_cases_chunk_level0(ws, name, monkeypatch):
    """Small texts take the small path (keys regrouped by length, one finishing job per bucket); the same
    edge cases through the level-0 chunk path (count0 / scatter0) that large texts take."""
    monkeypatch.setenv("WSORT_NO_SMALL", "1")
    check(ws, EDGE[name], "dense_msd")


def _split_cases():
    """MSD children of > 128K keys, which the streaming finish splits into parts of 32K keys (one CTA
    each) merged by the last part: one word (all-equal runs), few distinct words (merged), too many
    distinct words in every part or only in their union (the job re-enters the MSD), for 2-word keys
    (L = 7..9) and wider keys (L = 14, 20)."""
    rng = np.random.default_rng(1411)

    def words(prefix: bytes, L: int, n_distinct: int, n: int, blocks: bool = False):
        letters = rng.integers(97, 123, size=(n_distinct, L - len(prefix)), dtype=np.uint8)
        vocab = [prefix + bytes(r) for r in letters]
        if blocks:   # consecutive runs of 32K words drawn from disjoint eighths of the vocabulary
            q = n_distinct // 8
            idx = np.concatenate([(i % 8) * q + rng.integers(0, q, size=32768) for i in range(n // 32768 + 1)])[:n]
        else:
            idx = rng.integers(0, n_distinct, size=n)
        # a few words of the same length with other first letters: the bucket is split at the first digit
        # (not skipped), so the prefix's child is one job of n keys
        decoy = [bytes([97 + i % 26, 97 + (i // 26) % 26]) + b"x" * (L - 2) for i in range(40)]
        return b" ".join(vocab[i] for i in idx) + b" " + b" ".join(decoy) + b" "

    return {
        "split_one_word": b"quietly " * 300_000 + b"quintessential " * 200_000 + b"abcdefg nopqrstuvwxyza ",
        "split_few_distinct": words(b"qu", 9, 600, 300_000),
        "split_few_distinct_wide": words(b"qu", 20, 400, 300_000),
        "split_overflow_parts": words(b"qu", 8, 50_000, 200_000),
        "split_overflow_union": words(b"qu", 8, 8 * 900, 270_000, blocks=True),
        "split_overflow_wide": words(b"qu", 14, 3000, 200_000),
    }


SPLIT = _split_cases()


@pytest.mark.parametrize("algo", ["dense_msd", "msd_oets", "lsd_radix"])
@pytest.mark.parametrize("name", list(SPLIT))
def test_split_jobs(ws, name, algo):
    check(ws, SPLIT[name], algo)


@pytest.mark.parametrize("algo", ALGOS)
def test_word_too_long(ws, algo):
    from paper_1411_5283_b200 import WSortError

    for text in (b"x " + b"Q" * 256, b"Q" * 300 + b" a", b" " * 8190 + b"L" * 400):
        ws.load_text(text)
        with pytest.raises(WSortError) as e:
            ws.tokenize()
        assert e.value.status == -7
        with pytest.raises(oracle.OracleError) as e2:
            oracle.sort(text)
        assert e2.value.status == -7


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("seed", range(12))
def test_random_texts(ws, seed, algo):
    rng = random.Random(seed)
    n = rng.choice([1, 100, 8191, 8192, 8193, 65_536 + 17, 300_001, 2_000_003])
    alpha = rng.choice([b"abcde ", b"abcdeABCDE \n.,1", bytes(range(256)), b"ab", b"aZ9 " * 3 + b"qwertyuiop"])
    rs = np.random.default_rng(seed)
    text = np.frombuffer(alpha, np.uint8)[rs.integers(0, len(alpha), n)].tobytes()
    try:
        oracle.histogram(text)
    except oracle.OracleError as e:   # a run of more than 255 letters: both sides must refuse it
        from paper_1411_5283_b200 import WSortError

        assert e.status == -7
        ws.load_text(text)
        with pytest.raises(WSortError) as g:
            ws.tokenize()
        assert g.value.status == -7
        return
    check(ws, text, algo)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_configs_exact(ws, cfg, algo):
    text, ntok = gen.generate(cfg)
    ref = check(ws, text, algo)
    assert ref.n_words == ntok


def test_deterministic_repeats(ws):
    text, _ = gen.generate(2)
    outs = [gpu_sort(ws, text) for _ in range(3)]
    assert all(o[0] == outs[0][0] and o[1] == outs[0][1] for o in outs)
    assert all(np.array_equal(o[2], outs[0][2]) for o in outs)


def test_auto_repeats_exact_c3_prefix_families(ws):
    """Races in the multi-chunk level 0 (k_msd_count0 / k_msd_scatter0 slices of several chunks, the ring
    of published chunk ids in K1) and the finishing jobs show up as run-to-run differences: AUTO is
    repeated on config 3 (64 MiB, every slice several chunks long) and on a text of long prefix
    families (config 5's shape: many chunks per class, wide keys, split jobs), each run byte-compared
    with the oracle."""
    text, _ = gen.generate(3)
    ref = oracle.sort(text, oracle.MERGE)
    fam = gen.generate(5, n=24 << 20)[0]
    ref5 = oracle.sort(fam, oracle.MERGE)
    for _ in range(3):
        for t, r in ((text, ref), (fam, ref5)):
            w, off, _ = gpu_sort(ws, t, "auto", src=False)
            assert off == r.off
            assert w == r.words


def test_tokenize_graph_replays_with_new_text(ws):
    """wsort_tokenize captures its launch sequence as a CUDA graph for a text size and replays it for the
    next text of the same size: different contents (and the COUNT / STAGE modes alternating) must each
    give the oracle's result."""
    a = gen.generate(2)[0]
    b = gen.generate(2, seed=77)[0]
    c = np.frombuffer(bytes(reversed(a.tobytes())), dtype=np.uint8)
    assert len(a) == len(b) == len(c)
    refs = {id(t): oracle.sort(t, oracle.MERGE) for t in (a, b, c)}
    for algo in ("dense_msd", "auto_count", "dense_msd"):
        for t in (a, b, c, a):
            w, off, _ = gpu_sort(ws, t, algo, src=False)
            assert off == refs[id(t)].off and w == refs[id(t)].words, algo


def test_auto_equals_radix(ws):
    text, _ = gen.generate(1)
    assert gpu_sort(ws, text, "auto")[0] == gpu_sort(ws, text, "lsd_radix")[0]
    assert gpu_sort(ws, text, "auto", src=False)[0] == gpu_sort(ws, text, "msd_radix", src=False)[0]
    assert gpu_sort(ws, text, "auto", src=False)[0] == gpu_sort(ws, text, "dense_msd", src=False)[0]


def test_dense_msd_repeat_sorts(ws):
    """One tokenize, several sorts: the dense tables and staged keys are read-only inputs of the sort."""
    text, _ = gen.generate(2)
    ref = oracle.sort(text, oracle.MERGE)
    ws.load_text(text)
    ws.tokenize()
    for algo in ("dense_msd", "lsd_radix", "dense_msd", "msd_oets", "auto"):
        ws.sort(algo)
        w, off = ws.fetch()
        assert w.tobytes() == ref.words and off == ref.off, algo


@pytest.mark.parametrize("algo", ALGOS)
def test_keys_only_path(ws, algo):
    """Without src_off the scatter and the sort take their keys-only (unordered-slot) paths."""
    text, _ = gen.generate(2)
    ref = oracle.sort(text, oracle.MERGE)
    words, off, _ = gpu_sort(ws, text, algo, src=False)
    assert words == ref.words and off == ref.off


# ---------------------------------------------------------------- ABI behaviour
def test_abi_state_machine_and_errors(ws, tmp_path):
    import ctypes

    from paper_1411_5283_b200 import WSort, WSortError, _lib as L

    w = WSort(0)
    with pytest.raises(WSortError) as e:
        w.tokenize()
    assert e.value.status == L.E_STATE
    w.load_text(b"b a")
    with pytest.raises(WSortError) as e:
        w.sort()
    assert e.value.status == L.E_STATE
    w.tokenize()
    assert w.offsets() == [0, 0, 2]
    r = L.Result()
    r.mem = L.MEM_HOST
    buf = (ctypes.c_uint8 * 16)()
    r.words = ctypes.addressof(buf)
    r.words_cap = 16
    assert w._lib.wsort_fetch(w._h, ctypes.byref(r)) == L.E_STATE      # words before sort
    w.sort()
    r.words_cap = 2
    assert w._lib.wsort_fetch(w._h, ctypes.byref(r)) == L.E_BUFFER_TOO_SMALL
    assert r.words_len == 4
    with pytest.raises(WSortError) as e:
        w.fetch(src_off=True)                                            # not requested
    assert e.value.status == L.E_STATE
    with pytest.raises(WSortError) as e:
        w.load_file(str(tmp_path / "missing.txt"))
    assert e.value.status == L.E_NOFILE
    p = tmp_path / "t.txt"
    p.write_bytes(b"To be, or not to be")
    w.load_file(str(p))
    w.tokenize()
    w.sort()
    assert w.fetch()[0].tobytes() == b"be\nbe\nor\nto\nto\nnot\n"
    with pytest.raises(WSortError) as e:
        w.sort("bogus_algo" if False else 7)
    assert e.value.status == L.E_INVALID_ARG
    w.close()


def test_device_text_and_device_fetch(ws):
    import torch

    text, _ = gen.generate(1)
    t = torch.from_numpy(text.copy()).cuda()
    ws.load_text(t)
    ws.tokenize()
    ws.sort()
    dw, off = ws.fetch_device()
    ref = oracle.sort(text, oracle.MERGE)
    assert dw.cpu().numpy().tobytes() == ref.words and off == ref.off


def test_fetch_async_pipeline(ws):
    """wsort_fetch_async + wsort_sync: two contexts in a pipeline (the e2e bench pattern) give the
    oracle's output for every text."""
    import torch

    from paper_1411_5283_b200 import WSort

    texts = [gen.generate(1)[0], gen.generate(2)[0], gen.generate(1)[0]]
    refs = [oracle.sort(t, oracle.MERGE) for t in texts]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ctxs = [WSort(0, stream=s.cuda_stream) for s in streams]
    outs = [np.empty(len(r.words) + 64, np.uint8) for r in refs]
    got = []
    try:
        ctxs[0].load_text(texts[0])
        for i, t in enumerate(texts):
            cur = ctxs[i % 2]
            cur.tokenize()
            if i + 1 < len(texts):
                ctxs[(i + 1) % 2].load_text(texts[i + 1])
            cur.sort("auto")
            got.append(cur.fetch_async(outs[i]))
        for c in ctxs:
            c.sync()
        for (w, off), r in zip(got, refs):
            assert off == r.off
            assert w.tobytes() == r.words
    finally:
        for c in ctxs:
            c.close()


# ---------------------------------------------------------------- no cliff for words of 67..255 letters
def test_very_long_words_stay_on_the_counting_path(ws):
    """Config 3 (8 MiB prefix) plus a few words of 67..255 letters: the hash-mode ingest counts them like any
    long word (no second text pass, no fallback to K3 + LSD), and the output is the oracle's."""
    base, _ = gen.generate(3, n=8 << 20)
    extra = b" " + b" ".join([b"Q" * 200, b"abc" * 40, b"z" * 67, b"Q" * 200, b"y" * 255]) + b" "
    text = np.concatenate([base, np.frombuffer(extra, np.uint8)])
    ref = oracle.sort(text, oracle.MERGE)
    ws.load_text(text)
    ws.tokenize()
    info = ws.ingest_info()
    ws.sort("auto")
    w, off = ws.fetch()
    assert off == ref.off and w.tobytes() == ref.words
    assert info["mode"] == 1 and info["overflow"] == 0


def test_many_distinct_very_long_words_fall_back(ws):
    """More distinct words of > 48 letters in one bucket than the wide-key rank sort holds: the library takes
    the staged / K3 path instead; the output is still the oracle's."""
    rng = np.random.default_rng(7)
    words = [bytes(rng.integers(97, 123, 200, dtype=np.uint8)) for _ in range(300)]
    text = b" ".join(words * 2 + [b"the", b"cat", b"sat", b"on", b"a", b"mat"] * 100)
    ref = oracle.sort(text, oracle.MERGE)
    ws.load_text(text)
    ws.tokenize()
    ws.sort("auto")
    w, off = ws.fetch()
    assert off == ref.off and w.tobytes() == ref.words


# ---------------------------------------------------------------- streamed ingest (NEXT-4)
@pytest.mark.parametrize("case", ["c1", "c2", "c3", "cross_every_step", "ends_mid_word", "empty", "long_words_65_255"])
def test_ingest_host_streamed_equals_oracle(ws, case):
    """wsort_ingest_host: the text copied to the device in stages under K1 (8 stages of K1 CTAs) gives the
    oracle's output (stage boundaries fall inside words: each stage copies 32 KiB beyond its range)."""
    import torch

    text = {"c1": lambda: gen.generate(1)[0], "c2": lambda: gen.generate(2)[0],
            "c3": lambda: gen.generate(3, n=24 << 20)[0]}.get(case, lambda: np.frombuffer(EDGE[case], np.uint8))()
    host = torch.from_numpy(np.ascontiguousarray(text)).pin_memory()
    ref = oracle.sort(text, oracle.MERGE)
    n = ws.ingest_host(host)
    assert n == ref.n_words
    ws.sort("auto")
    w, off = ws.fetch()
    assert off == ref.off and w.tobytes() == ref.words
