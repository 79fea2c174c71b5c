"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/wsort_oracle.c) is pinned to things other than itself:
  * hand-worked golden fixtures (tests/golden/*.json, each with its citation);
  * a library routine: Python's `re.findall(rb'[A-Za-z]+')` + `sorted(key=(len, bytes))`
    (independent tokenizer and sort, not a retyping of the C code);
  * closed forms: bubble-sort comparison counts n(n-1)/2, SPEC.md:158-170 examples,
    the chunked count p*(n/p)(n/p-1)/2, the ChunkPlan examples;
  * invariants: permutation, sortedness, off = histogram prefix sums, bytes in a-z or '\\n';
  * brute force / cross-method agreement: bubble == merge == qsort on random corpora.
"""
import glob
import json
import os
import random
import re

import numpy as np
import pytest

import oracle
from conftest import GOLDEN


def py_reference(text: bytes):
    """Library-routine pin: regex tokenizer + Python's stable sorted() on (len, bytes)."""
    toks = [(m.start(), m.group().lower()) for m in re.finditer(rb"[A-Za-z]+", text)]
    order = sorted(toks, key=lambda t: (len(t[1]), t[1]))  # stable: ties keep source order
    words = b"".join(w + b"\n" for _, w in order)
    lmax = max((len(w) for _, w in toks), default=0)
    hist = [0] * (lmax + 1)
    for _, w in toks:
        hist[len(w)] += 1
    off = [0]
    for L in range(lmax + 1):
        off.append(off[-1] + hist[L])
    return words, off, [p for p, _ in order]


def load_golden():
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.json"))):
        d = json.load(open(p))
        if "text_latin1" in d:
            out.append(d)
    return out


GOLD = load_golden()


@pytest.mark.parametrize("fx", GOLD, ids=[g["name"] for g in GOLD])
@pytest.mark.parametrize("method", [oracle.BUBBLE, oracle.MERGE, oracle.BRUTE])
def test_golden_fixtures(fx, method):
    text = fx["text_latin1"].encode("latin-1")
    out = oracle.sort(text, method, want_src=True)
    assert out.words == b"".join(w.encode() + b"\n" for w in fx["words"])
    assert out.off == fx["off"]
    assert [int(x) for x in out.src_off] == fx["src_off"]
    assert out.n_words == len(fx["words"])


def test_golden_fixtures_agree_with_library_routine():
    # the fixtures themselves are re-derived by an independent implementation
    for fx in GOLD:
        text = fx["text_latin1"].encode("latin-1")
        words, off, src = py_reference(text)
        assert words == b"".join(w.encode() + b"\n" for w in fx["words"]), fx["name"]
        assert off == fx["off"], fx["name"]
        assert src == fx["src_off"], fx["name"]


def _rand_text(rng: random.Random, n: int, alphabet: bytes) -> bytes:
    return bytes(rng.choice(alphabet) for _ in range(n))


@pytest.mark.parametrize("seed", range(40))
def test_tokenizer_all_byte_values_vs_regex(seed):
    rng = random.Random(seed)
    # every byte value 0..255 can appear; letters boosted so words form
    alpha = bytes(range(256)) + b"abcxyzABCXYZ" * 20
    text = _rand_text(rng, rng.randint(0, 3000), alpha)
    pos, ln = oracle.tokenize(text)
    ref = [(m.start(), m.end() - m.start()) for m in re.finditer(rb"[A-Za-z]+", text)]
    assert list(zip(pos.tolist(), ln.tolist())) == ref


@pytest.mark.parametrize("seed", range(200))
def test_random_ae_corpora_all_methods_vs_library_routine(seed):
    """SPEC.md:431 (200 randomized corpora over alphabet a-e) — bubble == merge == brute == sorted()."""
    rng = random.Random(1000 + seed)
    text = _rand_text(rng, rng.randint(0, 1500), b"abcdeABCDE  \n,.'1")
    words, off, src = py_reference(text)
    for m in (oracle.BUBBLE, oracle.MERGE, oracle.BRUTE):
        o = oracle.sort(text, m, want_src=True)
        assert o.words == words and o.off == off and o.src_off.tolist() == src
    assert oracle.verify(text, words, off) == 0


def test_config1_bubble_merge_brute_agree():
    import gen

    text, _ = gen.generate(1)
    b = oracle.sort(text, oracle.BUBBLE, want_src=True)
    m = oracle.sort(text, oracle.MERGE, want_src=True)
    q = oracle.sort(text, oracle.BRUTE, want_src=True)
    assert b.words == m.words == q.words
    assert b.off == m.off == q.off
    assert np.array_equal(b.src_off, m.src_off) and np.array_equal(m.src_off, q.src_off)
    words, off, src = py_reference(text.tobytes())
    assert m.words == words and m.off == off and m.src_off.tolist() == src
    assert oracle.verify(text, m.words, m.off) == 0


def test_config2_merge_vs_library_routine():
    import gen

    text, _ = gen.generate(2)
    m = oracle.sort(text, oracle.MERGE)
    words, off, _ = py_reference(text.tobytes())
    assert m.words == words and m.off == off


# ---------------------------------------------------------------- bubble closed forms
def _words_text(words):
    return " ".join(words).encode()


def test_bubble_spec_examples():
    # [3,1,2] -> swaps 2; comparisons 3 and passes 2 follow from the shrinking range
    o = oracle.sort(_words_text(["c", "a", "b"]), oracle.BUBBLE)
    assert o.words == b"a\nb\nc\n" and (o.swaps, o.comparisons, o.passes) == (2, 3, 2)
    # reverse-sorted n=5 -> comparisons = 10 = n(n-1)/2
    o = oracle.sort(_words_text(list("edcba")), oracle.BUBBLE)
    assert (o.comparisons, o.passes, o.swaps) == (10, 4, 10)
    # sorted n=5 -> passes 1, comparisons 4, swaps 0
    o = oracle.sort(_words_text(list("abcde")), oracle.BUBBLE)
    assert (o.comparisons, o.passes, o.swaps) == (4, 1, 0)
    # SURVEY hand example: bucket L=1 of the zebra fixture is [a, s, a] -> comparisons 3, swaps 1, passes 2
    o = oracle.sort(b"a s a", oracle.BUBBLE)
    assert (o.comparisons, o.swaps, o.passes) == (3, 1, 2)


def _distinct_words(n, L=2):
    letters = "abcdefghijklmnopqrstuvwxyz"
    out = []
    for i in range(n):
        w = ""
        x = i
        for _ in range(L):
            w = letters[x % 26] + w
            x //= 26
        out.append(w)
    return out


def test_bubble_worst_case_exhaustive_0_200():
    """PAPER.md:50 "n(n-1)/2"; strictly reverse-sorted distinct input, n in [0,200]."""
    for n in range(0, 201):
        ws = list(reversed(_distinct_words(n)))
        o = oracle.sort(_words_text(ws), oracle.BUBBLE)
        assert o.comparisons == n * (n - 1) // 2, n
        assert o.swaps == n * (n - 1) // 2


def test_paper_mpi_chunk_comparisons_n4096():
    """n=4096 reverse-sorted distinct, p in {2,4,8,16}: worker comparisons p*(n/p)(n/p-1)/2."""
    n = 4096
    ws = list(reversed(_distinct_words(n, L=3)))
    text = _words_text(ws)
    seq = oracle.sort(text, oracle.BUBBLE)
    assert seq.comparisons == n * (n - 1) // 2 == 8_386_560
    expect = {2: 4_192_256, 4: 2_095_104, 8: 1_046_528, 16: 522_240}
    for p, e in expect.items():
        o = oracle.sort_paper_mpi(text, p, oracle.BUBBLE)
        assert o.comparisons == p * (n // p) * (n // p - 1) // 2 == e
        assert o.words == seq.words


@pytest.mark.parametrize("seed", range(20))
def test_paper_mpi_equals_sequential(seed):
    rng = random.Random(seed)
    text = _rand_text(rng, rng.randint(0, 4000), b"abcdeABCDE  \n,.")
    seq = oracle.sort(text, oracle.MERGE)
    for p in (1, 2, 3, 4, 7):
        for inner in (oracle.BUBBLE, oracle.MERGE):
            o = oracle.sort_paper_mpi(text, p, inner)
            assert o.words == seq.words and o.off == seq.off


def test_partition_examples():
    # 40 elements, 4 processors -> chunk 10; 2 processors -> 20
    assert oracle.partition(40, 4) == [0, 10, 20, 30, 40]
    assert oracle.partition(40, 2) == [0, 20, 40]
    # (10, 3) -> sizes [4, 3, 3]
    assert oracle.partition(10, 3) == [0, 4, 7, 10]
    for n in range(0, 300, 7):
        for p in range(1, 20):
            b = oracle.partition(n, p)
            sizes = [b[i + 1] - b[i] for i in range(p)]
            assert b[0] == 0 and b[-1] == n and max(sizes) - min(sizes) <= 1
            assert sizes == sorted(sizes, reverse=True)


# ---------------------------------------------------------------- errors, invariants, verify
def test_max_word_length_255_ok_256_error():
    w255 = b"q" * 255
    o = oracle.sort(b"ab " + w255 + b" c", oracle.MERGE)
    assert o.max_len == 255 and o.words == b"c\nab\n" + w255 + b"\n"
    assert len(o.off) == 257 and o.off[-1] == 3
    with pytest.raises(oracle.OracleError) as e:
        oracle.sort(b"x " + b"Q" * 256, oracle.MERGE)
    assert e.value.status == oracle.E_WORD_TOO_LONG


def test_invariants_on_config1():
    import gen

    text, _ = gen.generate(1)
    o = oracle.sort(text, oracle.MERGE)
    hist, off, lmax = oracle.histogram(text)
    assert o.off == [int(x) for x in off[: lmax + 2]]
    assert o.off[-1] == o.n_words
    C = sum(L * int(hist[L]) for L in range(256))
    assert len(o.words) == C + o.n_words
    assert set(o.words) <= set(b"abcdefghijklmnopqrstuvwxyz\n")
    lines = o.words.split(b"\n")[:-1]
    assert all(len(a) < len(b) or (len(a) == len(b) and a <= b) for a, b in zip(lines, lines[1:]))
    # multiset = the text's tokens
    assert sorted(lines) == sorted(m.lower() for m in re.findall(rb"[A-Za-z]+", text.tobytes()))


def test_verify_detects_errors():
    text = b"the cat sat on the mat with a hat"
    o = oracle.sort(text, oracle.MERGE)
    assert oracle.verify(text, o.words, o.off) == 0
    lines = o.words.split(b"\n")[:-1]
    swapped = lines[:]
    swapped[-1], swapped[-2] = swapped[-2], swapped[-1]
    assert oracle.verify(text, b"".join(x + b"\n" for x in swapped), o.off) > 0
    assert oracle.verify(text, b"".join(x + b"\n" for x in lines[1:]), o.off) != 0
    bad_off = list(o.off)
    bad_off[2] += 1
    assert oracle.verify(text, o.words, bad_off) != 0
    # same sortedness and counts, different multiset: replace a word by another of equal length
    mutated = o.words.replace(b"cat", b"cau")
    assert oracle.verify(text, mutated, o.off) != 0


def test_fingerprint_is_order_independent():
    a = oracle.fingerprint(b"b a c a")
    assert a == oracle.fingerprint(b"A, C; a b")
    assert a == oracle.fingerprint_words(b"a\na\nb\nc\n")
    assert a != oracle.fingerprint(b"a a b d")


@pytest.mark.parametrize("seed", range(12))
def test_sort_length_vs_library_routine(seed):
    """oracle_sort_length (one sub-array, paper-mpi shape) against regex + sorted() per length, and its
    concatenation over the lengths against the whole-text oracle (the full-size golden script relies on
    this: tools/golden_full_size.py)."""
    rng = np.random.default_rng(seed)
    alpha = [b"abcde ", b"aAbB \n.,", b"the quick brown fox jumps over a lazy dog ", bytes(range(256))][seed % 4]
    text = np.frombuffer(alpha, np.uint8)[rng.integers(0, len(alpha), 1 + seed * 9973)].tobytes()
    ref_words, ref_off, _ = py_reference(text)
    toks = [m.group().lower() for m in re.finditer(rb"[A-Za-z]+", text)]
    lmax = max((len(w) for w in toks), default=0)
    p = [1, 2, 3, 8][seed % 4]
    parts = []
    for L in range(1, lmax + 2):
        got = oracle.sort_length(text, L, p)
        assert got == b"".join(w + b"\n" for w in sorted(w for w in toks if len(w) == L))
        parts.append(got)
    assert b"".join(parts) == ref_words


def test_sort_length_concat_equals_sort_config2():
    import gen

    text, _ = gen.generate(2)
    ref = oracle.sort(text, oracle.MERGE)
    assert b"".join(oracle.sort_length(text, L, 4) for L in range(1, ref.max_len + 1)) == ref.words
    with pytest.raises(oracle.OracleError):
        oracle.sort_length(b"ok " + b"z" * 256, 2)


@pytest.mark.parametrize("ranges", [[(1, 3), (4, 4), (5, 255)], [(1, 255)], [(1, 1), (2, 9), (10, 40), (41, 255)]])
def test_sort_lengths_ranges_concat(ranges):
    text = np.frombuffer(b" ".join(bytes([97 + (i * j * 7 + j) % 26 for j in range(1 + i % 45)]) * (1 + i % 3)
                                   for i in range(3000)), np.uint8)
    ref_words, _, _ = py_reference(text.tobytes())
    assert b"".join(oracle.sort_lengths(text, a, b, 3) for a, b in ranges) == ref_words
