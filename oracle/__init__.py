"""ctypes binding of the CPU oracle (oracle/wsort_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` arm may import this module. The product
package (paper_1411_5283_b200) never imports it, and the two share no code.
Every function cites the passage it follows in wsort_oracle.c.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

BUBBLE, MERGE, BRUTE = 0, 1, 2
E_WORD_TOO_LONG = -7


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what} failed with status {status}")
        self.status = status


class _Stats(ctypes.Structure):
    _fields_ = [("comparisons", ctypes.c_uint64), ("swaps", ctypes.c_uint64), ("passes", ctypes.c_uint64)]


class _Result(ctypes.Structure):
    _fields_ = [("n_words", ctypes.c_uint64), ("words_len", ctypes.c_uint64), ("max_len", ctypes.c_uint32)]


_lib = None
_P = ctypes.c_void_p
_U64 = ctypes.c_uint64


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_tokenize.restype = ctypes.c_int64
        L.oracle_tokenize.argtypes = [_P, _U64, _P, _P, _U64]
        L.oracle_histogram.restype = ctypes.c_int
        L.oracle_histogram.argtypes = [_P, _U64, _P, _P]
        L.oracle_sort.restype = ctypes.c_int
        L.oracle_sort.argtypes = [_P, _U64, ctypes.c_int, _P, _U64, _P, _P, _U64,
                                  ctypes.POINTER(_Result), ctypes.POINTER(_Stats)]
        L.oracle_sort_paper_mpi.restype = ctypes.c_int
        L.oracle_sort_paper_mpi.argtypes = [_P, _U64, ctypes.c_uint32, ctypes.c_int, _P, _U64, _P,
                                            ctypes.POINTER(_Result), ctypes.POINTER(_Stats)]
        L.oracle_sort_lengths.restype = ctypes.c_int
        L.oracle_sort_lengths.argtypes = [_P, _U64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _P, _U64,
                                          ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_partition.restype = None
        L.oracle_partition.argtypes = [_U64, ctypes.c_uint32, _P]
        L.oracle_fingerprint.restype = ctypes.c_int
        L.oracle_fingerprint.argtypes = [_P, _U64, _P]
        L.oracle_fingerprint_words.restype = ctypes.c_int
        L.oracle_fingerprint_words.argtypes = [_P, _U64, _P]
        L.oracle_verify.restype = ctypes.c_int64
        L.oracle_verify.argtypes = [_P, _U64, _P, _U64, _P, ctypes.c_uint32]
        _lib = L
    return _lib


def _buf(text) -> np.ndarray:
    if isinstance(text, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(text), dtype=np.uint8)
    a = np.ascontiguousarray(text, dtype=np.uint8)
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


@dataclass
class OracleOutput:
    words: bytes           # "w\n" per word, (length, alphabetical) order
    off: list              # off[0..Lmax+1]
    src_off: np.ndarray | None
    n_words: int
    max_len: int
    comparisons: int
    swaps: int
    passes: int


def tokenize(text):
    """(pos uint64[W], len uint32[W]) of every word, text order (phase 1)."""
    t = _buf(text)
    L = _load()
    w = L.oracle_tokenize(_ptr(t), t.size, None, None, 0)
    if w < 0:
        raise OracleError(w, "oracle_tokenize")
    pos = np.empty(max(w, 1), np.uint64)
    ln = np.empty(max(w, 1), np.uint32)
    w2 = L.oracle_tokenize(_ptr(t), t.size, pos.ctypes.data, ln.ctypes.data, w)
    assert w2 == w
    return pos[:w], ln[:w]


def histogram(text):
    """(hist[256], off[257], Lmax) — PAPER.md:13 sub-array sizes."""
    t = _buf(text)
    hist = np.zeros(256, np.uint64)
    off = np.zeros(257, np.uint64)
    lmax = _load().oracle_histogram(_ptr(t), t.size, hist.ctypes.data, off.ctypes.data)
    if lmax < 0:
        raise OracleError(lmax, "oracle_histogram")
    return hist, off, lmax


def sort(text, method: int = MERGE, want_src: bool = False) -> OracleOutput:
    """Full oracle: tokenize → bucket by length → sort each bucket → emit."""
    t = _buf(text)
    L = _load()
    res = _Result()
    st = _Stats()
    off = np.zeros(257, np.uint64)
    rc = L.oracle_sort(_ptr(t), t.size, method, None, 0, off.ctypes.data, None, 0, ctypes.byref(res), ctypes.byref(st))
    if rc < 0:
        raise OracleError(rc, "oracle_sort(size)")
    words = np.empty(max(res.words_len, 1), np.uint8)
    src = np.empty(max(res.n_words, 1), np.uint64) if want_src else None
    rc = L.oracle_sort(_ptr(t), t.size, method, words.ctypes.data, res.words_len, off.ctypes.data,
                       src.ctypes.data if want_src else None, res.n_words, ctypes.byref(res), ctypes.byref(st))
    if rc < 0:
        raise OracleError(rc, "oracle_sort")
    return OracleOutput(words[: res.words_len].tobytes(), [int(x) for x in off[: res.max_len + 2]],
                        src[: res.n_words] if want_src else None, res.n_words, res.max_len,
                        st.comparisons, st.swaps, st.passes)


def sort_paper_mpi(text, p: int, inner: int = BUBBLE) -> OracleOutput:
    """paper-mpi shape: per bucket, p chunks sorted on p threads, k-way merge."""
    t = _buf(text)
    L = _load()
    res = _Result()
    st = _Stats()
    off = np.zeros(257, np.uint64)
    rc = L.oracle_sort_paper_mpi(_ptr(t), t.size, p, inner, None, 0, off.ctypes.data, ctypes.byref(res), ctypes.byref(st))
    if rc < 0:
        raise OracleError(rc, "oracle_sort_paper_mpi(size)")
    words = np.empty(max(res.words_len, 1), np.uint8)
    rc = L.oracle_sort_paper_mpi(_ptr(t), t.size, p, inner, words.ctypes.data, res.words_len, off.ctypes.data,
                                 ctypes.byref(res), ctypes.byref(st))
    if rc < 0:
        raise OracleError(rc, "oracle_sort_paper_mpi")
    return OracleOutput(words[: res.words_len].tobytes(), [int(x) for x in off[: res.max_len + 2]], None,
                        res.n_words, res.max_len, st.comparisons, st.swaps, st.passes)


def sort_lengths(text, lmin: int, lmax: int, p: int = 1, as_array: bool = False):
    """The sorted sub-arrays of the words of lengths lmin..lmax as "w\\n" bytes, shorter first (PAPER.md:58
    phases 2-3 for those lengths, paper-mpi shape on p threads). Concatenated over consecutive length
    ranges it is sort(text).words (length-major)."""
    t = _buf(text)
    lib = _load()
    nw, nb = ctypes.c_uint64(0), ctypes.c_uint64(0)
    rc = lib.oracle_sort_lengths(_ptr(t), t.size, lmin, lmax, p, None, 0, ctypes.byref(nw), ctypes.byref(nb))
    if rc < 0:
        raise OracleError(rc, "oracle_sort_lengths(size)")
    out = np.empty(max(nb.value, 1), np.uint8)
    rc = lib.oracle_sort_lengths(_ptr(t), t.size, lmin, lmax, p, out.ctypes.data, out.size, ctypes.byref(nw),
                                 ctypes.byref(nb))
    if rc < 0:
        raise OracleError(rc, "oracle_sort_lengths")
    out = out[: nb.value]
    return out if as_array else out.tobytes()


def sort_length(text, L: int, p: int = 1) -> bytes:
    """The sorted sub-array of the words of length L (sort_lengths(text, L, L, p))."""
    return sort_lengths(text, L, L, p)


def partition(n: int, p: int) -> list:
    """ChunkPlan bounds[0..p] (remainder to the lowest chunks)."""
    b = np.zeros(p + 1, np.uint64)
    _load().oracle_partition(n, p, b.ctypes.data)
    return [int(x) for x in b]


def fingerprint(text) -> tuple:
    t = _buf(text)
    fp = np.zeros(2, np.uint64)
    rc = _load().oracle_fingerprint(_ptr(t), t.size, fp.ctypes.data)
    if rc < 0:
        raise OracleError(rc, "oracle_fingerprint")
    return int(fp[0]), int(fp[1])


def fingerprint_words(words) -> tuple:
    w = _buf(words)
    fp = np.zeros(2, np.uint64)
    rc = _load().oracle_fingerprint_words(_ptr(w), w.size, fp.ctypes.data)
    if rc < 0:
        raise OracleError(rc, "oracle_fingerprint_words")
    return int(fp[0]), int(fp[1])


def verify(text, words, off) -> int:
    """0 if `words`/`off` is THE sorted output of `text` (sorted, offsets, multiset); else >0 = 1+first bad
    word index, <0 = structural failure (SPEC.md:398-411 cmd_verify, restated)."""
    t = _buf(text)
    w = _buf(words)
    o = np.ascontiguousarray(np.asarray(off, dtype=np.uint64))
    return int(_load().oracle_verify(_ptr(t), t.size, _ptr(w), w.size, o.ctypes.data, o.size))
