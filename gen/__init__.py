"""Seeded synthetic corpora for wsort (input generator only).

The paper's two datasets (§3 Methodology: Hamlet text files of
190 KB and 1.38 MB) are not available, so every input is synthetic, with the
shapes BASELINE.json's ``configs`` describe.
This module holds none of the method's arithmetic: it emits bytes only, and is
the one module that both ``oracle/`` users (tests, bench's cpu_baseline) and the
CUDA path's callers share.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwsortgen.so")

LEN_GEOM, LEN_FIXED, LEN_PREFIX_FAMILY = 0, 1, 2


class _Sub(ctypes.Structure):
    _fields_ = [
        ("V", ctypes.c_uint32),
        ("mode", ctypes.c_int),
        ("lmin", ctypes.c_int),
        ("lmax", ctypes.c_int),
        ("exclude_len", ctypes.c_int),
        ("p", ctypes.c_double),
        ("zipf_s", ctypes.c_double),
        ("mix", ctypes.c_double),
    ]


class _Params(ctypes.Structure):
    _fields_ = [
        ("nsub", ctypes.c_int),
        ("sub", _Sub * 3),
        ("cap_prob", ctypes.c_double),
        ("punct_prob", ctypes.c_double),
        ("punct_suffix_prob", ctypes.c_double),
        ("newline_prob", ctypes.c_double),
    ]


@dataclass
class SubVocab:
    V: int
    lmin: int = 1
    lmax: int = 16
    mode: int = LEN_GEOM
    exclude_len: int = 0
    p: float = 0.20
    zipf_s: float = 1.1
    mix: float = 1.0


@dataclass
class CorpusConfig:
    """One BASELINE.json config: N bytes, seed, vocabulary mix."""

    name: str
    n: int
    seed: int
    subs: list = field(default_factory=list)
    cap_prob: float = 0.10
    punct_prob: float = 0.12
    punct_suffix_prob: float = 0.75
    newline_prob: float = 1.0 / 12.0


# BASELINE.json configs[0..4]; sizes per DESIGN.md reading A14 (190·1024 B and ⌊1.38·2^20⌋ B).
CONFIGS = {
    1: CorpusConfig("c1-190KB", 194_560, 1, [SubVocab(5_000, 1, 16)]),
    2: CorpusConfig("c2-1.38MB", 1_447_034, 2, [SubVocab(12_000, 1, 18)]),
    3: CorpusConfig("c3-64MB", 64 << 20, 3, [SubVocab(200_000, 1, 24)]),
    4: CorpusConfig("c4-1GB", 1 << 30, 4, [SubVocab(1_000_000, 1, 32)]),
    5: CorpusConfig(
        "c5-8GB-adversarial",
        8 << 30,
        5,
        [
            SubVocab(400_000, 5, 5, mode=LEN_FIXED, mix=0.70),
            SubVocab(500_000, 13, 64, mode=LEN_PREFIX_FAMILY, mix=0.04),
            SubVocab(100_000, 1, 64, exclude_len=5, mix=0.26),
        ],
    ),
}

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        lib.wsort_gen_text.restype = ctypes.c_int
        lib.wsort_gen_text.argtypes = [
            ctypes.c_void_p,
            ctypes.c_uint64,
            ctypes.c_uint64,
            ctypes.POINTER(_Params),
            ctypes.c_int,
            ctypes.POINTER(ctypes.c_uint64),
        ]
        _lib = lib
    return _lib


def _params(cfg: CorpusConfig) -> _Params:
    P = _Params()
    P.nsub = len(cfg.subs)
    for i, s in enumerate(cfg.subs):
        P.sub[i] = _Sub(s.V, s.mode, s.lmin, s.lmax, s.exclude_len, s.p, s.zipf_s, s.mix)
    P.cap_prob = cfg.cap_prob
    P.punct_prob = cfg.punct_prob
    P.punct_suffix_prob = cfg.punct_suffix_prob
    P.newline_prob = cfg.newline_prob
    return P


def generate(config: int | CorpusConfig, n: int | None = None, seed: int | None = None,
             out: np.ndarray | None = None, threads: int | None = None):
    """Return (text: np.ndarray[uint8] of n bytes, n_tokens_emitted).

    ``n`` overrides the config size (a prefix-consistent-per-1MiB-block corpus
    with the same vocabulary); ``seed`` overrides the seed. ``out`` may be a
    preallocated (e.g. pinned) uint8 buffer of at least n bytes.
    """
    cfg = CONFIGS[config] if isinstance(config, int) else config
    n = cfg.n if n is None else int(n)
    seed = cfg.seed if seed is None else int(seed)
    if out is None:
        out = np.empty(n, dtype=np.uint8)
    assert out.dtype == np.uint8 and out.size >= n and out.flags["C_CONTIGUOUS"]
    threads = threads or max(1, min(os.cpu_count() or 1, 64))
    ntok = ctypes.c_uint64(0)
    P = _params(cfg)
    rc = _load().wsort_gen_text(out.ctypes.data if n else None, n, seed, ctypes.byref(P), threads, ctypes.byref(ntok))
    if rc != 0:
        raise RuntimeError(f"wsort_gen_text failed rc={rc}")
    return out[:n], int(ntok.value)
