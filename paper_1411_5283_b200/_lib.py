"""ctypes declarations of libwsort's C ABI (include/wsort.h). Argument marshalling only."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WSORT_LIB", os.path.join(_HERE, "libwsort.so"))   # override: experiments only

OK = 0
E_INVALID_ARG = -1
E_STATE = -2
E_NOMEM = -3
E_CUDA = -4
E_NCCL = -5
E_TOO_LARGE = -6
E_WORD_TOO_LONG = -7
E_BUFFER_TOO_SMALL = -8
E_NOFILE = -9
E_IO = -10

MEM_HOST = 0
MEM_DEVICE = 1

ALGO_AUTO = 0
ALGO_OETS_MERGE = 1
ALGO_LSD_RADIX = 2
ALGO_MSD_RADIX = 3
ALGO_MSD_OETS = 4
ALGO_DENSE_MSD = 5
ALGO_RAGGED = 6
ALGOS = {"auto": ALGO_AUTO, "oets_merge": ALGO_OETS_MERGE, "lsd_radix": ALGO_LSD_RADIX,
         "msd_radix": ALGO_MSD_RADIX, "msd_oets": ALGO_MSD_OETS, "dense_msd": ALGO_DENSE_MSD,
         "ragged": ALGO_RAGGED}

FLAG_SRC_OFF = 0x1
MAX_WORD_LEN = 255

# every symbol include/wsort.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "wsort_create", "wsort_set_stream", "wsort_load_text", "wsort_load_file", "wsort_tokenize",
    "wsort_sort", "wsort_fetch", "wsort_device_results", "wsort_last_error", "wsort_strerror",
    "wsort_destroy", "wsort_set_profiling", "wsort_kernel_stats", "wsort_reset_kernel_stats",
    "wsort_launch_count", "wsort_histogram", "wsort_pack", "wsort_sample", "wsort_select_splitters",
    "wsort_partition", "wsort_load_keys", "wsort_set_global", "wsort_fetch_async", "wsort_sync",
    "wsort_pack_long", "wsort_dense_range", "wsort_get_ingest_info", "wsort_get_unique_id", "wsort_attach_comm",
    "wsort_group_create", "wsort_group_destroy", "wsort_attach_group", "wsort_detach_comm", "wsort_get_slices", "wsort_set_ingest", "wsort_ingest_host",
]
INGEST = {"auto": 0, "stage": 1, "count": 2}
UNIQUE_ID_BYTES = 128


class Result(ctypes.Structure):
    _fields_ = [
        ("mem", ctypes.c_int),
        ("words", ctypes.c_void_p),
        ("words_cap", ctypes.c_uint64),
        ("words_len", ctypes.c_uint64),
        ("bucket_off", ctypes.c_void_p),
        ("bucket_cap", ctypes.c_uint32),
        ("max_len", ctypes.c_uint32),
        ("src_off", ctypes.c_void_p),
        ("src_cap", ctypes.c_uint64),
        ("n_words", ctypes.c_uint64),
        ("word_base", ctypes.c_uint64),
        ("byte_base", ctypes.c_uint64),
    ]


class IngestInfo(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int32),
        ("overflow", ctypes.c_uint32),
        ("distinct_narrow", ctypes.c_uint64),
        ("distinct_wide", ctypes.c_uint64),
        ("narrow_slots", ctypes.c_uint64),
        ("wide_slots", ctypes.c_uint64),
        ("grow", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
    ]


class Slice(ctypes.Structure):
    _fields_ = [
        ("local_byte", ctypes.c_uint64),
        ("bytes", ctypes.c_uint64),
        ("words", ctypes.c_uint64),
        ("global_byte", ctypes.c_uint64),
        ("global_word", ctypes.c_uint64),
    ]


class KernelStat(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 32),
        ("launches", ctypes.c_uint64),
        ("total_ms", ctypes.c_double),
        ("bytes", ctypes.c_double),
    ]


_lib = None


def load():
    """Load libwsort.so. Raises if it is missing: there is no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`. "
            "wsort has no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    P, U64, I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
    L.wsort_create.argtypes = [ctypes.POINTER(P), I, ctypes.c_size_t]
    L.wsort_set_stream.argtypes = [P, ctypes.c_size_t]
    L.wsort_load_text.argtypes = [P, P, U64, I, U64]
    L.wsort_load_file.argtypes = [P, ctypes.c_char_p]
    L.wsort_tokenize.argtypes = [P, ctypes.POINTER(U64)]
    L.wsort_sort.argtypes = [P, I, ctypes.c_uint]
    L.wsort_fetch.argtypes = [P, ctypes.POINTER(Result)]
    L.wsort_fetch_async.argtypes = [P, ctypes.POINTER(Result)]
    L.wsort_sync.argtypes = [P]
    L.wsort_device_results.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P)]
    L.wsort_last_error.argtypes = [P, ctypes.c_char_p, ctypes.c_size_t]
    L.wsort_strerror.argtypes = [I]
    L.wsort_strerror.restype = ctypes.c_char_p
    L.wsort_destroy.argtypes = [P]
    L.wsort_destroy.restype = None
    L.wsort_set_profiling.argtypes = [P, I]
    L.wsort_kernel_stats.argtypes = [P, ctypes.POINTER(KernelStat), I, ctypes.POINTER(I)]
    L.wsort_reset_kernel_stats.argtypes = [P]
    L.wsort_launch_count.argtypes = [P]
    L.wsort_launch_count.restype = U64
    L.wsort_histogram.argtypes = [P, P]
    L.wsort_get_ingest_info.argtypes = [P, P]
    L.wsort_set_ingest.argtypes = [P, I]
    L.wsort_ingest_host.argtypes = [P, P, U64, U64, ctypes.POINTER(U64)]
    L.wsort_get_unique_id.argtypes = [P]
    L.wsort_attach_comm.argtypes = [P, I, I, P]
    L.wsort_group_create.argtypes = [ctypes.POINTER(P), I]
    L.wsort_group_destroy.argtypes = [P]
    L.wsort_group_destroy.restype = None
    L.wsort_attach_group.argtypes = [P, P, I]
    L.wsort_detach_comm.argtypes = [P]
    L.wsort_get_slices.argtypes = [P, ctypes.POINTER(Slice), I, ctypes.POINTER(I)]
    L.wsort_pack.argtypes = [P]
    L.wsort_sample.argtypes = [P, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, P]
    L.wsort_select_splitters.argtypes = [P, U64, ctypes.c_uint32, ctypes.c_uint32, P]
    L.wsort_partition.argtypes = [P, P, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, P, U64, P, P]
    L.wsort_load_keys.argtypes = [P, P, P, ctypes.c_uint32]
    L.wsort_set_global.argtypes = [P, P, U64, U64]
    L.wsort_pack_long.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(U64)]
    L.wsort_dense_range.argtypes = [P, P, U64, U64]
    for name in EXPORTS:
        if name not in ("wsort_strerror", "wsort_destroy", "wsort_launch_count", "wsort_group_destroy"):
            getattr(L, name).restype = I
    _lib = L
    return L
