"""High-level Python API over libwsort (argument marshalling only).

    ws = WSort(device=0)                    # one context = one GPU stream + owned device scratch
    ws.load_text(text)                      # bytes / np.uint8 / torch.uint8 (host or cuda)
    n = ws.tokenize()                       # phases 1-2: K1 + K2
    ws.sort("auto", src_off=False)          # phase 3: K3 pack+scatter, K4 sort, K5 emit
    words, off = ws.fetch()                 # b"w\\n"*, off[0..Lmax+1]

or simply ``words, off = sort(text)``.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L


class WSortError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"wsort error {status} ({L.load().wsort_strerror(status).decode()}): {msg}")
        self.status = status


def _torch():
    import torch

    return torch


class WSort:
    """One libwsort context on one CUDA device."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._lib = L.load()
        h = ctypes.c_void_p()
        if stream is None:
            torch = _torch()
            if not torch.cuda.is_available():
                raise WSortError(L.E_CUDA, "no CUDA device (wsort has no CPU fallback)")
            with torch.cuda.device(device):
                stream = torch.cuda.current_stream(device).cuda_stream
        rc = self._lib.wsort_create(ctypes.byref(h), int(device), int(stream))
        if rc != L.OK:
            raise WSortError(rc, f"wsort_create(device={device})")
        self._h = h
        self.device = device
        self._src = False
        self._keep = None

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            self._lib.wsort_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc: int, what: str):
        if rc != L.OK:
            buf = ctypes.create_string_buffer(512)
            self._lib.wsort_last_error(self._h, buf, 512)
            raise WSortError(rc, f"{what}: {buf.value.decode(errors='replace')}")

    def set_stream(self, stream: int):
        self._check(self._lib.wsort_set_stream(self._h, int(stream)), "wsort_set_stream")

    # ------------------------------------------------------------------ pipeline
    def load_text(self, text, global_base: int = 0):
        """Copy `text` into the context (bytes, bytearray, numpy uint8 or torch uint8, host or cuda)."""
        mem, ptr, n, keep = _as_buffer(text)
        self._keep = keep   # host source must live until the next synchronising call
        self._check(self._lib.wsort_load_text(self._h, ptr, n, mem, int(global_base)), "wsort_load_text")

    def load_file(self, path: str):
        self._check(self._lib.wsort_load_file(self._h, path.encode()), "wsort_load_file")

    def tokenize(self) -> int:
        n = ctypes.c_uint64(0)
        rc = self._lib.wsort_tokenize(self._h, ctypes.byref(n))
        self._keep = None
        self._check(rc, "wsort_tokenize")
        return int(n.value)

    def sort(self, algo: str | int = "auto", src_off: bool = False):
        a = L.ALGOS[algo] if isinstance(algo, str) else int(algo)
        self._check(self._lib.wsort_sort(self._h, a, L.FLAG_SRC_OFF if src_off else 0), "wsort_sort")
        self._src = src_off

    def sizes(self) -> L.Result:
        r = L.Result()
        r.mem = L.MEM_HOST
        self._check(self._lib.wsort_fetch(self._h, ctypes.byref(r)), "wsort_fetch(sizes)")
        return r

    def offsets(self) -> list:
        """off[0..Lmax+1] (available after tokenize)."""
        r = self.sizes()
        off = np.zeros(r.max_len + 2, np.uint64)
        r.bucket_off = off.ctypes.data
        r.bucket_cap = off.size
        self._check(self._lib.wsort_fetch(self._h, ctypes.byref(r)), "wsort_fetch(off)")
        return [int(x) for x in off]

    def fetch(self, src_off: bool = False, out: np.ndarray | None = None):
        """Host results: (words: bytes-like, off: list[int]) or (words, off, src_off: np.uint64[W])."""
        r = self.sizes()
        words = out if out is not None else np.empty(max(r.words_len, 1), np.uint8)
        off = np.zeros(r.max_len + 2, np.uint64)
        src = np.empty(max(r.n_words, 1), np.uint64) if src_off else None
        r.words = words.ctypes.data
        r.words_cap = words.size
        r.bucket_off = off.ctypes.data
        r.bucket_cap = off.size
        if src_off:
            r.src_off = src.ctypes.data
            r.src_cap = src.size
        self._check(self._lib.wsort_fetch(self._h, ctypes.byref(r)), "wsort_fetch")
        w = words[: r.words_len]
        offl = [int(x) for x in off]
        if src_off:
            return w, offl, src[: r.n_words]
        return w, offl

    def fetch_async(self, out: np.ndarray):
        """Enqueue the copy of the sorted words into `out` (pinned host or any host uint8 array of at least
        words_len bytes); returns (words view, off). `out` holds the words after sync()."""
        r = self.sizes()
        off = np.zeros(r.max_len + 2, np.uint64)
        r.words = out.ctypes.data
        r.words_cap = out.size
        r.bucket_off = off.ctypes.data
        r.bucket_cap = off.size
        self._check(self._lib.wsort_fetch_async(self._h, ctypes.byref(r)), "wsort_fetch_async")
        return out[: r.words_len], [int(x) for x in off]

    def sync(self):
        self._check(self._lib.wsort_sync(self._h), "wsort_sync")

    def fetch_device(self):
        """(words: torch.uint8 cuda tensor (a copy), off: list[int])."""
        torch = _torch()
        r = self.sizes()
        words = torch.empty(max(r.words_len, 1), dtype=torch.uint8, device=f"cuda:{self.device}")
        off = np.zeros(r.max_len + 2, np.uint64)
        rr = L.Result()
        rr.mem = L.MEM_DEVICE
        rr.words = words.data_ptr()
        rr.words_cap = words.numel()
        self._check(self._lib.wsort_fetch(self._h, ctypes.byref(rr)), "wsort_fetch(device)")
        return words[: r.words_len], self.offsets()

    # ------------------------------------------------------------------ multi-GPU stages (dist.py)
    torch_device = property(lambda self: f"cuda:{self.device}")

    def histogram(self) -> np.ndarray:
        h = np.zeros(256, np.uint64)
        self._check(self._lib.wsort_histogram(self._h, h.ctypes.data), "wsort_histogram")
        return h

    def pack(self):
        self._check(self._lib.wsort_pack(self._h), "wsort_pack")

    def pack_long(self):
        """Split variant: pack the words of >= 6 letters; returns the context's dense count table as a
        zero-copy cuda int32 tensor (u32 counts; the caller may all-reduce it in place)."""
        torch = _torch()
        p = ctypes.c_void_p()
        n = ctypes.c_uint64(0)
        self._check(self._lib.wsort_pack_long(self._h, ctypes.byref(p), ctypes.byref(n)), "wsort_pack_long")
        return torch.as_tensor(_DeviceArray(p.value, int(n.value)), device=self.torch_device)

    def dense_range(self, ghist: np.ndarray, lo: int, hi: int):
        g = np.ascontiguousarray(ghist, dtype=np.uint64)
        self._check(self._lib.wsort_dense_range(self._h, g.ctypes.data, int(lo), int(hi)), "wsort_dense_range")

    def sample(self, nsamples: int, rank: int, rec_words: int, out):
        """Write nsamples sample records into `out` (cuda int32/uint32 tensor [nsamples, rec_words])."""
        assert out.is_cuda and out.numel() >= nsamples * rec_words
        self._check(self._lib.wsort_sample(self._h, nsamples, rank, rec_words, out.data_ptr()), "wsort_sample")

    def partition(self, splitters: np.ndarray, nparts: int, rec_words: int, rank: int, send):
        """Partition packed keys into `send` (cuda int32 tensor); returns (counts[P,256], send_words[P])."""
        sp = np.ascontiguousarray(splitters, dtype=np.uint32)
        counts = np.zeros((nparts, 256), np.uint64)
        sw = np.zeros(nparts, np.uint64)
        self._check(self._lib.wsort_partition(self._h, sp.ctypes.data if sp.size else None, nparts, rec_words, rank,
                                              send.data_ptr(), send.numel(), counts.ctypes.data, sw.ctypes.data),
                    "wsort_partition")
        return counts, sw

    def load_keys(self, recv, counts: np.ndarray):
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        self._check(self._lib.wsort_load_keys(self._h, recv.data_ptr() if recv.numel() else None, c.ctypes.data,
                                              c.shape[0]), "wsort_load_keys")

    def set_global(self, ghist: np.ndarray, word_base: int, byte_base: int):
        g = np.ascontiguousarray(ghist, dtype=np.uint64)
        self._check(self._lib.wsort_set_global(self._h, g.ctypes.data, int(word_base), int(byte_base)), "wsort_set_global")

    # ------------------------------------------------------------------ measurement
    def set_profiling(self, on):
        """False / True (per-kernel CUDA events) / 2 (also every kernel on the context's stream)."""
        self._check(self._lib.wsort_set_profiling(self._h, 2 if on == 2 else (1 if on else 0)), "wsort_set_profiling")

    def kernel_stats(self) -> dict:
        arr = (L.KernelStat * 64)()
        n = ctypes.c_int(0)
        self._check(self._lib.wsort_kernel_stats(self._h, arr, 64, ctypes.byref(n)), "wsort_kernel_stats")
        return {arr[i].name.decode(): {"launches": int(arr[i].launches), "ms": arr[i].total_ms,
                                       "bytes": arr[i].bytes} for i in range(n.value)}

    def reset_kernel_stats(self):
        self._check(self._lib.wsort_reset_kernel_stats(self._h), "wsort_reset_kernel_stats")

    def ingest_host(self, text, global_base: int = 0) -> int:
        """load_text + tokenize of a HOST text with the copy streamed under K1 (wsort_ingest_host)."""
        mem, ptr, n, keep = _as_buffer(text)
        if mem != L.MEM_HOST:
            raise ValueError("ingest_host takes host memory")
        nw = ctypes.c_uint64(0)
        self._check(self._lib.wsort_ingest_host(self._h, ptr, n, int(global_base), ctypes.byref(nw)), "wsort_ingest_host")
        return int(nw.value)

    def set_ingest(self, mode: str):
        """"auto" (default), "stage" or "count" (include/wsort.h wsort_set_ingest)."""
        self._check(self._lib.wsort_set_ingest(self._h, L.INGEST[mode]), "wsort_set_ingest")

    def ingest_info(self) -> dict:
        """How the last tokenize counted the words of >= 6 letters (wsort_get_ingest_info)."""
        info = L.IngestInfo()
        self._check(self._lib.wsort_get_ingest_info(self._h, ctypes.byref(info)), "wsort_get_ingest_info")
        return {k: int(getattr(info, k)) for k, _ in L.IngestInfo._fields_}

    # ---- multi-GPU with the library-owned communicator (include/wsort.h) ----
    def attach_comm(self, rank: int, nranks: int, unique_id: bytes):
        """Rank `rank` of `nranks` (one process per GPU, NCCL); collective over the ranks."""
        buf = (ctypes.c_uint8 * L.UNIQUE_ID_BYTES).from_buffer_copy(bytes(unique_id))
        self._check(self._lib.wsort_attach_comm(self._h, rank, nranks, buf), "wsort_attach_comm")

    def attach_group(self, group: "Group", rank: int):
        """Rank `rank` of an in-process group (one thread per rank); collective over the group's threads."""
        self._check(self._lib.wsort_attach_group(self._h, group._h, rank), "wsort_attach_group")

    def detach(self):
        self._check(self._lib.wsort_detach_comm(self._h), "wsort_detach_comm")

    def slices(self) -> list:
        """[(local byte, bytes, words, global byte, global word)] of this context's output."""
        out = (L.Slice * 4)()
        n = ctypes.c_int(0)
        self._check(self._lib.wsort_get_slices(self._h, out, 4, ctypes.byref(n)), "wsort_get_slices")
        return [(int(x.local_byte), int(x.bytes), int(x.words), int(x.global_byte), int(x.global_word))
                for x in out[: n.value]]

    def launch_count(self) -> int:
        return int(self._lib.wsort_launch_count(self._h))


def get_unique_id() -> bytes:
    """NCCL unique id for attach_comm (rank 0; broadcast it to the other ranks)."""
    lib = L.load()
    buf = (ctypes.c_uint8 * L.UNIQUE_ID_BYTES)()
    rc = lib.wsort_get_unique_id(buf)
    if rc:
        raise WSortError(rc, "wsort_get_unique_id")
    return bytes(buf)


class Group:
    """In-process ranks (include/wsort.h wsort_group): one WSort per rank, each driven by its own thread."""

    def __init__(self, nranks: int):
        self._lib = L.load()
        h = ctypes.c_void_p()
        rc = self._lib.wsort_group_create(ctypes.byref(h), nranks)
        if rc:
            raise WSortError(rc, "wsort_group_create")
        self._h, self.nranks = h, nranks

    def close(self):
        if self._h:
            self._lib.wsort_group_destroy(self._h)
            self._h = None


def select_splitters(samples: np.ndarray, nparts: int) -> np.ndarray:
    """Host-side splitter choice (libwsort wsort_select_splitters): records sorted by (L, key, rank)."""
    lib = L.load()
    smp = np.ascontiguousarray(samples, dtype=np.uint32)
    n, rw = smp.shape
    out = np.zeros((max(nparts - 1, 0), rw), np.uint32)
    if nparts > 1:
        rc = lib.wsort_select_splitters(smp.ctypes.data, n, rw, nparts, out.ctypes.data)
        if rc != L.OK:
            raise WSortError(rc, "wsort_select_splitters")
    return out


class _DeviceArray:
    """A library-owned device int32 array, exposed to torch through __cuda_array_interface__."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr or 0, False),
                                         "strides": None, "version": 2}


def _as_buffer(text):
    """(mem, pointer, nbytes, keepalive) for bytes / numpy / torch inputs."""
    if isinstance(text, (bytes, bytearray, memoryview)):
        a = np.frombuffer(bytes(text), dtype=np.uint8)
        return L.MEM_HOST, (a.ctypes.data if a.size else None), a.size, a
    if isinstance(text, np.ndarray):
        a = np.ascontiguousarray(text).view(np.uint8).reshape(-1)
        return L.MEM_HOST, (a.ctypes.data if a.size else None), a.size, a
    torch = _torch()
    if isinstance(text, torch.Tensor):
        t = text.contiguous().view(torch.uint8).reshape(-1)
        mem = L.MEM_DEVICE if t.is_cuda else L.MEM_HOST
        return mem, (t.data_ptr() if t.numel() else None), t.numel(), t
    raise TypeError(f"unsupported text type {type(text)}")


def sort(text, algo: str = "auto", src_off: bool = False, device: int = 0):
    """One-shot: (words: bytes, bucket_off: list[int]) [+ src_off] for `text` on cuda:`device`."""
    with WSort(device) as ws:
        ws.load_text(text)
        ws.tokenize()
        ws.sort(algo, src_off=src_off)
        res = ws.fetch(src_off=src_off)
        return (res[0].tobytes(),) + tuple(res[1:])
