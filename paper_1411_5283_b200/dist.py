"""Multi-GPU orchestration: byte-range shards + one sample-sort exchange.

One process per GPU (torchrun); torch.distributed (NCCL over NVLink on B200, gloo on CPU for the
host-logic tests) carries the collectives; every data step between them is a libwsort kernel:

    rank r:  load_text(shard_r, global_base=cut_r) -> tokenize (K1 ingest, K2) -> histogram
             all_reduce(histogram)                                   -> global bucket offsets
             split:  pack_long (K3c: words >= 6 letters)  + all_reduce(dense count table, in place)
             legacy: pack (K3: every word)
             sample (K6a)               ->  all_gather(samples)      -> select_splitters (host, same on all ranks)
             partition (K6b)            ->  all_to_all(counts), all_to_all_v(keys)
             load_keys (K6c regroup) [-> dense_range] -> sort
             all_gather(local sizes)                                 -> word_base, byte_base

Split mode (every word <= 66 letters, decided from the global histogram so all ranks agree): the
words of <= 5 letters (about two thirds of the tokens) never travel; their dense count tables
 are summed by one all-reduce and every rank emits an equal share of the
global dense words straight from the summed table. Only the staged keys of the longer words are
exchanged. The global output is the ranks' dense slices in rank order, then their key slices in
rank order (RankResult.slices gives each slice's place). Legacy mode: one slice per rank, and the
concatenation of the ranks' outputs in rank order is the one-GPU output.
The global order is (length, key, source rank) in both; the assembled output is byte-identical to
the one-GPU output (tests/test_gpu_dist.py, tests/test_dist_cpu.py). This replaces the paper's MPI
master/slave scatter-gather by a symmetric exchange.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def kw_of(L):
    return (np.asarray(L) + 5) // 6


KW = kw_of(np.arange(256)).astype(np.uint64)
DENSE_MAX_LEN = 5        # words of <= 5 letters are counted in dense tables (K1 ingest)
MAX_STAGED_LEN = 66      # words of <= 66 letters are staged as keys by K1 (split mode needs all of them)


def split_mode(ghist: np.ndarray) -> bool:
    nz = np.nonzero(np.asarray(ghist)[1:])[0]
    return nz.size == 0 or int(nz[-1]) + 1 <= MAX_STAGED_LEN


def dense_words(ghist) -> int:
    return int(np.asarray(ghist, np.uint64)[1: DENSE_MAX_LEN + 1].sum())


def dense_range(ghist, rank: int, nparts: int):
    """Rank r emits the global dense words [r*Wd/P, (r+1)*Wd/P)."""
    wd = dense_words(ghist)
    return (rank * wd) // nparts, ((rank + 1) * wd) // nparts


def dense_byte_pos(ghist, w: int) -> int:
    """Byte offset of global dense word w in the output ("word\n" per word, lengths ascending)."""
    g = b = 0
    for L in range(1, DENSE_MAX_LEN + 1):
        n = int(ghist[L])
        if w <= g + n:
            return b + (w - g) * (L + 1)
        g += n
        b += n * (L + 1)
    return b


def _is_letter(c: int) -> bool:
    return ((c | 0x20) - 0x61) & 0xFF < 26


def shard_cuts(text, nparts: int) -> list:
    """Reading A13: nominal cut g*N/P moved forward while text[cut-1] and text[cut] are both letters."""
    n = len(text)
    cuts = [0]
    for g in range(1, nparts):
        c = max(cuts[-1], (g * n) // nparts)
        while 0 < c < n and _is_letter(int(text[c - 1])) and _is_letter(int(text[c])):
            c += 1
        cuts.append(c)
    cuts.append(n)
    return cuts


# ---------------------------------------------------------------------------------------- comms
class TorchComm:
    """The four collectives over torch.distributed (NCCL for cuda tensors, gloo for cpu tensors)."""

    def __init__(self, device: str):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.device = torch, dist, device
        self.rank, self.size = dist.get_rank(), dist.get_world_size()
        # gloo carries cpu tensors only: stage device data through host memory (host-logic tests)
        self.wire = "cpu" if dist.get_backend() == "gloo" else device

    def all_reduce_u64(self, x: np.ndarray) -> np.ndarray:
        t = self.torch.from_numpy(x.astype(np.int64)).to(self.wire)
        self.dist.all_reduce(t)
        return t.cpu().numpy().astype(np.uint64)

    def all_gather_rows(self, x):
        """x: tensor [n, w] -> numpy [size*n, w]."""
        x = x.contiguous().to(self.wire)
        out = self.torch.empty((self.size * x.shape[0], x.shape[1]), dtype=x.dtype, device=x.device)
        self.dist.all_gather_into_tensor(out, x)
        return out.cpu().numpy()

    def all_to_all_counts(self, counts: np.ndarray) -> np.ndarray:
        """counts[dest, L] (this rank's) -> recv[src, L] (what every src sends to this rank)."""
        t = self.torch.from_numpy(counts.astype(np.int64)).to(self.wire)
        out = self.torch.empty_like(t)
        self.dist.all_to_all_single(out, t)
        return out.cpu().numpy().astype(np.uint64)

    def all_to_all_v(self, send, send_words, recv_words):
        dev = send.device
        src = send[: int(sum(send_words))].to(self.wire)
        out = self.torch.empty(int(sum(recv_words)), dtype=send.dtype, device=self.wire)
        self.dist.all_to_all_single(out, src, [int(x) for x in recv_words], [int(x) for x in send_words])
        return out.to(dev)

    def all_reduce_(self, t):
        """In-place sum of a tensor over the ranks (the dense count tables)."""
        if str(t.device) == str(self.wire) or (self.wire != "cpu" and t.is_cuda):
            self.dist.all_reduce(t)
        else:
            w = t.to(self.wire)
            self.dist.all_reduce(w)
            t.copy_(w)

    def barrier(self):
        self.dist.barrier()


# ---------------------------------------------------------------------------------------- stages
@dataclass
class RankResult:
    n_words: int
    words_len: int
    word_base: int          # of the first slice
    byte_base: int
    slices: list = None     # [(local byte offset, bytes, global byte base, words, global word base)]


def assemble(outputs) -> bytes:
    """The global output from every rank's (words, RankResult) (tests / tools)."""
    total = sum(r.words_len for _, r in outputs)
    buf = bytearray(total)
    for words, r in outputs:
        for off, nb, gb, _, _ in r.slices:
            buf[gb: gb + nb] = bytes(words[off: off + nb])
    return bytes(buf)


class DistSorter:
    """The per-rank stages between collectives (a small state machine over one WSort context)."""

    def __init__(self, ws, rank: int, nparts: int, nsamples: int = 1024, mode: str = "auto"):
        import torch

        if mode not in ("auto", "split", "legacy"):
            raise ValueError(f"mode {mode!r}")
        self.mode = mode

        self.torch = torch
        self.ws, self.rank, self.nparts, self.nsamples = ws, rank, nparts, nsamples
        self.device = ws.torch_device

    def stage_tokenize(self, shard, global_base: int) -> np.ndarray:
        self.ws.load_text(shard, global_base)
        self.ws.tokenize()
        return self.ws.histogram()

    def stage_sample(self, ghist: np.ndarray):
        """Pack (split mode: the long words only, and expose the dense table) and sample the keys."""
        self.ghist = ghist
        self.split = self.mode != "legacy" and split_mode(ghist)
        if self.mode == "split" and not self.split:
            raise ValueError("split mode needs every word <= %d letters" % MAX_STAGED_LEN)
        nz = np.nonzero(ghist[1:])[0]
        lmax = int(nz[-1]) + 1 if nz.size else 1
        self.rec_words = 2 + int(kw_of(lmax))
        self.dense_table = None
        if self.split:
            self.dense_table = self.ws.pack_long()
        else:
            self.ws.pack()
        rec = self.torch.zeros((self.nsamples, self.rec_words), dtype=self.torch.int32, device=self.device)
        self._torch_before_ws()
        self.ws.sample(self.nsamples, self.rank, self.rec_words, rec)
        self.ws.sync()   # the collectives (torch's stream) read rec and the dense table
        return rec

    def _torch_before_ws(self):
        """Order the library's stream after torch's current stream (buffers torch wrote or received)."""
        if self.torch.cuda.is_available():
            self.torch.cuda.current_stream(self.device).synchronize()

    def stage_partition(self, all_samples: np.ndarray):
        from .api import select_splitters

        spl = select_splitters(all_samples.view(np.uint32), self.nparts)
        local_words = int((self.ws.histogram() * KW).sum())
        send = self.torch.empty(max(local_words, 1), dtype=self.torch.int32, device=self.device)
        self._torch_before_ws()
        counts, send_words = self.ws.partition(spl, self.nparts, self.rec_words, self.rank, send)
        self.ws.sync()   # all_to_all (torch's stream) reads send
        return counts, send, send_words

    @staticmethod
    def recv_words(recv_counts: np.ndarray) -> np.ndarray:
        return (recv_counts.astype(np.uint64) * KW[None, :]).sum(axis=1)

    def stage_sort(self, recv, recv_counts: np.ndarray, algo: str = "auto"):
        """Regroup the received keys and sort; returns this rank's (key words, key bytes)."""
        self._torch_before_ws()   # recv (all_to_all) and the summed dense table (all_reduce)
        self.ws.load_keys(recv, recv_counts)
        self.dlo = self.dhi = 0
        if self.split:
            self.dlo, self.dhi = dense_range(self.ghist, self.rank, self.nparts)
            self.ws.dense_range(self.ghist, self.dlo, self.dhi)
        self.ws.sort(algo)
        s = self.ws.sizes()
        self.dbytes = dense_byte_pos(self.ghist, self.dhi) - dense_byte_pos(self.ghist, self.dlo)
        return np.array([s.n_words - (self.dhi - self.dlo), s.words_len - self.dbytes], np.uint64)

    def stage_finish(self, all_sizes: np.ndarray) -> RankResult:
        """Global places of this rank's slices from every rank's key-slice sizes."""
        kw_words, kw_bytes = int(all_sizes[self.rank, 0]), int(all_sizes[self.rank, 1])
        wb = int(all_sizes[: self.rank, 0].sum())
        bb = int(all_sizes[: self.rank, 1].sum())
        if not self.split:
            self.ws.set_global(self.ghist, wb, bb)
            return RankResult(kw_words, kw_bytes, wb, bb, [(0, kw_bytes, bb, kw_words, wb)])
        wd = dense_words(self.ghist)
        bd = dense_byte_pos(self.ghist, wd)
        dwb, dbb = self.dlo, dense_byte_pos(self.ghist, self.dlo)
        self.ws.set_global(self.ghist, dwb, dbb)
        slices = [(0, self.dbytes, dbb, self.dhi - self.dlo, dwb), (self.dbytes, kw_bytes, bd + bb, kw_words, wd + wb)]
        return RankResult(kw_words + self.dhi - self.dlo, kw_bytes + self.dbytes, dwb, dbb, slices)


def sort_distributed(ws, shard, global_base: int, comm, algo: str = "auto", nsamples: int = 1024,
                     mode: str = "auto") -> RankResult:
    """One distributed sort step on this rank (all ranks must call it). mode: "auto" (split when every
    word has <= 66 letters), "split" or "legacy" (every word exchanged; `algo` picks the local sort)."""
    ds = DistSorter(ws, comm.rank, comm.size, nsamples, mode)
    hist = ds.stage_tokenize(shard, global_base)
    ghist = comm.all_reduce_u64(hist)
    rec = ds.stage_sample(ghist)
    if ds.split:
        comm.all_reduce_(ds.dense_table)
    all_samples = comm.all_gather_rows(rec)
    counts, send, send_words = ds.stage_partition(all_samples)
    recv_counts = comm.all_to_all_counts(counts)
    recv = comm.all_to_all_v(send, send_words, ds.recv_words(recv_counts))
    sizes = ds.stage_sort(recv, recv_counts, algo)
    all_sizes = comm.all_gather_rows(ds.torch.from_numpy(sizes.astype(np.int64)).view(1, 2).to(comm.device))
    return ds.stage_finish(all_sizes.astype(np.uint64))


def sort_emulated(make_ws, text: np.ndarray, nparts: int, algo: str = "auto", nsamples: int = 1024,
                  mode: str = "auto"):
    """Run the P-rank pipeline for P virtual ranks in one process (one GPU), performing the
    collectives by host-side concatenation. No kernel waits on another: stages run in lockstep.
    Returns (list of (ws, RankResult), cuts)."""
    import torch

    cuts = shard_cuts(text, nparts)
    sorters = [DistSorter(make_ws(), r, nparts, nsamples, mode) for r in range(nparts)]
    hists = [s.stage_tokenize(np.ascontiguousarray(text[cuts[r]: cuts[r + 1]]), cuts[r]) for r, s in enumerate(sorters)]
    ghist = np.sum(hists, axis=0).astype(np.uint64)
    recs = [s.stage_sample(ghist) for s in sorters]
    if sorters and sorters[0].split:   # the all-reduce of the dense tables
        total = torch.stack([s.dense_table for s in sorters]).sum(dim=0, dtype=torch.int32)
        for s in sorters:
            s.dense_table.copy_(total)
    all_samples = torch.cat(recs).cpu().numpy()
    parts = [s.stage_partition(all_samples) for s in sorters]
    sizes = []
    for r, s in enumerate(sorters):
        recv_counts = np.stack([parts[src][0][r] for src in range(nparts)]).astype(np.uint64)
        pieces = []
        for src in range(nparts):
            counts_src, send_src, sw_src = parts[src]
            start = int(sw_src[:r].sum())
            pieces.append(send_src[start: start + int(sw_src[r])])
        recv = torch.cat(pieces) if pieces else torch.empty(0, dtype=torch.int32, device=s.device)
        sizes.append(s.stage_sort(recv, recv_counts, algo))
    all_sizes = np.stack(sizes).astype(np.uint64)
    return [(s.ws, s.stage_finish(all_sizes)) for s in sorters], cuts


# ---------------------------------------------------------------------------------------- C-owned comm
def sort_group(text: np.ndarray, nparts: int, device: int = 0, make_ws=None):
    """P ranks as threads of this process (include/wsort.h wsort_group): each rank's context attaches to one
    in-process group, loads its byte-range shard (reading A13) and runs the collective wsort_tokenize /
    wsort_sort; the exchange (splitters, count matrix, records stored into the owners' windows, dense
    all-reduce) happens inside libwsort. Returns ([(words bytes, slices, global offsets, status)], cuts)."""
    import threading

    from .api import Group, WSort, WSortError

    cuts = shard_cuts(text, nparts)
    group = Group(nparts)
    ctxs = [make_ws() if make_ws else WSort(device) for _ in range(nparts)]
    out = [None] * nparts

    def run(r):
        ws = ctxs[r]
        try:
            ws.attach_group(group, r)
            ws.load_text(np.ascontiguousarray(text[cuts[r]: cuts[r + 1]]), cuts[r])
            ws.tokenize()
            ws.sort("auto")
            words, off = ws.fetch()
            out[r] = (words.tobytes(), ws.slices(), off, 0)
        except WSortError as e:
            out[r] = (None, None, None, e.status)

    threads = [threading.Thread(target=run, args=(r,)) for r in range(nparts)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for ws in ctxs:
        ws.close()
    group.close()
    return out, cuts


def assemble_slices(outs) -> bytes:
    """The global output from every rank's (words, slices) (tests / tools)."""
    pieces = []
    for words, slices, _, _ in outs:
        for lo, nb, _, gb, _ in slices:
            pieces.append((gb, words[lo: lo + nb]))
    pieces.sort(key=lambda p: p[0])
    return b"".join(p for _, p in pieces)
