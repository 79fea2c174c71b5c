"""Multi-rank host logic on CPU (-m "not gpu"): torch.distributed gloo, world_size 2.

The per-rank kernels cannot run here, so a test double (FakeWS, numpy) stands in for the libwsort
context: it implements the same stage API with the same semantics (packed keys, regular samples,
partition by (length, key, rank) splitters, regroup, sort). What is under test is everything around
the kernels: shard cutting (reading A13), TorchComm's collectives over gloo, the real host-side
splitter selection of libwsort (wsort_select_splitters), count/offset bookkeeping, and that the
concatenation of the ranks' outputs equals the oracle's output.
"""
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_1411_5283_b200.dist import (DistSorter, KW, RankResult, TorchComm, assemble, dense_byte_pos,
                                       dense_range, kw_of, shard_cuts, sort_distributed, split_mode)

DENSE_BASE = [0, 0, 26, 702, 18278, 475254, 12356630]   # entries of the dense tables of lengths < L


def dense_index(w: bytes) -> int:
    x = 0
    for ch in w:
        x = x * 26 + (ch - 97)
    return DENSE_BASE[len(w)] + x


def dense_word(e: int) -> bytes:
    L = max(l for l in range(1, 6) if DENSE_BASE[l] <= e)
    x = e - DENSE_BASE[L]
    out = []
    for _ in range(L):
        out.append(97 + x % 26)
        x //= 26
    return bytes(reversed(out))


def pack_word(w: bytes) -> list:
    kw = int(kw_of(len(w)))
    out = []
    for q in range(kw):
        x = 0
        for j in range(6):
            i = 6 * q + j
            c = (w[i] & 31) if i < len(w) else 0
            x |= c << (25 - 5 * j)
        out.append(x)
    return out


class FakeWS:
    """numpy stand-in for WSort's multi-GPU stage API (test double; CPU tensors)."""

    torch_device = "cpu"

    def sync(self):
        pass

    def load_text(self, text, global_base=0):
        self.text = bytes(np.asarray(text, dtype=np.uint8))

    def tokenize(self):
        self.words = [m.group().lower() for m in re.finditer(rb"[A-Za-z]+", self.text)]
        return len(self.words)

    def histogram(self):
        h = np.zeros(256, np.uint64)
        for w in self.words:
            h[len(w)] += 1
        return h

    def pack(self):
        self.dense = None
        self.buckets = {}
        for w in self.words:
            self.buckets.setdefault(len(w), []).append(pack_word(w))
        self.flat = [(L, k) for L in sorted(self.buckets) for k in self.buckets[L]]

    def pack_long(self):
        """Split variant: dense table (the real indexing) for L <= 5; only longer words are packed."""
        table = np.zeros(DENSE_BASE[6], np.int32)
        for w in self.words:
            if len(w) <= 5:
                table[dense_index(w)] += 1
        self.words = [w for w in self.words if len(w) > 5]
        self.pack()
        self.dense = torch.from_numpy(table)
        return self.dense

    def dense_range(self, ghist, lo, hi):
        self.dlo, self.dhi = lo, hi

    def sample(self, n, rank, rec_words, out):
        W = len(self.flat)
        for i in range(n):
            rec = [0] * rec_words
            if W:
                L, k = self.flat[((2 * i + 1) * W) // (2 * n)]
                rec[0], rec[1] = L, rank
                rec[2: 2 + len(k)] = k
            out[i] = torch.tensor(np.array(rec, np.uint32).view(np.int32))

    def partition(self, spl, nparts, rec_words, rank, send):
        spl = [tuple(int(x) for x in r) for r in spl]

        def dest(L, k):
            d = 0
            for s in spl:
                sk = list(s[2: 2 + len(k)])
                if (s[0], sk, s[1]) < (L, k, rank):
                    d += 1
            return d

        per = [[[] for _ in range(256)] for _ in range(nparts)]
        for L, k in self.flat:
            per[dest(L, k)][L].append(k)
        counts = np.zeros((nparts, 256), np.uint64)
        words = []
        sw = np.zeros(nparts, np.uint64)
        for d in range(nparts):
            for L in range(256):
                counts[d, L] = len(per[d][L])
                for k in per[d][L]:
                    words.extend(k)
                sw[d] += len(per[d][L]) * int(kw_of(L))
        if words:
            send[: len(words)] = torch.tensor(np.array(words, np.uint32).view(np.int32))
        return counts, sw

    def load_keys(self, recv, counts):
        self.dlo = self.dhi = 0
        r = recv.numpy().view(np.uint32)
        pos = 0
        self.recv = {}
        for src in range(counts.shape[0]):
            for L in range(256):
                kw = int(kw_of(L))
                for _ in range(int(counts[src, L])):
                    self.recv.setdefault(L, []).append(tuple(int(x) for x in r[pos: pos + kw]))
                    pos += kw

    def sort(self, algo="auto"):
        self.out = b""
        if self.dense is not None and self.dhi > self.dlo:   # this rank's share of the summed dense table
            t = self.dense.numpy()
            nz = np.nonzero(t)[0]
            ends = np.cumsum(t[nz].astype(np.int64))
            for e, end in zip(nz, ends):
                a, b = max(int(end) - int(t[e]), self.dlo), min(int(end), self.dhi)
                if b > a:
                    self.out += (dense_word(int(e)) + b"\n") * (b - a)
        for L in sorted(self.recv):
            for k in sorted(self.recv[L]):
                w = bytes(((k[j // 6] >> (25 - 5 * (j % 6))) & 31) | 0x60 for j in range(L))
                self.out += w + b"\n"
        self.n = sum(len(v) for v in self.recv.values()) + (self.dhi - self.dlo)

    def sizes(self):
        class S:
            pass

        s = S()
        s.n_words, s.words_len = self.n, len(self.out)
        return s

    def set_global(self, ghist, wb, bb):
        self.ghist, self.wb, self.bb = ghist, wb, bb


def _worker(rank, world, port, text, q, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cuts = shard_cuts(text, world)
        ws = FakeWS()
        comm = TorchComm("cpu")
        res = sort_distributed(ws, text[cuts[rank]: cuts[rank + 1]], cuts[rank], comm, nsamples=64, mode=mode)
        q.put((rank, ws.out, res, [int(x) for x in ws.ghist]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["split", "legacy"])
@pytest.mark.parametrize("src", ["config1", "dups"])
def test_gloo_world2_matches_oracle(src, mode):
    if src == "config1":
        text = gen.generate(1)[0][:60_000].copy()
    else:   # heavy duplicates: splitters fall inside runs of one word
        text = np.frombuffer(b"the a the of the cat a of the " * 1500, np.uint8).copy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, text, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.sort(text, oracle.MERGE)
    assert assemble([(r[1], r[2]) for r in res]) == ref.words
    if mode == "legacy":
        assert b"".join(r[1] for r in res) == ref.words
        assert res[0][2].word_base == 0 and res[1][2].word_base == ref.words.count(b"\n") - res[1][1].count(b"\n")
        assert res[1][2].byte_base == len(res[0][1])
    else:
        assert all(len(r[2].slices) == 2 for r in res)
        assert res[0][2].slices[0][2] == 0                      # rank 0's dense slice opens the output
    hist = oracle.histogram(text)[0]
    assert res[0][3] == [int(x) for x in hist]


def test_shard_cuts_never_split_a_word():
    text = np.frombuffer(b"aaaa bbbb cccccccc d e fffffffffff " * 50, np.uint8)
    for p in (1, 2, 3, 5, 8, 13):
        cuts = shard_cuts(text, p)
        assert cuts[0] == 0 and cuts[-1] == len(text) and cuts == sorted(cuts)
        for c in cuts[1:-1]:
            assert not (chr(text[c - 1]).isalpha() and chr(text[c]).isalpha())
        # the shards' word lists concatenate to the whole text's word list
        words = []
        for a, b in zip(cuts, cuts[1:]):
            words += re.findall(rb"[A-Za-z]+", text[a:b].tobytes())
        assert words == re.findall(rb"[A-Za-z]+", text.tobytes())


def test_select_splitters_host_function():
    """libwsort's host splitter choice: records sorted by (L, key words, rank); quantiles d*n/P."""
    from paper_1411_5283_b200.api import select_splitters

    rng = np.random.default_rng(0)
    n, rw = 400, 4
    rec = np.zeros((n, rw), np.uint32)
    rec[:, 0] = rng.integers(1, 6, n)
    rec[:, 1] = rng.integers(0, 4, n)
    rec[:, 2] = rng.integers(0, 50, n)
    rec[:, 3] = rng.integers(0, 3, n)
    for P in (1, 2, 4, 8):
        spl = select_splitters(rec, P)
        assert spl.shape == (P - 1, rw)
        order = sorted(range(n), key=lambda i: (rec[i, 0], rec[i, 2], rec[i, 3], rec[i, 1], i))
        for d in range(1, P):
            assert (spl[d - 1] == rec[order[(d * n) // P]]).all()


def test_dense_split_host_arithmetic():
    """dense_range / dense_byte_pos / split_mode against a direct count on a known histogram."""
    ghist = np.zeros(256, np.uint64)
    ghist[1], ghist[2], ghist[3], ghist[5], ghist[7] = 3, 4, 5, 2, 6
    wd = 3 + 4 + 5 + 2
    layout = b"a\n" * 3 + b"ab\n" * 4 + b"abc\n" * 5 + b"abcde\n" * 2
    for w in range(wd + 1):
        assert dense_byte_pos(ghist, w) == len(b"".join(layout.split(b"\n")[i] + b"\n" for i in range(w)))
    for P in (1, 2, 3, 5, 14, 20):
        rs = [dense_range(ghist, r, P) for r in range(P)]
        assert rs[0][0] == 0 and rs[-1][1] == wd
        assert all(rs[i][1] == rs[i + 1][0] for i in range(P - 1))
        assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    assert split_mode(ghist)
    ghist[67] = 1
    assert not split_mode(ghist)
    assert split_mode(np.zeros(256, np.uint64))


def test_assemble_places_slices():
    outs = [(b"aa\nccc\n", RankResult(2, 7, 0, 0, [(0, 3, 0, 1, 0), (3, 4, 6, 1, 2)])),
            (b"bb\nddd\n", RankResult(2, 7, 1, 3, [(0, 3, 3, 1, 1), (3, 4, 10, 1, 3)]))]
    assert assemble(outs) == b"aa\nbb\nccc\nddd\n"
