"""Multi-GPU with the library-owned communicator (-m gpu): P ranks as threads of one process on one GPU
(include/wsort.h wsort_group: collectives by host barriers + device copies, no kernel waiting on another
rank's), running the product path of wsort_tokenize / wsort_sort while attached: counting ingest per shard,
all-reduced histogram and error flags, dense tables all-reduced and emitted in equal shares, distinct long
words sent with their counts to the rank owning their (length, word) range (splitters from count-weighted
samples, records stored straight into the owner's window at device-computed offsets), sorted and emitted
there. The slices must tile the output and equal the oracle's output byte for byte."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


def run(text, P):
    from paper_1411_5283_b200.dist import sort_group

    return sort_group(np.asarray(text, np.uint8), P)


def check(outs, ref):
    from paper_1411_5283_b200.dist import assemble_slices

    assert all(o[3] == 0 for o in outs), [o[3] for o in outs]
    pos = 0
    for gb, nb in sorted((s[3], s[1]) for o in outs for s in o[1]):
        assert gb == pos, "slices do not tile the output"
        pos += nb
    assert pos == len(ref.words)
    for o in outs:
        assert o[2] == ref.off   # every rank reports the global offsets
    assert assemble_slices(outs) == ref.words


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("cfg", [1, 2])
def test_group_matches_oracle(cfg, P):
    text, _ = gen.generate(cfg)
    check(run(text, P)[0], oracle.sort(text, oracle.MERGE))


def test_group_config3_prefix_8_ranks():
    text, _ = gen.generate(3, n=16 << 20)
    check(run(text, 8)[0], oracle.sort(text, oracle.MERGE))


@pytest.mark.parametrize("P", [2, 4])
def test_group_heavy_duplicates_and_long_words(P):
    parts = [b"a " * 40000, b"the " * 30000, b"zz " * 20000, b"Q" * 200 + b" ", b"y" * 70 + b" ",
             b" ".join(bytes([97 + (i * j) % 26 for j in range(13 + i % 40)]) for i in range(4000))]
    text = np.frombuffer(b" ".join(parts), np.uint8).copy()
    check(run(text, P)[0], oracle.sort(text, oracle.MERGE))


@pytest.mark.parametrize("t", [b"", b"x", b"a b", b"   !!! ", b"abcdefgh", b"abcdefgh a", b"internationalization x"])
def test_group_empty_and_tiny(t):
    text = np.frombuffer(t, np.uint8).copy()
    check(run(text, 2)[0], oracle.sort(text, oracle.MERGE))


def test_group_word_too_long_on_one_rank_fails_every_rank():
    """A run of > 255 letters inside one rank's shard: every rank returns WSORT_E_WORD_TOO_LONG (-7), nobody
    blocks in a collective (the error flag is all-reduced before any exchange)."""
    text = np.frombuffer(b"alpha beta " * 5000 + b"q" * 300 + b" gamma " * 10, np.uint8).copy()
    outs, _ = run(text, 4)
    assert [o[3] for o in outs] == [-7] * 4


def test_nccl_single_rank_attach():
    """The NCCL-backed communicator (wsort_get_unique_id + wsort_attach_comm) with one rank: the collective
    path end to end on a real NCCL communicator (one GPU per process; more ranks need more GPUs)."""
    from paper_1411_5283_b200 import WSort
    from paper_1411_5283_b200.api import get_unique_id

    text, _ = gen.generate(2)
    ref = oracle.sort(text, oracle.MERGE)
    uid = get_unique_id()
    with WSort(0) as ws:
        ws.attach_comm(0, 1, uid)
        ws.load_text(text, 0)
        assert ws.tokenize() == ref.n_words
        ws.sort("auto")
        w, off = ws.fetch()
        assert off == ref.off and w.tobytes() == ref.words
        assert ws.slices()[0][3] == 0
        ws.detach()
