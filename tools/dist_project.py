"""Per-rank stage times of the multi-GPU pipeline, measured on ONE GPU by running P virtual ranks one
after another (sort_emulated's stages, each bracketed by a device sync), plus the bytes each
collective would move. This is a projection tool, not a bench: the collectives are host-side here, and
the real ranks run concurrently on their own GPUs.

    python tools/dist_project.py --config 4 --ranks 1,2,4,8 [--mode split|legacy]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_1411_5283_b200 import WSort  # noqa: E402
from paper_1411_5283_b200.dist import DistSorter, shard_cuts  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


def one(text, P, mode, nsamples, ctxs):
    cuts = shard_cuts(text, P)
    shards = [torch.from_numpy(np.ascontiguousarray(text[cuts[r]: cuts[r + 1]])).cuda() for r in range(P)]
    ds = [DistSorter(ctxs[r], r, P, nsamples, mode) for r in range(P)]
    t = {k: [0.0] * P for k in ("tokenize", "pack_sample", "partition", "sort")}
    hists = []
    for r in range(P):
        h, t["tokenize"][r] = timed(lambda: ds[r].stage_tokenize(shards[r], cuts[r]))
        hists.append(h)
    ghist = np.sum(hists, axis=0).astype(np.uint64)
    recs = []
    for r in range(P):
        rec, t["pack_sample"][r] = timed(lambda: ds[r].stage_sample(ghist))
        recs.append(rec)
    if ds[0].split:
        total = torch.stack([d.dense_table for d in ds]).sum(dim=0, dtype=torch.int32)
        for d in ds:
            d.dense_table.copy_(total)
    all_samples = torch.cat(recs).cpu().numpy()
    parts = []
    for r in range(P):
        p, t["partition"][r] = timed(lambda: ds[r].stage_partition(all_samples))
        parts.append(p)
    a2a_out = [int(parts[r][2].sum() - parts[r][2][r]) * 4 for r in range(P)]
    for r in range(P):
        recv_counts = np.stack([parts[s][0][r] for s in range(P)]).astype(np.uint64)
        pieces = []
        for s in range(P):
            sw = parts[s][2]
            st = int(sw[:r].sum())
            pieces.append(parts[s][1][st: st + int(sw[r])])
        recv = torch.cat(pieces)
        _, t["sort"][r] = timed(lambda: ds[r].stage_sort(recv, recv_counts))
    tot = [sum(t[k][r] for k in t) for r in range(P)]
    dense_bytes = int(ds[0].dense_table.numel()) * 4 if ds[0].split else 0
    return {"P": P, "mode": "split" if ds[0].split else "legacy", "stage_ms_max": {k: max(v) for k, v in t.items()},
            "rank_ms_max": max(tot), "rank_ms_min": min(tot), "a2a_bytes_out_max": max(a2a_out),
            "dense_allreduce_bytes": dense_bytes}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--nsamples", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    text, _ = gen.generate(a.config)
    for P in [int(x) for x in a.ranks.split(",")]:
        ctxs = [WSort(0) for _ in range(P)]
        res = None
        for i in range(a.reps):   # the last repetition is reported (warm contexts)
            if i == a.reps - 1:
                for c in ctxs:
                    c.reset_kernel_stats()
                    c.set_profiling(True)
            res = one(text, P, a.mode, a.nsamples, ctxs)
        st = ctxs[0].kernel_stats()
        res["rank0_kernels_ms"] = {k: round(v["ms"], 4) for k, v in sorted(st.items(), key=lambda kv: -kv[1]["ms"])}
        res["rank0_launches"] = {k: v["launches"] for k, v in st.items()}
        for c in ctxs:
            c.close()
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
