"""bench.py — wsort throughput on B200 (BASELINE.json metric: "words sorted/sec and input GB/s vs
HBM roofline at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--algo auto] [--impl wsort|reference]

A step is one pass of the whole hot path (wsort_tokenize + wsort_sort: K1 tokenize, K2 offsets,
K3 pack+scatter, K4 sort, K5 emit) over the config's synthetic text, device-resident when the timed
region starts. One JSON line on rank 0. Default workload: config 4 (1 GiB, seed 4; the config the
metric is quoted at 1/2/4/8 GPUs, and the largest single-GPU config). Inputs (1 GiB text, ~1 GB of
keys) are larger than the 126 MB L2, so no extra L2 flush is done between steps.

--impl reference times the CPU oracle (oracle/, the paper's sequential merge sort per length bucket)
as it stands on this host, on a bounded prefix of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "words sorted/sec (input GB/s and HBM roofline alongside)"
UNIT = "words/s"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)   # >= 10: the paper's 10 trials
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--algo", default="auto")
    ap.add_argument("--ingest", default="auto", choices=["auto", "stage", "count"],
                    help="how K1 treats the words of >= 6 letters (wsort_set_ingest; experiments)")
    ap.add_argument("--impl", default="wsort", choices=["wsort", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--cpu-sample-mb", type=int, default=96)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-inflight", dest="no_inflight", action="store_true", help="skip the two-texts-in-flight line")
    ap.add_argument("--e2e-streamed", dest="e2e_streamed", action="store_true",
                    help="e2e: wsort_ingest_host (H2D streamed under K1) instead of load_text two steps ahead "
                         "(measured slower in the 3-context pipeline: the ingest call returns only after K2)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the N>1 path with several ranks on one GPU (tests)")
    return ap.parse_args()


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def trials_summary(trial_ms):
    """The paper's protocol: each configuration "tested 10 times to get the average" (
    SPEC.md:284-293): every timed step is one trial; mean (the paper's statistic), median and minimum."""
    return {"n": len(trial_ms), "mean_ms": statistics.mean(trial_ms), "median_ms": statistics.median(trial_ms),
            "min_ms": min(trial_ms), "max_ms": max(trial_ms),
            "protocol": "per-step CUDA events on the launching stream; PAPER.md:31 10-trial average"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str):
    """Per-launch DRAM bytes of `kernel` from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    v = d.get(kernel)
    return None if v is None else float(v.get("dram_bytes_per_launch"))


def cpu_baseline(text, sample_mb: int):
    """The oracle as it stands (single thread, merge sort per bucket) on a bounded prefix."""
    import numpy as np

    import oracle

    n = min(len(text), sample_mb << 20)
    # cut at a separator so that the sample holds whole words of the workload
    while 0 < n < len(text) and (int(text[n - 1]) | 0x20) - 97 in range(26) and (int(text[n]) | 0x20) - 97 in range(26):
        n -= 1
    sample = np.ascontiguousarray(text[:n])
    t0 = time.perf_counter()
    out = oracle.sort(sample, oracle.MERGE)
    dt = time.perf_counter() - t0
    return {"value": out.n_words / dt, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"first {n} bytes ({n / 2**20:.0f} MiB, {out.n_words} words) of the workload; "
                      f"oracle_sort(MERGE): tokenize+bucket+merge sort+emit, {dt:.2f} s",
            "seconds": dt, "input_gbs": n / dt / 1e9}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_baseline_all_cores(text, sample_mb: int):
    """The oracle's paper-mpi shape (per length bucket, p chunks sorted on p threads, then
    the master's k-way merge) on the host's cores, on a bounded prefix of the workload."""
    import numpy as np

    import oracle

    ncpu = os.cpu_count() or 1
    p = max(1, min(ncpu, 32))   # (the k-way merge scans all p runs per word: more threads stop paying)
    n = min(len(text), sample_mb << 20)
    while 0 < n < len(text) and (int(text[n - 1]) | 0x20) - 97 in range(26) and (int(text[n]) | 0x20) - 97 in range(26):
        n -= 1
    sample = np.ascontiguousarray(text[:n])
    t0 = time.perf_counter()
    out = oracle.sort_paper_mpi(sample, p, oracle.MERGE)
    dt = time.perf_counter() - t0
    return {"value": out.n_words / dt, "unit": UNIT, "cores": p, "host_cpus": ncpu, "cpu_model": cpu_model(),
            "kind": "oracle paper-mpi (merge chunks + k-way merge)",
            "sample": f"first {n} bytes ({n / 2**20:.0f} MiB, {out.n_words} words) of the workload, {p} threads, "
                      f"{dt:.2f} s", "seconds": dt, "input_gbs": n / dt / 1e9}


def run_reference(args, rank, world):
    import numpy as np

    import build_native
    import gen

    if rank != 0:
        return
    build_native.build_gen()
    build_native.build_oracle()
    import oracle

    cfg = gen.CONFIGS[args.config]
    sample_mb = max(1, min(args.cpu_sample_mb, 32))
    n = min(cfg.n, sample_mb << 20)
    text, _ = gen.generate(args.config, n=n)
    for _ in range(args.warmup):
        oracle.sort(text, oracle.MERGE)
    times = []
    words = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out = oracle.sort(text, oracle.MERGE)
        times.append(time.perf_counter() - t0)
        words = out.n_words
    ms = 1000 * sum(times) / len(times)
    value = words / (ms / 1000)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": cfg.name, "n_bytes": cfg.n, "seed": cfg.seed, "sample_bytes": n,
                   "words_per_step": words},
        "input_gbs": n / (ms / 1000) / 1e9,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"first {n} bytes of {cfg.name} per step (oracle merge sort, 1 thread)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def run_wsort(args, rank, world, local_rank):
    import numpy as np
    import torch

    import build_native
    import gen

    build_native.build_gen()
    build_native.build_wsort()
    from paper_1411_5283_b200 import WSort

    torch.cuda.set_device(local_rank)
    dev = local_rank
    stream = torch.cuda.current_stream(dev)
    cfg = gen.CONFIGS[args.config]
    if world > 1:
        return run_wsort_dist(args, rank, world, local_rank)

    # host text in pinned memory (the e2e leg copies it every step)
    host = torch.empty(cfg.n, dtype=torch.uint8, pin_memory=True)
    text, _ = gen.generate(args.config, out=host.numpy())
    ws = WSort(dev, stream=stream.cuda_stream)
    if args.ingest != "auto":
        ws.set_ingest(args.ingest)
    ws.load_text(host)
    n_words = ws.tokenize()
    ws.sort(args.algo)
    sizes = ws.sizes()
    words_len = int(sizes.words_len)

    for _ in range(args.warmup):
        ws.tokenize()
        ws.sort(args.algo)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()

    ws.reset_kernel_stats()
    ws.set_profiling(True)
    l0 = ws.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    # inputs smaller than the L2 (configs 1-3): every step starts with the L2 flushed by writing 512 MiB
    # (outside the step's events); the value is then words / mean step time
    flush = cfg.n < (512 << 20)
    fbuf = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{dev}") if flush else None
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    with ClockSampler(dev) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            if flush:
                fbuf.fill_(i & 255)
            evs[2 * i].record(stream)
            ws.tokenize()
            ws.sort(args.algo)
            evs[2 * i + 1].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    trial_ms = [evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(args.steps)]
    ms = sum(trial_ms) / args.steps if flush else ev0.elapsed_time(ev1) / args.steps
    launches = ws.launch_count() - l0
    stats = ws.kernel_stats()
    ws.set_profiling(False)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())

    total_words = n_words * world
    value = total_words / (ms / 1000)
    input_gbs = cfg.n * world / (ms / 1000) / 1e9
    peak, peak_src = measured_peaks()

    # dominant kernel and its roofline
    dom = max(stats.items(), key=lambda kv: kv[1]["ms"])
    dname, d = dom
    avg_ms = d["ms"] / d["launches"]
    bytes_per_launch = d["bytes"] / d["launches"]
    achieved = bytes_per_launch / (avg_ms / 1000) / 1e9
    pipeline_bytes = sum(v["bytes"] for v in stats.values()) / args.steps
    # the per-kernel table from a separate, serialised pass (wsort_set_profiling(2): every kernel on the
    # context's stream, so each kernel's events time it alone and the shares add up to the serialised step;
    # the timed region above overlaps the dense buckets / split jobs on side streams)
    nser = max(1, min(args.steps, 5))
    ws.reset_kernel_stats()
    ws.set_profiling(2)
    for _ in range(nser):
        ws.tokenize()
        ws.sort(args.algo)
    sstats = ws.kernel_stats()
    ws.set_profiling(False)
    ser_total = sum(x["ms"] for x in sstats.values())
    kernels = {k: {"launches_per_step": v["launches"] / nser, "ms_per_step": v["ms"] / nser, "share": v["ms"] / ser_total,
                   "gbs": (v["bytes"] / (v["ms"] / 1000) / 1e9) if v["ms"] > 0 else None}
               for k, v in sorted(sstats.items(), key=lambda kv: -kv[1]["ms"])}
    kernels["_serialised_step_ms"] = ser_total / nser
    alg_min = cfg.n + words_len   # read the text once + write the output once

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": cfg.name, "n_bytes": cfg.n, "seed": cfg.seed, "words": n_words,
                   "output_bytes": words_len, "algo": args.algo,
                   "l2": ("L2 flushed before every step (512 MiB written outside the step's events); value = words / "
                          "mean step time" if flush else
                          "inputs larger than L2 (1 GiB text + ~1 GB keys per step); no extra flush"),
                   "latency_bound": cfg.n < (8 << 20)},
        "input_gbs": input_gbs,
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(dname), "peak_source": peak_src,
                     "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms},
        "pipeline": {"modelled_bytes_per_step": pipeline_bytes,
                     "modelled_gbs": pipeline_bytes / (ms / 1000) / 1e9,
                     "modelled_frac": pipeline_bytes / (ms / 1000) / 1e9 / peak,
                     "alg_min_bytes_per_step": alg_min,
                     "alg_min_frac": alg_min / (ms / 1000) / 1e9 / peak},
        "kernels": kernels,
        "trials": trials_summary(trial_ms),
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }

    if not args.no_e2e and rank == 0:
        line["e2e"] = e2e_pipelined(args, ws, host, stream, dev, n_words, words_len, sizes)
    if not flush and rank == 0 and not getattr(args, "no_inflight", False):
        line["two_in_flight"] = two_in_flight(args, host, dev, n_words)
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline(text, args.cpu_sample_mb)
        line["cpu_baseline_all_cores"] = cpu_baseline_all_cores(text, 128)
    ws.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def two_in_flight(args, host, dev, n_words):
    """Device-resident throughput with two texts in flight: two contexts on two streams, each driven by
    its own host thread (ctypes releases the GIL inside libwsort), so one text's K1 overlaps the other's
    MSD / finish. Informative next to `value` (one text at a time); same text, same step, CUDA events
    spanning both streams."""
    import threading

    import torch

    from paper_1411_5283_b200 import WSort

    K = max(2, args.steps - args.steps % 2)
    d_text = host.to(f"cuda:{dev}")
    streams = [torch.cuda.Stream(dev) for _ in range(2)]
    ctxs = [WSort(dev, stream=s.cuda_stream) for s in streams]
    for c in ctxs:
        c.load_text(d_text)
        for _ in range(max(1, args.warmup)):
            c.tokenize()
            c.sort(args.algo)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    streams[1].wait_event(e0)

    errors = []

    def work(c):
        try:
            for _ in range(K // 2):
                c.tokenize()
                c.sort(args.algo)
        except Exception as e:   # re-raised below: a failed thread must not pass for a fast one
            errors.append(e)

    ths = [threading.Thread(target=work, args=(c,)) for c in ctxs]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errors:
        raise errors[0]
    ev = torch.cuda.Event()
    ev.record(streams[1])
    streams[0].wait_event(ev)
    e1.record(streams[0])
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / K
    for c in ctxs:
        c.close()
    return {"value": n_words / (ms / 1000), "unit": UNIT, "ms_per_text": ms, "texts": K,
            "how": "2 contexts x 2 streams x 2 host threads: tokenize + sort of one text overlaps the other's"}


def e2e_pipelined(args, ws, host, stream, dev, n_words, words_len, sizes):
    """End to end through the public API, every step copying its text in (pinned host -> device) and its
    sorted words out (device -> pinned host): load_text -> tokenize -> sort -> fetch_async. Three contexts
    on three streams take the steps round-robin and each text's load_text is issued two steps ahead, so
    the host->device copies run back to back while earlier steps sort and copy their words out (PCIe is
    full duplex). Timed with CUDA events spanning all streams."""
    import torch

    from paper_1411_5283_b200 import WSort

    D = 3
    streams = [torch.cuda.Stream(dev) for _ in range(D)]
    ctx = [WSort(dev, stream=s.cuda_stream) for s in streams]
    outs = [torch.empty(words_len + 64, dtype=torch.uint8, pin_memory=True).numpy() for _ in range(D)]
    for c, o in zip(ctx, outs):   # warm every context (allocations)
        c.load_text(host)
        c.tokenize()
        c.sort(args.algo)
        c.fetch_async(o)
        c.sync()
    K = max(D, args.e2e_steps)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(streams[0])
    for s in streams[1:]:
        s.wait_event(e0)
    streamed = getattr(args, "e2e_streamed", False)
    if not streamed:
        for j in range(min(D - 1, K)):
            ctx[j].load_text(host)
    for i in range(K):
        cur = ctx[i % D]
        if streamed:   # wsort_ingest_host: this text's H2D copy in stages under K1, while earlier texts sort / copy out
            cur.ingest_host(host)
        else:
            cur.tokenize()
            if i + D - 1 < K:
                ctx[(i + D - 1) % D].load_text(host)   # two steps ahead
        cur.sort(args.algo)
        cur.fetch_async(outs[i % D])
    for s in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(s)
        streams[0].wait_event(ev)
    e1.record(streams[0])
    torch.cuda.synchronize(dev)
    ems = e0.elapsed_time(e1) / K
    for c in ctx:
        c.close()
    return {"value": n_words / (ems / 1000), "unit": UNIT, "h2d_bytes_per_step": int(host.numel()),
            "d2h_bytes_per_step": words_len + 8 * (sizes.max_len + 2), "ms_per_step": ems, "steps": K,
            "path": ("wsort_ingest_host(pinned host: H2D streamed in 8 stages under K1) + wsort_sort + "
                     "wsort_fetch_async(pinned host); 3 contexts round-robin: a text's copy in overlaps its K1 and the "
                     "earlier texts' sorts and copies out" if streamed else
                     "wsort_load_text(pinned host) + wsort_tokenize + wsort_sort + wsort_fetch_async(pinned host); "
                     "3 contexts round-robin, texts loaded 2 steps ahead: copies in, copies out and sorts overlap")}


def run_wsort_dist(args, rank, world, local_rank):
    """N > 1: the config text sharded by byte range over the ranks (strong scaling: the total text is fixed).
    libwsort owns the NCCL communicator (wsort_attach_comm; the unique id is broadcast with torch.distributed):
    wsort_tokenize / wsort_sort are collective, the exchange (dense all-reduce, count-weighted splitters,
    (word, count) records stored into the owners' windows over NVLink) runs inside the library."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import gen
    from paper_1411_5283_b200 import WSort
    from paper_1411_5283_b200.api import get_unique_id
    from paper_1411_5283_b200.dist import shard_cuts

    dev = local_rank
    stream = torch.cuda.current_stream(dev)
    cfg = gen.CONFIGS[args.config]
    text, _ = gen.generate(args.config)
    cuts = shard_cuts(text, world)
    a, b = cuts[rank], cuts[rank + 1]
    host = torch.empty(b - a, dtype=torch.uint8, pin_memory=True)
    host.numpy()[:] = text[a:b]
    shard = host.to(f"cuda:{dev}")
    del text
    obj = [get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ws = WSort(dev, stream=stream.cuda_stream)
    ws.attach_comm(rank, world, obj[0])
    ws.load_text(shard, a)
    n_words = ws.tokenize()
    ws.sort(args.algo)
    for _ in range(args.warmup):
        ws.tokenize()
        ws.sort(args.algo)
    torch.cuda.synchronize(dev)
    dist.barrier()
    ws.reset_kernel_stats()
    ws.set_profiling(True)
    l0 = ws.launch_count()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(dev) as clk:
        evs[0].record(stream)
        for i in range(args.steps):
            ws.tokenize()
            ws.sort(args.algo)
            evs[i + 1].record(stream)
        torch.cuda.synchronize(dev)
    trial_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    ms = sum(trial_ms) / args.steps
    launches = ws.launch_count() - l0
    stats = ws.kernel_stats()
    ws.set_profiling(False)
    t = torch.tensor([ms], device=f"cuda:{dev}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    sizes = ws.sizes()
    tot = torch.tensor([int(sizes.words_len)], dtype=torch.int64, device=f"cuda:{dev}")
    dist.all_reduce(tot)
    out_bytes = int(tot[0])
    peak, peak_src = measured_peaks()
    dname, d = max(stats.items(), key=lambda kv: kv[1]["ms"])
    achieved = d["bytes"] / d["launches"] / (d["ms"] / d["launches"] / 1000) / 1e9
    line = {
        "metric": METRIC, "value": n_words / (ms / 1000), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": cfg.name, "n_bytes": cfg.n, "seed": cfg.seed, "words": n_words, "output_bytes": out_bytes,
                   "algo": args.algo, "parallelism": f"byte-range shards x{world}; library-owned NCCL communicator: "
                   "dense all-reduce + (word, count) records into the owners' windows",
                   "l2": "inputs larger than L2; no extra flush"},
        "input_gbs": cfg.n / (ms / 1000) / 1e9,
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(dname), "peak_source": peak_src, "rank": rank},
        "kernels": {k: {"launches_per_step": v["launches"] / args.steps, "ms_per_step": v["ms"] / args.steps}
                    for k, v in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])},
        "trials": trials_summary(trial_ms),
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_e2e:
        out = torch.empty(int(sizes.words_len) + 64, dtype=torch.uint8, pin_memory=True).numpy()
        dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            ws.load_text(host, a)
            ws.tokenize()
            ws.sort(args.algo)
            ws.fetch(out=out)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        ems = torch.tensor([f0.elapsed_time(f1) / args.e2e_steps], device=f"cuda:{dev}")
        dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        line["e2e"] = {"value": n_words / (float(ems.item()) / 1000), "unit": UNIT, "h2d_bytes_per_step": cfg.n,
                       "d2h_bytes_per_step": out_bytes, "ms_per_step": float(ems.item()),
                       "path": "per rank: pinned host shard -> wsort_load_text -> collective tokenize + sort -> "
                               "wsort_fetch(pinned host)"}
    ws.close()
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch

        local_rank = local_rank % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group(args.dist_backend)
    try:
        run_wsort(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch

            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
