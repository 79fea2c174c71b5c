"""Native builds for the repo (used by __graft_entry__.build() and tests/conftest.py).

* paper_1411_5283_b200/libwsort.so — the product: CUDA kernels + C ABI for sm_100a (nvcc).
* oracle/liboracle.so            — the CPU oracle (gcc; test infrastructure only).
* gen/libwsortgen.so             — the seeded input generator (gcc).

Everything is built in-tree so the .so files travel to the GPU box with the snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1411_5283_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target: str, sources: list) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list, cwd: str | None = None) -> None:
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def build_gen(force: bool = False) -> str:
    src = os.path.join(ROOT, "gen", "wsort_gen.c")
    out = os.path.join(ROOT, "gen", "libwsortgen.so")
    if force or _stale(out, [src]):
        _run(["gcc", "-O2", "-Wall", "-shared", "-fPIC", "-pthread", "-o", out, src, "-lm"])
    return out


def build_oracle(force: bool = False) -> str:
    src = os.path.join(ROOT, "oracle", "wsort_oracle.c")
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or _stale(out, [src]):
        _run(["gcc", "-O2", "-Wall", "-shared", "-fPIC", "-pthread", "-o", out, src])
    return out


def wsort_sources() -> list:
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cuh"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def build_wsort(force: bool = False, verbose_ptxas: bool = False) -> str:
    out = os.path.join(PKG, "libwsort.so")
    srcs = wsort_sources()
    if not (force or _stale(out, srcs)):
        return out
    cu = [s for s in srcs if s.endswith(".cu")]
    # one object per translation unit, compiled in parallel (no device symbol crosses files), then linked
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", os.path.join(ROOT, "include")]
    if verbose_ptxas:
        flags.insert(0, "-Xptxas=-v")
    headers = [s for s in srcs if not s.endswith(".cu")]
    objs, jobs = [], []
    for s in cu:
        o = os.path.join(objdir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers]):
            jobs.append([NVCC, *flags, "-c", "-o", o, s])
    if jobs:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            list(ex.map(_run, jobs))
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-ldl", "-o", out, *objs])
    return out


def build_all(force: bool = False) -> None:
    build_gen(force)
    build_oracle(force)
    build_wsort(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built")
