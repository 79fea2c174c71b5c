"""Experiments only: build a variant of libwsort.so with extra -D flags on some translation units.

usage: python tools/build_variant.py NAME "k_ingest.cu:-DWSORT_D12_COPIES=1 -DX=2" [...]
Writes build/var_NAME/libwsort.so (load it with WSORT_LIB=...). The other objects come from build/obj
(python build_native.py first)."""
import os
import shlex
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import build_native as bn  # noqa: E402

name = sys.argv[1]
over = {}
for spec in sys.argv[2:]:
    f, flags = spec.split(":", 1)
    over[f] = shlex.split(flags)
bn.build_wsort()
out_dir = os.path.join(ROOT, "build", "var_" + name)
os.makedirs(out_dir, exist_ok=True)
objs = []
for s in sorted(f for f in os.listdir(os.path.join(bn.PKG, "csrc")) if f.endswith(".cu")):
    if s in over:
        o = os.path.join(out_dir, s[:-3] + ".o")
        subprocess.run([bn.NVCC, *bn.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I",
                        os.path.join(ROOT, "include"), *over[s], "-c", "-o", o, os.path.join(bn.PKG, "csrc", s)], check=True)
        objs.append(o)
    else:
        objs.append(os.path.join(ROOT, "build", "obj", s[:-3] + ".o"))
subprocess.run([bn.NVCC, *bn.ARCH, "-shared", "-cudart", "static", "-ldl", "-o", os.path.join(out_dir, "libwsort.so"), *objs],
               check=True)
print(os.path.join(out_dir, "libwsort.so"))
