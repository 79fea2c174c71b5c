"""The C ABI library loads and exports every symbol include/wsort.h declares (no GPU needed)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import build_native

    build_native.build_wsort()
    from paper_1411_5283_b200 import _lib

    return _lib.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "wsort.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wsort_[a-z_]+)\s*\(", src)))


def test_header_declares_binding_exports():
    from paper_1411_5283_b200 import _lib

    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_1411_5283_b200", "libwsort.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (wsort_\w+)", out))
    assert set(declared_symbols()) <= exported


def test_strerror_and_create_without_gpu(lib):
    import ctypes

    assert lib.wsort_strerror(-7) == b"word longer than 255 letters"
    assert lib.wsort_strerror(0) == b"ok"
    h = ctypes.c_void_p()
    rc = lib.wsort_create(ctypes.byref(h), 0, 0)
    try:
        import torch

        gpu = torch.cuda.is_available()
    except Exception:
        gpu = False
    if not gpu:
        assert rc == -4 and not h.value       # CUDA error, no context, no fallback
    else:
        assert rc == 0
        lib.wsort_destroy(h)
    assert lib.wsort_create(None, 0, 0) == -1


def test_sm100a_code_in_library():
    so = os.path.join(ROOT, "paper_1411_5283_b200", "libwsort.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
