"""wsort — B200-native (sm_100a) word sort by (length, alphabetical), the hot path of
arXiv 1411.5283 (§3 Methodology, Pre-processing).

Python binding of the C ABI in include/wsort.h (libwsort.so). Argument marshalling only:
every step of the path runs in the library's CUDA kernels; torch provides device memory and
streams. There is no CPU fallback: without libwsort.so or a CUDA device the calls raise.
"""
from .api import WSort, WSortError, sort  # noqa: F401
from . import _lib  # noqa: F401

__all__ = ["WSort", "WSortError", "sort"]
