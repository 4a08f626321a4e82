"""paper_2605_09100_b200 -- B200-native hybrid paged attention (HPA).

Thin Python binding over the C ABI in include/hpa.h (libhpa.so, built in-tree
by `python paper_2605_09100_b200/build.py`). Argument marshalling only: every step of the
path runs in the library's CUDA kernels. There is no CPU fallback -- importing
the binding raises if the library is missing, and cache creation fails on a
host without an sm_100 GPU.

PAPER.md §3 "Hybrid paged attention for LLM serving".
"""
from ._lib import HPAError, kv_bytes, lib_path  # noqa: F401
from .cache import Cache, merge_partials  # noqa: F401

__all__ = ["Cache", "HPAError", "kv_bytes", "lib_path", "merge_partials"]
