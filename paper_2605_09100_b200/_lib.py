"""ctypes declarations for libhpa.so (see include/hpa.h for the contract)."""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# HPA_LIB_PATH overrides the library (A/B experiments with variant builds)
_LIB_PATH = os.environ.get("HPA_LIB_PATH") or os.path.join(_PKG, "libhpa.so")

c_i32 = ctypes.c_int32
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_u16p = ctypes.POINTER(ctypes.c_uint16)
c_vp = ctypes.c_void_p
c_st = ctypes.c_int  # hpa_status_t


class HPAConfig(ctypes.Structure):
    _fields_ = [
        ("num_layers", c_i32), ("num_q_heads", c_i32), ("num_kv_heads", c_i32),
        ("head_dim", c_i32), ("page_size", c_i32), ("num_pages", c_i32),
        ("max_seqs", c_i32), ("max_pages_per_seq", c_i32), ("device", c_i32),
        ("placement_seed", ctypes.c_uint64),
        ("token_kv_dtype", c_i32), ("num_token_pages", c_i32),
    ]


STATUS = {
    0: "HPA_OK", 1: "HPA_ERR_INVALID_ARG", 2: "HPA_ERR_OUT_OF_PAGES", 3: "HPA_ERR_SEQ_CAPACITY",
    4: "HPA_ERR_UNKNOWN_SEQ", 5: "HPA_ERR_UNKNOWN_SET", 6: "HPA_ERR_CUDA", 7: "HPA_ERR_UNSUPPORTED",
}

# name -> (restype, argtypes); mirrors include/hpa.h one to one.
SIGNATURES = {
    "hpa_last_error": (ctypes.c_char_p, []),
    "hpa_status_string": (ctypes.c_char_p, [c_st]),
    "hpa_kv_bytes": (ctypes.c_uint64, [ctypes.c_int64] * 5),
    "hpa_cache_create": (c_st, [ctypes.POINTER(HPAConfig), ctypes.POINTER(c_vp)]),
    "hpa_cache_destroy": (c_st, [c_vp]),
    "hpa_cache_pools": (c_st, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp),
                               ctypes.POINTER(ctypes.c_uint64)]),
    "hpa_cache_stats": (c_st, [c_vp, c_i32p, c_i32p, c_i32p]),
    "hpa_cache_token_pool": (c_st, [c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_i32p]),
    "hpa_seq_create": (c_st, [c_vp, c_i32p]),
    "hpa_seq_release": (c_st, [c_vp, c_i32]),
    "hpa_append_kv": (c_st, [c_vp, c_i32, c_i32p, c_i32p, c_vp, c_vp, c_vp]),
    "hpa_latent_set_install": (c_st, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_i32p]),
    "hpa_latent_set_install_batch": (c_st, [c_vp, c_i32, c_i32p, c_i32p, c_i32p,
                                            ctypes.POINTER(c_vp), c_vp, c_i32p]),
    "hpa_latent_set_remove": (c_st, [c_vp, c_i32, c_i32]),
    "hpa_seq_compress": (c_st, [c_vp, c_i32, c_i32, c_i32, c_vp, c_i32p]),
    "hpa_seq_compress_batch": (c_st, [c_vp, c_i32, c_i32p, c_i32p, c_i32p, c_vp, c_i32p]),
    "hpa_latent_set_share": (c_st, [c_vp, c_i32, c_i32, c_i32, c_i32p]),
    "hpa_seq_fork": (c_st, [c_vp, c_i32, c_i32, c_i32p]),
    "hpa_latent_set_install_host": (c_st, [c_vp, c_i32, c_i32p, c_i32p, c_i32p, ctypes.POINTER(c_vp), c_vp,
                                           c_i32p]),
    "hpa_decode": (c_st, [c_vp, c_i32, c_i32, c_i32p, c_vp, c_vp, ctypes.c_float, c_vp]),
    "hpa_append_decode": (c_st, [c_vp, c_i32, c_i32, c_i32p, c_vp, c_vp, c_vp, c_vp, ctypes.c_float, c_vp]),
    "hpa_decode_partial": (c_st, [c_vp, c_i32, c_i32, c_i32p, c_vp, c_vp, c_vp, ctypes.c_float, c_vp]),
    "hpa_merge_partials": (c_st, [c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "hpa_prefill": (c_st, [c_vp, c_i32, c_i32, c_i32p, c_i32p, c_vp, c_vp, ctypes.c_float, c_vp]),
    "hpa_prefill_span": (c_st, [c_vp, c_i32, c_i32, c_i32p, c_i32p, c_i32p, c_vp, c_vp, ctypes.c_float, c_vp]),
    "hpa_seq_info": (c_st, [c_vp, c_i32, c_i32p, c_i32p, c_i32p]),
    "hpa_export_logical_kv": (c_st, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "hpa_export_table": (c_st, [c_vp, c_i32, c_i32p, c_i32p, c_u16p, c_i32, c_i32p]),
    "hpa_set_decode_splits": (c_st, [c_vp, c_i32]),
    "hpa_set_decode_cascade": (c_st, [c_vp, c_i32]),
    "hpa_decode_plan_info": (c_st, [c_vp, c_i32p, c_i32p, c_i32p]),
    "hpa_set_prefill_splits": (c_st, [c_vp, c_i32]),
    "hpa_set_prefill_ctas": (c_st, [c_vp, c_i32]),
    "hpa_prefill_plan_info": (c_st, [c_vp, c_i32p, c_i32p, c_i32p, c_i32p]),
    "hpa_launch_count": (c_st, [c_vp, ctypes.POINTER(ctypes.c_uint64)]),
    "hpa_debug_trace": (c_st, [c_vp, c_vp]),
}


class HPAError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


def lib_path() -> str:
    return _LIB_PATH


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python paper_2605_09100_b200/build.py` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()


def check(status: int) -> None:
    if status != 0:
        raise HPAError(status, LIB.hpa_last_error().decode())


def kv_bytes(num_layers: int, num_kv_heads: int, head_dim: int, seq_len: int, elem_bytes: int = 2) -> int:
    """KV size = 2 x L x H_kv x d_h x N x bytes."""
    return int(LIB.hpa_kv_bytes(num_layers, num_kv_heads, head_dim, seq_len, elem_bytes))
