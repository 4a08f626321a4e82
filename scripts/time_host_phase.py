"""Host time of hpa_append_decode through the C ABI at batch B (env, default 8), for the
HPA_HOST_PROF diagnostics build (per-phase averages printed at exit)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from paper_2605_09100_b200._lib import LIB  # noqa: E402
from paper_2605_09100_b200.cache import _p32, _stream  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

B, N = int(os.environ.get("B", "8")), 400
cache, seqs, _ = bench.build_decode_cache(torch, Cache, qwen3_8b_shape(16), B, 8, 4095, N + 40, 0, seed=1)
ids = np.asarray(seqs, dtype=np.int32)
kn = torch.randn((1, B, 8, 128), device="cuda").to(torch.bfloat16)
q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
args = (cache._h, 0, B, _p32(ids), ctypes.c_void_p(kn.data_ptr()), ctypes.c_void_p(kn.data_ptr()),
        ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(o.data_ptr()), 0.0, _stream(0, None))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(N):
    LIB.hpa_append_decode(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"B={B}: hpa_append_decode {1e6 * (t1 - t0) / N:.1f} us/call host", flush=True)
