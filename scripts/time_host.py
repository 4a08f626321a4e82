"""Host cost of the public API calls (no device sync inside the timed loop; the GPU runs behind):
hpa_append_decode at configs[1] (B = 64) and B = 8, hpa_decode, hpa_prefill (B = 1)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

shape = qwen3_8b_shape(16)
for B in (64, 8):
    N = 200
    cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, N + 40, 0, seed=1)
    ids = np.asarray(seqs, dtype=np.int32)
    kn = torch.randn((1, B, 8, 128), device="cuda").to(torch.bfloat16)
    q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    for _ in range(10):
        cache.append_decode(0, ids, kn, kn, q, o)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        cache.append_decode(0, ids, kn, kn, q, o)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for _ in range(N):
        cache.decode(0, ids, q, o)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"B={B}: append_decode host {1e6 * (t1 - t0) / N:.1f} us/call (wall incl. GPU {1e6 * (t2 - t0) / N:.1f}); "
          f"decode host {1e6 * (t3 - t2) / N:.1f} us/call (wall {1e6 * (t4 - t2) / N:.1f})", flush=True)
    cache.close()

# the C ABI alone: arguments marshalled once, hpa_append_decode / hpa_decode called directly
import ctypes  # noqa: E402
from paper_2605_09100_b200._lib import LIB  # noqa: E402
from paper_2605_09100_b200.cache import _p32, _stream  # noqa: E402

for B in (64, 8):
    N = 200
    cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, N + 40, 0, seed=1)
    ids = np.asarray(seqs, dtype=np.int32)
    kn = torch.randn((1, B, 8, 128), device="cuda").to(torch.bfloat16)
    q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    args = (cache._h, 0, B, _p32(ids), ctypes.c_void_p(kn.data_ptr()), ctypes.c_void_p(kn.data_ptr()),
            ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(o.data_ptr()), 0.0, _stream(0, None))
    dargs = (cache._h, 0, B, _p32(ids), ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(o.data_ptr()), 0.0,
             _stream(0, None))
    for _ in range(10):
        LIB.hpa_append_decode(*args)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        LIB.hpa_append_decode(*args)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for _ in range(N):
        LIB.hpa_decode(*dargs)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"B={B} direct C ABI: append_decode host {1e6 * (t1 - t0) / N:.1f} us/call; decode {1e6 * (t3 - t2) / N:.1f} us/call",
          flush=True)
    cache.close()
