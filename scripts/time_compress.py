"""Per-call host time of hpa_seq_compress (NEXT-1) and the kernels it launches."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache
from paper_2605_09100_b200 import Cache
from workloads import qwen3_8b_shape
shape = qwen3_8b_shape(16)
cache, seqs, _ = build_decode_cache(torch, Cache, shape, 64, 8, 4096 + 128, 0, 0, seed=41)
torch.cuda.synchronize()
ts = []
for s in seqs:
    t0 = time.perf_counter()
    cache.compress(s, 4096, 128)
    ts.append((time.perf_counter() - t0) * 1e6)
torch.cuda.synchronize()
print("host us per call: first 5", [round(x, 1) for x in ts[:5]], "median", sorted(ts)[len(ts) // 2])

# host cost of one configs[1] decode step (append 1 token + decode), launches are async
import numpy as np
cache.close()
cache, seqs, _ = build_decode_cache(torch, Cache, shape, 64, 8, 4095, 200, 0, seed=1)
ids = np.asarray(seqs, dtype=np.int32)
ones = np.ones(64, dtype=np.int32)
k = torch.randn((60, 1, 64, 8, 128), device="cuda").to(torch.bfloat16)
q = torch.randn((64, 32, 128), device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
for i in range(10):
    cache.append_kv(ids, ones, k[i], k[i]); cache.decode(0, ids, q, out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(10, 60):
    cache.append_kv(ids, ones, k[i], k[i]); cache.decode(0, ids, q, out)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("host us per decode step (append + decode):", round((t1 - t0) / 50 * 1e6, 1))
