"""Python-side cost of Cache.append_decode (B = 8): cProfile over 2000 calls (GPU runs behind)."""
import cProfile, os, pstats, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402
shape = qwen3_8b_shape(16)
B, N = 8, 2000
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, N + 40, 0, seed=1)
ids = np.asarray(seqs, dtype=np.int32)
kn = torch.randn((1, B, 8, 128), device="cuda").to(torch.bfloat16)
q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
for _ in range(20):
    cache.append_decode(0, ids, kn, kn, q, o)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(N):
    cache.append_decode(0, ids, kn, kn, q, o)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
