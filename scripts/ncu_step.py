"""The bench's configs[1] decode step (hpa_append_decode, B = 64) for a few steps: ncu target
for the fused decode kernel (decode_persistent_kernel<128, 1, 64, 0, 0>) and the combine."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

shape = qwen3_8b_shape(16)
B, N = 64, 8
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, N + 8, 0, seed=1234)
ids = np.asarray(seqs, dtype=np.int32)
g = torch.Generator(device="cuda").manual_seed(4321)
kn = torch.randn((N, 1, B, 8, 128), generator=g, device="cuda").to(torch.bfloat16)
q = torch.randn((N, B, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
o = torch.empty((B, 32, 128), dtype=torch.bfloat16, device="cuda")
for i in range(N):
    cache.append_decode(0, ids, kn[i], kn[i], q[i], o)
torch.cuda.synchronize()
print("ok", float(o.float().abs().max()))
