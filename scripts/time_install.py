"""configs[3] latent-set replacement alone: B=256 requests, one 128-row set each per call
(one batched install, one scatter launch); CUDA events over 20 calls."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

B = 256
shape = qwen3_8b_shape(16)
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, 40, 0, seed=555)
g = torch.Generator(device="cuda:0").manual_seed(1)
stage = torch.randn((2, B, 1, 2, 128, 8, 128), generator=g, device="cuda:0").to(torch.bfloat16)
ids = np.asarray(seqs, dtype=np.int32)
sets = [np.full(B, k, dtype=np.int32) for k in range(8)]
for i in range(5):
    cache.latent_install_packed(ids, sets[i % 8], stage[i % 2])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import time  # noqa: E402
e0.record()
h0 = time.perf_counter()
for i in range(20):
    cache.latent_install_packed(ids, sets[i % 8], stage[i % 2])
host_us = (time.perf_counter() - h0) / 20 * 1e6
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
moved = B * 128 * 8 * 128 * 2 * 2 * 2  # K and V rows, bf16, read + written
print(f"install B={B}: {ms * 1e3:.1f} us per call, {moved / (ms / 1e3) / 1e9:.0f} GB/s (read + write), "
      f"host {host_us:.1f} us per call")
