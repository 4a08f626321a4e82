"""configs[1] decode call (bf16, P = 16) at forced split counts (hpa_set_decode_splits; 0 = planner):
median of 5 windows of 20 calls. Usage: python scripts/time_decode_splits.py"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

shape = qwen3_8b_shape(int(os.environ.get("P", "16")))
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, 64, 8, 4095, 0, 0, seed=1234)
ids = np.asarray(seqs, dtype=np.int32)
q = torch.randn((64, 32, 128), device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
res = []
for S in [int(x) for x in os.environ.get("SPLITS", "0,1,2,3,4,5,6,8,10").split(",")]:
    cache.set_decode_splits(S)
    for _ in range(5):
        cache.decode(0, ids, q, out)
    ws = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            cache.decode(0, ids, q, out)
        e1.record()
        torch.cuda.synchronize()
        ws.append(e0.elapsed_time(e1) / 20 * 1e3)
    info = cache.decode_plan_info()
    res.append(f"S={S} ({info['units']} units, max {info['splits']}): {statistics.median(ws):.1f} us")
print(" | ".join(res), flush=True)
