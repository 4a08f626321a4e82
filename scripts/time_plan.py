"""Decode planner knobs (HPA_PLAN_C0, HPA_PLAN_COMBINE env): configs[1] fused step (the bench's
region A: 50 back-to-back hpa_append_decode calls, bf16) and the fp8-token-page decode call.
Usage: HPA_PLAN_C0=1.0 python scripts/time_plan.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

shape = qwen3_8b_shape(int(os.environ.get("P", "16")))
B, K, W = 64, 50, 5
st = torch.cuda.current_stream()
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, 3 * K + W + 16, 0, seed=1234)
g = torch.Generator(device="cuda").manual_seed(4321)
kn = torch.randn((K + W, 1, B, 8, 128), generator=g, device="cuda").to(torch.bfloat16)
vn = torch.randn((K + W, 1, B, 8, 128), generator=g, device="cuda").to(torch.bfloat16)
qs = torch.randn((K + W, B, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
out = torch.empty((B, 32, 128), dtype=torch.bfloat16, device="cuda")
ids = np.asarray(seqs, dtype=np.int32)
for i in range(W):
    cache.append_decode(0, ids, kn[i], vn[i], qs[i], out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
for i in range(K):
    cache.append_decode(0, ids, kn[W + i], vn[W + i], qs[W + i], out)
e1.record(st)
torch.cuda.synchronize()
step_us = e0.elapsed_time(e1) / K * 1e3
cache.close()
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4096, 0, 0, seed=1234, token_kv_dtype="fp8")
fp8_us = bench.time_decode_calls(torch, cache, seqs, shape, 0, st, 50, 5) * 1e3
print(f"C0={os.environ.get('HPA_PLAN_C0', '-')} COMB={os.environ.get('HPA_PLAN_COMBINE', '-')}: "
      f"bf16 step {step_us:.1f} us ({B / step_us * 1e6:.0f} tok/s) | fp8 decode {fp8_us:.1f} us", flush=True)
