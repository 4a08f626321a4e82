"""configs[2] prefill (B=4) over fp8 token pages, a few calls (ncu launch-list target)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

shape = qwen3_8b_shape(16)
bp, c_rows, prior = 4, 2048, 16384
tok_pages = bp * (math.ceil((prior + c_rows) / shape.page_size) + 1)
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, bp, 8, prior + c_rows, 0, 0, seed=777,
                                          token_kv_dtype="fp8", bf16_headroom_pages=tok_pages)
q = torch.randn((bp * c_rows, 32, 128), device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(4):
    e0.record()
    cache.prefill(0, seqs, [c_rows] * bp, q, o)
    e1.record()
    torch.cuda.synchronize()
    print(f"fp8 prefill B=4: {e0.elapsed_time(e1) * 1e3:.1f} us")
