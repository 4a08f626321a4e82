"""One configs[1] decode call with fp8 token pages (ncu target, NEXT-4c)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402
shape = qwen3_8b_shape(16)
cache, seqs, _ = build_decode_cache(torch, Cache, shape, 64, 8, 4096, 0, 0, seed=1234, token_kv_dtype="fp8")
q = torch.randn((64, 32, 128), device="cuda").to(torch.bfloat16)
ids = np.asarray(seqs, np.int32)
for _ in range(4):
    out = cache.decode(0, ids, q)
torch.cuda.synchronize()
print("ok", float(out.float().abs().max()))
