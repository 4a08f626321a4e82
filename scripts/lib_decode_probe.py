"""configs[1] decode (P=16): our hpa_decode and flashinfer's trtllm-gen decode on the same pools,
a few calls each -- for an ncu launch list of both (grid, block, registers, shared memory, time)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from scripts.lib_compare import tables  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

import flashinfer  # noqa: E402

dev = torch.device("cuda:0")
ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
shape = qwen3_8b_shape(16)
cache, seqs, _ = build_decode_cache(torch, Cache, shape, 64, 8, 4096, 0, 0, seed=1234)
bt, lens = tables(cache, seqs, dev)
k, v = cache.pools()
q = torch.randn((64, 32, 128), device=dev).to(torch.bfloat16)
ids = np.asarray(seqs, np.int32)
out = torch.empty_like(q)
sl = torch.tensor(lens, dtype=torch.int32, device=dev)
for _ in range(3):
    cache.decode(0, ids, q, out)
    flashinfer.decode.trtllm_batch_decode_with_kv_cache(q, (k[0], v[0]), ws, bt, sl, max(lens),
                                                       bmm1_scale=1.0 / math.sqrt(128), bmm2_scale=1.0,
                                                       kv_layout="HND", backend="trtllm-gen")
torch.cuda.synchronize()
print("ok")
