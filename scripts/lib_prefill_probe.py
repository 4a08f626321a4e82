"""configs[2] prefill B=4: our hpa_prefill and flashinfer's trtllm-gen context kernel on the same
pools, a few calls each -- for an ncu launch list of both."""
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
B, C = int(os.environ.get("B", "4")), 2048
shape = qwen3_8b_shape(16)
cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, 8, 16384 + C, 0, 0, seed=77)
bt, lens = tables(cache, seqs, dev)
k, v = cache.pools()
q = torch.randn((B * C, 32, 128), device=dev).to(torch.bfloat16)
ids = np.asarray(seqs, np.int32)
sl = torch.tensor(lens, dtype=torch.int32, device=dev)
cq = torch.arange(0, (B + 1) * C, C, dtype=torch.int32, device=dev)
ckv = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device=dev)
for _ in range(2):
    cache.prefill(0, ids, [C] * B, q)
    flashinfer.prefill.trtllm_batch_context_with_kv_cache(q, (k[0], v[0]), ws, bt, sl, C, max(lens),
                                                          1.0 / math.sqrt(128), 1.0, B, cq, ckv,
                                                          kv_layout="HND", causal=True)
torch.cuda.synchronize()
print("ok")
