"""B=64 in-cache compressions in one hpa_seq_compress_batch call (ncu target / timing)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402
shape = qwen3_8b_shape(16)
B = 64
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4096 + 128, 0, 0, seed=41)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cache.compress_batch(seqs, [4096] * B, [128] * B)
e1.record()
torch.cuda.synchronize()
print("compress batch", e0.elapsed_time(e1), "ms")
