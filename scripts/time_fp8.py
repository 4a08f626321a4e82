"""configs[1] decode call time: bf16 token pages vs fp8 token pages (NEXT-4c)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache, time_decode_calls
from paper_2605_09100_b200 import Cache
from workloads import qwen3_8b_shape
shape = qwen3_8b_shape(int(os.environ.get("P", "16")))
stream = torch.cuda.current_stream()
for dt in ("bf16", "fp8"):
    cache, seqs, _ = build_decode_cache(torch, Cache, shape, 64, 8, 4096, 0, 0, seed=1234, token_kv_dtype=dt)
    ms = time_decode_calls(torch, cache, seqs, shape, 0, stream, 50, 5)
    print(f"P={shape.page_size} {dt}: decode call {ms * 1e3:.1f} us")
    cache.close()
