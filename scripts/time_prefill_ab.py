"""configs[2] prefill timing for A/B of variant builds (HPA_LIB_PATH): B = 4 and B = 1,
median of 5 windows of 5 calls (CUDA events), TFLOP/s. Usage: python scripts/time_prefill_ab.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import build_decode_cache, prefill_flops  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

shape = qwen3_8b_shape(16)
tag = os.path.basename(os.environ.get("HPA_LIB_PATH", "libhpa.so"))
out = []
for bp in [int(x) for x in os.environ.get("BATCHES", "4,1").split(",")]:
    cache, seqs, _ = build_decode_cache(torch, Cache, shape, bp, 8, 16384 + 2048, 0, 0, seed=777)
    if os.environ.get("PF_CTAS"):  # prefill CTA mode (hpa_set_prefill_ctas): 0 = persistent
        cache.set_prefill_ctas(int(os.environ["PF_CTAS"]))
    g = torch.Generator(device="cuda:0").manual_seed(99)
    q = torch.randn((bp * 2048, 32, 128), generator=g, device="cuda:0").to(torch.bfloat16)
    o = torch.empty_like(q)
    for _ in range(3):
        cache.prefill(0, seqs, [2048] * bp, q, o)
    ws = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            cache.prefill(0, seqs, [2048] * bp, q, o)
        e1.record()
        torch.cuda.synchronize()
        ws.append(e0.elapsed_time(e1) / 5)
    ms = statistics.median(ws)
    out.append(f"B{bp} {ms:.4f} ms {bp * prefill_flops(17408, 2048, shape) / ms / 1e9:.1f} TFLOP/s")
    cache.close()
tag += f" ctas={os.environ.get('PF_CTAS', '-1')}"
print(tag, " | ".join(out), flush=True)
