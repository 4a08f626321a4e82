"""Runs configs[2] chunked prefill (C=2048 over 1024 latent + 16384 token rows) a few
times; used for ncu captures of the prefill kernel."""
import argparse, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache, prefill_flops
from paper_2605_09100_b200 import Cache
from workloads import qwen3_8b_shape

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--page-size", type=int, default=16)
a = ap.parse_args()
shape = qwen3_8b_shape(a.page_size)
cache, seqs, _ = build_decode_cache(torch, Cache, shape, a.batch, 8, 16384 + 2048, 0, 0, seed=777)
q = torch.randn((a.batch * 2048, 32, 128), device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(a.reps):
    e0.record(); cache.prefill(0, seqs, [2048] * a.batch, q, o); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"prefill B{a.batch} P{a.page_size}: {ms:.3f} ms, {a.batch * prefill_flops(17408, 2048, shape) / ms / 1e9:.1f} TFLOP/s")
