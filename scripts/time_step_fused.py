"""configs[1] decode step: the two-call step (hpa_append_kv + hpa_decode) vs the fused
hpa_append_decode, interleaved windows of N steps on one cache (lengths grow equally for both).
Also each with an event pair around every call (the bench's region B) to show the event cost.
Usage: python scripts/time_step_fused.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

dev = 0
torch.cuda.set_device(dev)
st = torch.cuda.current_stream(dev)
shape = qwen3_8b_shape(16)
B, N, ROUNDS = 64, 50, 5
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, 4 * N * ROUNDS + 200, dev, seed=1234)
ids = np.asarray(seqs, dtype=np.int32)
ones = np.ones(B, dtype=np.int32)
g = torch.Generator(device="cuda").manual_seed(1)
kn = torch.randn((1, B, 8, 128), generator=g, device="cuda").to(torch.bfloat16)
q = torch.randn((B, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)


def two():
    cache.append_kv(ids, ones, kn, kn)
    cache.decode(0, ids, q, o)


def fused():
    cache.append_decode(0, ids, kn, kn, q, o)


def window(fn, events):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * N)]
    torch.cuda.synchronize()
    e0.record(st)
    for i in range(N):
        if events:
            ev[2 * i].record(st)
        fn()
        if events:
            ev[2 * i + 1].record(st)
    e1.record(st)
    torch.cuda.synchronize()
    per_call = [ev[2 * i].elapsed_time(ev[2 * i + 1]) * 1e3 for i in range(N)] if events else []
    return e0.elapsed_time(e1) / N * 1e3, (float(np.mean(per_call)) if per_call else None)


for _ in range(5):
    two()
    fused()
res = {k: [] for k in ("two", "fused", "two+ev", "fused+ev", "fused call (ev)")}
for r in range(ROUNDS):
    res["two"].append(window(two, False)[0])
    res["fused"].append(window(fused, False)[0])
    t, c = window(two, True)
    res["two+ev"].append(t)
    t, c = window(fused, True)
    res["fused+ev"].append(t)
    res["fused call (ev)"].append(c)
for k, v in res.items():
    print(f"{k:16s} median {np.median(v):7.2f} us/step  windows {[round(x, 1) for x in v]}", flush=True)
