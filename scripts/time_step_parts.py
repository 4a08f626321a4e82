"""Where does the configs[1] decode step's time go? Back-to-back loops (CUDA events on the
launch stream) of: decode only, append only, append + decode, decode with S = 1 forced
(no combine), and append + decode with S = 1. Usage: python scripts/time_step_parts.py"""
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
B, K = 64, 200
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, 2000, dev, seed=1234)
ids = np.asarray(seqs, dtype=np.int32)
ones = np.ones(B, dtype=np.int32)
g = torch.Generator(device="cuda").manual_seed(1)
kn = torch.randn((1, B, 8, 128), generator=g, device="cuda").to(torch.bfloat16)
q = torch.randn((B, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)


def loop(fn, n=K, reps=5):
    for _ in range(10):
        fn()
    res = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(n // reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / (n // reps) * 1e3)
    return round(float(np.median(res)), 2), [round(x, 1) for x in res]


def dec():
    cache.decode(0, ids, q, o)


def app():
    cache.append_kv(ids, ones, kn, kn)


def both():
    app()
    dec()


for splits in (0, 1, 2, 3, 4):
    cache.set_decode_splits(splits)
    print(f"S={splits}: decode only {loop(dec)} us; append+decode {loop(both)} us", flush=True)
cache.set_decode_splits(0)
print(f"append only {loop(app, n=100)} us", flush=True)

# the bench's timed loop records an event between the append and the decode call
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def both_ev():
    app()
    ev[0].record(st)
    dec()
    ev[1].record(st)


print(f"append+decode with events (bench loop) {loop(both_ev)} us", flush=True)
