"""Is the bench's configs[1] step time (append + decode, K steps) perturbed by its own
instrumentation? Same loop as bench.run_ours with: per-step CUDA events on/off, the NVML clock
sampler (0.5 ms polling) on/off, K = 20 / 200. Prints ms per step for each combination."""
import os
import sys
import time

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
B = 64
ones = np.ones(B, dtype=np.int32)
g = torch.Generator(device="cuda").manual_seed(1)
NS = 420
knew = torch.randn((NS, 1, B, 8, 128), generator=g, device="cuda").to(torch.bfloat16)
qs = torch.randn((NS, B, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
out = torch.empty((B, 32, 128), dtype=torch.bfloat16, device="cuda")
pos = [0]


def run(K, events, sampler):
    cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, K + 16, dev, seed=1234)
    ids = np.asarray(seqs, dtype=np.int32)
    for _ in range(5):
        i = pos[0] % NS
        cache.append_kv(ids, ones, knew[i], knew[i])
        cache.decode(0, ids, qs[i], out)
        pos[0] += 1
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = bench.ClockSampler(dev) if sampler else None
    torch.cuda.synchronize()
    if clk:
        clk.start()
    t0.record(st)
    for k in range(K):
        i = pos[0] % NS
        cache.append_kv(ids, ones, knew[i], knew[i])
        if events:
            evs[k][0].record(st)
        cache.decode(0, ids, qs[i], out)
        if events:
            evs[k][1].record(st)
        pos[0] += 1
    t1.record(st)
    torch.cuda.synchronize()
    if clk:
        clk.stop()
        clk.summary()
    cache.close()
    return t0.elapsed_time(t1) / K * 1e3


for rep in range(3):
    for K in (20, 200):
        for events in (False, True):
            for sampler in (False, True):
                us = run(K, events, sampler)
                print(f"rep {rep} K={K} events={events} sampler={sampler}: {us:.1f} us/step", flush=True)
