"""Cascade decode (NEXT-2) vs plain on forked-prompt batches: B requests forked from one
n_prompt-token prompt + n_own own tokens each, Qwen3-8B-shaped layer. Prints one line per case.
Usage: python scripts/time_cascade.py  (CASES="B:prompt:own,...")"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_09100_b200 import Cache  # noqa: E402

P = 16
st = torch.cuda.current_stream()
g = torch.Generator(device="cuda").manual_seed(5)
cases = os.environ.get("CASES", "64:1024:1024,64:4096:1024,64:16384:1024,256:4096:1024,16:16384:4096,64:16384:64")
for cs in cases.split(","):
    B, n_prompt, n_own = (int(x) for x in cs.split(":"))
    pages = n_prompt // P + B * (n_own // P + 2) + 64
    if os.environ.get("DTYPE", "bf16") == "fp8":  # token pages in the fp8 pool (NEXT-4c)
        cache = Cache(1, 32, 8, 128, P, 64, B + 1, (n_prompt + n_own) // P + 4, 0, 99, "fp8", pages)
    else:
        cache = Cache(1, 32, 8, 128, P, pages, B + 1, (n_prompt + n_own) // P + 4, 0, 99)
    src = cache.seq_create()
    kp = torch.randn((1, n_prompt, 8, 128), generator=g, device="cuda").to(torch.bfloat16)
    cache.append_kv([src], [n_prompt], kp, kp)
    seqs = [cache.seq_fork(src, n_prompt) for _ in range(B)]
    ko = torch.randn((1, B * n_own, 8, 128), generator=g, device="cuda").to(torch.bfloat16)
    cache.append_kv(seqs, [n_own] * B, ko, ko)
    ids = np.asarray(seqs, dtype=np.int32)
    q = torch.randn((B, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    res = {}
    for on in (False, True, False, True):
        cache.set_decode_cascade(on)
        for _ in range(3):
            cache.decode(0, ids, q, o)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(20):
            cache.decode(0, ids, q, o)
        e1.record(st)
        torch.cuda.synchronize()
        res.setdefault(on, []).append(e0.elapsed_time(e1) / 20 * 1e3)
        if on:
            info = cache.decode_plan_info()
    off, on = min(res[False]), min(res[True])
    print(f"{os.environ.get('DTYPE', 'bf16')} B={B} prompt={n_prompt} own={n_own}: plain {off:.1f} us, cascade {on:.1f} us (x{off / on:.2f}), "
          f"plan {info}", flush=True)
    cache.close()
