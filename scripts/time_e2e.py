"""Where the e2e step time goes (configs[1], B = 64, hpa_append_decode): device-only loop, the
same loop with a cross-stream event wait per step, and the bench's e2e loop (3 H2D copies + 1
D2H per step on a copy stream) vs one consolidated H2D copy per step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

shape = qwen3_8b_shape(16)
B, K = 64, 50
st = torch.cuda.current_stream()
cs = torch.cuda.Stream()
cs2 = torch.cuda.Stream()  # ahead2: D2H on its own copy stream
cache = ids = None


def fresh():
    """Every run starts from the same cache state (appends grow the sequences)."""
    global cache, ids
    if cache is not None and os.environ.get("NOFRESH"):
        return
    if cache is not None:
        cache.close()
        torch.cuda.empty_cache()
    cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4095, 20 * K + 40, 0, seed=1234)
    ids = np.asarray(seqs, dtype=np.int32)
g = torch.Generator(device="cuda").manual_seed(1)
kvq_elems = 2 * B * 8 * 128 + B * 32 * 128
host = torch.randn((K, kvq_elems), generator=g, device="cuda").to(torch.bfloat16).cpu().pin_memory()
pin_o = torch.empty((K, B, 32, 128), dtype=torch.bfloat16).pin_memory()
dbuf = [torch.empty(kvq_elems, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
douts = [torch.empty((B, 32, 128), dtype=torch.bfloat16, device="cuda") for _ in range(2)]


def views(buf):
    k = buf[:B * 8 * 128].view(1, B, 8, 128)
    v = buf[B * 8 * 128:2 * B * 8 * 128].view(1, B, 8, 128)
    q = buf[2 * B * 8 * 128:].view(B, 32, 128)
    return k, v, q


def run(mode):
    """device: no copies; wait: a cross-stream event wait per step; ahead / ahead_noD2H: the
    bench's pipelining (step i+1's inputs copied while step i runs), one consolidated H2D."""
    fresh()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    dummy = torch.cuda.Event()
    for i in range(2):
        dbuf[i].copy_(host[i])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def h2d(i):
        sl = i % 2
        with torch.cuda.stream(cs):
            if i >= 2:
                cs.wait_event(ev_done[sl])
            dbuf[sl].copy_(host[i], non_blocking=True)
            ev_in[sl].record(cs)

    e0.record(st)
    ahead = mode.startswith("ahead")
    if ahead:
        h2d(0)
    for i in range(K):
        sl = i % 2
        if ahead:
            if i + 1 < K:
                h2d(i + 1)
            st.wait_event(ev_in[sl])
        elif mode == "wait":
            dummy.record(cs)
            st.wait_event(dummy)
        elif mode == "record":
            dummy.record(st)
        k, v, q = views(dbuf[sl])
        cache.append_decode(0, ids, k, v, q, douts[sl])
        if ahead:
            ev_done[sl].record(st)
            if mode in ("ahead", "ahead2"):
                ds = cs2 if mode == "ahead2" else cs
                with torch.cuda.stream(ds):
                    ds.wait_event(ev_done[sl])
                    pin_o[i].copy_(douts[sl], non_blocking=True)
                if mode == "ahead2":  # the H2D into this slot two steps on waits for this D2H
                    ev_done[sl].record(cs2)
    st.wait_stream(cs)
    st.wait_stream(cs2)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3


for r in range(3):
    print(" | ".join(f"{m} {run(m):.1f} us" for m in ("device", "record", "wait", "ahead", "ahead2", "ahead_noD2H")), flush=True)
