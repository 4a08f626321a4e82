"""configs[2] prefill (C = 2048 over 1024 latent + 16384 cached token rows) at B = 1..4:
unsplit grid vs the split-KV planner vs forced split counts (CUDA events, 10 calls)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402


def main():
    dev = 0
    torch.cuda.set_device(dev)
    shape = qwen3_8b_shape(16)
    stream = torch.cuda.current_stream()
    # a mode is a split setting, suffixed "p" for the persistent kernel, "c" for forced 2-CTA
    # clusters (else one CTA per item)
    modes = os.environ.get("MODES", "1,0,2,3,4,6").split(",")
    for bp in [int(x) for x in os.environ.get("BATCHES", "1,2,3,4").split(",")]:
        c_rows, prior = int(os.environ.get("C_ROWS", "2048")), 16384
        cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, bp, 8, prior + c_rows, 0, dev, seed=777)
        g = torch.Generator(device="cuda:0").manual_seed(99)
        q = torch.randn((bp * c_rows, 32, 128), generator=g, device="cuda:0").to(torch.bfloat16)
        o = torch.empty_like(q)
        flops = bp * bench.prefill_flops(8 * 128 + prior, c_rows, shape)
        ref = None
        res = {}
        for mode in modes * int(os.environ.get("ROUNDS", "1")):
            cache.set_prefill_splits(int(mode.rstrip("pc")))
            cache.set_prefill_ctas(0 if mode.endswith("p") else -2 if mode.endswith("c") else -1)
            for _ in range(3):
                cache.prefill(0, seqs, [c_rows] * bp, q, o)
            torch.cuda.synchronize()
            if ref is None:
                ref = o.clone()
            err = (o.float() - ref.float()).abs().max().item()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            h0 = time.perf_counter()
            for _ in range(10):
                cache.prefill(0, seqs, [c_rows] * bp, q, o)
            host_us = (time.perf_counter() - h0) / 10 * 1e6
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            res.setdefault(mode, []).append(ms)
            print(f"B={bp} splits={mode:>3}: {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TFLOP/s  "
                  f"max|diff vs splits=1| {err:.4f}  host {host_us:.0f} us/call", flush=True)
        for mode, v in res.items():
            print(f"  B={bp} splits={mode:>3}: min {min(v) * 1e3:7.1f} us  median {sorted(v)[len(v) // 2] * 1e3:7.1f} us "
                  f"({flops / min(v) / 1e9:.1f} TFLOP/s at min)", flush=True)
        cache.close()


if __name__ == "__main__":
    main()
