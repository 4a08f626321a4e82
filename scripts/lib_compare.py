"""Library comparison on identical data (context for the roofline numbers, not part of
the product path): flashinfer's precompiled trtllm-gen Blackwell attention kernels run
zero-copy on OUR KV pools -- our pool layout [NP][H_kv][P][d] per layer is flashinfer's
"HND" paged layout -- with our block tables, for configs[1] (decode, B=64, Lb=5120) and
configs[2] (chunked prefill, C=2048 over 17408 prior rows, B=1 and 4).

Prints one JSON line per case: our time, the library's time, and the max |ours - lib|
(an independent cross-check of the outputs on the same inputs).

Usage (GPU box): python scripts/lib_compare.py
"""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import build_decode_cache, decode_bytes, prefill_flops  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402


def timed(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def tables(cache, seqs, dev):
    pages = [cache.export_table(s)[0] for s in seqs]
    lens = [cache.seq_info(s)[0] for s in seqs]
    mp = max(len(p) for p in pages)
    bt = np.zeros((len(seqs), mp), np.int32)
    for i, p in enumerate(pages):
        bt[i, :len(p)] = p
    return torch.from_numpy(bt).to(dev), lens


def main():
    import flashinfer
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
    scale = 1.0 / math.sqrt(128)

    # ---------------------------------------------------------------- configs[1] decode
    for P in (16, 64):
        shape = qwen3_8b_shape(P)
        cache, seqs, _ = build_decode_cache(torch, Cache, shape, 64, 8, 4096, 0, 0, seed=1234)
        bt, lens = tables(cache, seqs, dev)
        k, v = cache.pools()
        q = torch.randn((64, 32, 128), device=dev).to(torch.bfloat16)
        ids = np.asarray(seqs, np.int32)
        out = torch.empty_like(q)
        ours_ms = timed(lambda: cache.decode(0, ids, q, out))
        sl = torch.tensor(lens, dtype=torch.int32, device=dev)

        def lib():
            return flashinfer.decode.trtllm_batch_decode_with_kv_cache(
                q, (k[0], v[0]), ws, bt, sl, max(lens), bmm1_scale=scale, bmm2_scale=1.0,
                kv_layout="HND", backend="trtllm-gen")
        lib_ms = timed(lib)
        diff = (lib().float() - out.float()).abs().max().item()
        byts = decode_bytes(lens, shape)
        print(json.dumps({"case": f"configs[1] decode B=64 Lb=5120 P={P}", "ours_ms": round(ours_ms, 4),
                          "flashinfer_trtllm_gen_ms": round(lib_ms, 4),
                          "ours_gbs": round(byts / ours_ms / 1e6, 1), "lib_gbs": round(byts / lib_ms / 1e6, 1),
                          "max_abs_diff": diff}), flush=True)
        cache.close()
        torch.cuda.empty_cache()

    # ---------------------------------------------------------------- configs[2] prefill
    C, prior = 2048, 16384
    for B in (1, 4):
        shape = qwen3_8b_shape(16)
        cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, 8, prior + C, 0, 0, seed=77)
        bt, lens = tables(cache, seqs, dev)
        k, v = cache.pools()
        q = torch.randn((B * C, 32, 128), device=dev).to(torch.bfloat16)
        ids = np.asarray(seqs, np.int32)
        ours_out = [None]

        def ours():
            ours_out[0] = cache.prefill(0, ids, [C] * B, q)
        ours_ms = timed(ours, iters=10, warm=3)
        sl = torch.tensor(lens, dtype=torch.int32, device=dev)
        cq = torch.arange(0, (B + 1) * C, C, dtype=torch.int32, device=dev)
        ckv = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device=dev)

        def lib():
            return flashinfer.prefill.trtllm_batch_context_with_kv_cache(
                q, (k[0], v[0]), ws, bt, sl, C, max(lens), scale, 1.0, B, cq, ckv,
                kv_layout="HND", causal=True)
        lib_ms = timed(lib, iters=10, warm=3)
        diff = (lib().float() - ours_out[0].float()).abs().max().item()
        fl = B * prefill_flops(lens[0] - C, C, shape)
        print(json.dumps({"case": f"configs[2] prefill B={B} C=2048 prior=17408", "ours_ms": round(ours_ms, 4),
                          "flashinfer_trtllm_gen_ms": round(lib_ms, 4),
                          "ours_tflops": round(fl / ours_ms / 1e9, 1), "lib_tflops": round(fl / lib_ms / 1e9, 1),
                          "max_abs_diff": diff}), flush=True)
        cache.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
