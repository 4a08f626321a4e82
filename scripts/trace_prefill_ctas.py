"""Per-CTA timeline of the prefill kernel (needs a -DHPA_TRACE=1 build loaded via HPA_LIB_PATH):
entry / setup done / first S / o_full / exit (globaltimer ns) and SM of every CTA, for
configs[2] at batch B with forced split count SPLITS. Prints the per-CTA phase durations, a
least-squares fit duration = a + b * n_tiles, and the gap between a CTA's exit and the next
CTA's entry on the same SM."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from paper_2605_09100_b200._lib import LIB  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

B = int(os.environ.get("B", "4"))
C = int(os.environ.get("C", "2048"))
for splits in [int(x) for x in os.environ.get("SPLITS", "1,2").split(",")]:
    shape = qwen3_8b_shape(16)
    cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, 8, 16384 + C, 0, 0, seed=777)
    cache.set_prefill_splits(splits)
    cache.set_prefill_ctas(int(os.environ.get("PF_CTAS", "-1")))  # 0: persistent (n_tiles column = items)
    n_cta_max = B * 16 * 16 * 16
    buf = torch.zeros(4096 + 8 * n_cta_max, dtype=torch.int64, device="cuda")
    LIB.hpa_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    LIB.hpa_debug_trace(cache._h, ctypes.c_void_p(buf.data_ptr()))
    q = torch.randn((B * C, 32, 128), device="cuda").to(torch.bfloat16)
    for _ in range(3):
        buf.zero_()
        cache.prefill(0, seqs, [C] * B, q)
        torch.cuda.synchronize()
    t = buf[4096:].view(-1, 8).cpu().numpy()
    t = t[t[:, 7] == 1]
    t0 = t[:, 0].min()
    ent, setup, firsts, ofull, ex, sm, nt = (t[:, k] for k in range(7))
    dur = (ex - ent) / 1e3
    print(f"B={B} splits={splits}: {len(t)} CTAs, kernel span {(ex.max() - t0) / 1e3:.1f} us")
    print(f"  entry->setup {np.median(setup - ent) / 1e3:.2f} us, setup->first S {np.median(firsts - setup) / 1e3:.2f} us,"
          f" o_full->exit {np.median(ex - ofull) / 1e3:.2f} us (medians)")
    A = np.stack([np.ones_like(nt, dtype=float), nt.astype(float)], 1)
    coef, *_ = np.linalg.lstsq(A, dur, rcond=None)
    print(f"  fit: CTA us = {coef[0]:.2f} + {coef[1]:.3f} * n_tiles (n_tiles {nt.min()}..{nt.max()})")
    gaps = []
    for s in np.unique(sm):
        idx = np.where(sm == s)[0]
        o = idx[np.argsort(ent[idx])]
        gaps += list((ent[o[1:]] - ex[o[:-1]]) / 1e3)
    gaps = np.array(gaps)
    print(f"  SM gap exit->next entry: median {np.median(gaps):.2f} us, p90 {np.percentile(gaps, 90):.2f} us")
    first_end = np.array([ex[sm == s].max() for s in np.unique(sm)])
    print(f"  per-SM last exit: min {(first_end.min() - t0) / 1e3:.1f} max {(first_end.max() - t0) / 1e3:.1f} us")
    cache.close()
