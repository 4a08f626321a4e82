"""Per-CTA timeline of the persistent decode kernel (needs a -DHPA_TRACE=1 build loaded via
HPA_LIB_PATH): entry and last-consumer exit (globaltimer) and units per CTA for configs[1]
(B=64, Lb=5120). Prints the kernel span, the spread of CTA finish times (the tail) and units."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from paper_2605_09100_b200._lib import LIB  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

shape = qwen3_8b_shape(16)
B = int(os.environ.get("B", "64"))
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, B, 8, 4096, 64, 0, seed=1234)
buf = torch.zeros(4 * 2048, dtype=torch.int64, device="cuda")
LIB.hpa_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
LIB.hpa_debug_trace(cache._h, ctypes.c_void_p(buf.data_ptr()))
q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
o = torch.empty_like(q)
ids = np.asarray(seqs, dtype=np.int32)
for it in range(4):
    buf.zero_()
    cache.decode(0, ids, q, o)
    torch.cuda.synchronize()
t = buf.view(-1, 4).cpu().numpy()
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
ent, ex, units = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, t[:, 2]
print(f"B={B}: {len(t)} CTAs; entry spread {ent.min():.1f}..{ent.max():.1f} us; "
      f"finish min {ex.min():.1f} median {np.median(ex):.1f} p90 {np.percentile(ex, 90):.1f} max {ex.max():.1f} us")
print(f"  units per CTA: min {units.min()} median {np.median(units)} max {units.max()}")
print(f"  idle at the tail (sum over CTAs of max - finish) / (CTAs x max): {np.sum(ex.max() - ex) / (len(ex) * ex.max()):.3f}")
