"""Host cost of hpa_decode (C ABI called directly) on forked batches, cascade on vs off."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_09100_b200 import Cache  # noqa: E402
from paper_2605_09100_b200._lib import LIB  # noqa: E402
from paper_2605_09100_b200.cache import _p32, _stream  # noqa: E402

P = 16
for B, n_prompt, n_own in ((64, 4096, 1024), (256, 4096, 1024)):
    pages = n_prompt // P + B * (n_own // P + 2) + 64
    cache = Cache(1, 32, 8, 128, P, pages, B + 1, (n_prompt + n_own) // P + 4, 0, 99)
    src = cache.seq_create()
    kp = torch.randn((1, n_prompt, 8, 128), device="cuda").to(torch.bfloat16)
    cache.append_kv([src], [n_prompt], kp, kp)
    seqs = [cache.seq_fork(src, n_prompt) for _ in range(B)]
    ko = torch.randn((1, B * n_own, 8, 128), device="cuda").to(torch.bfloat16)
    cache.append_kv(seqs, [n_own] * B, ko, ko)
    ids = np.asarray(seqs, dtype=np.int32)
    q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    args = (cache._h, 0, B, _p32(ids), ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(o.data_ptr()), 0.0,
            _stream(0, None))
    res = []
    for on in (False, True):
        cache.set_decode_cascade(on)
        for _ in range(5):
            LIB.hpa_decode(*args)
        torch.cuda.synchronize()
        N = 100
        t0 = time.perf_counter()
        for _ in range(N):
            LIB.hpa_decode(*args)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        res.append(1e6 * (t1 - t0) / N)
    print(f"B={B} prompt={n_prompt}: host per hpa_decode: plain {res[0]:.1f} us, cascade {res[1]:.1f} us", flush=True)
    cache.close()
