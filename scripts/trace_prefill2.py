"""Prefill phase trace of CTA 0 (needs a -DHPA_TRACE=1 build loaded via HPA_LIB_PATH).
Events (clock64): 0 K issue, 1 mma got K(j+1), 2 mma got V(j), 3/4 mma got P0/P1 half0,
5/6 mma got P0/P1 half1, 7/8 softmax s_full passed, 9/10 S in registers, 11..14 P halves stored."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache
from paper_2605_09100_b200 import Cache
from paper_2605_09100_b200._lib import LIB
from workloads import qwen3_8b_shape
shape = qwen3_8b_shape(16)
cache, seqs, _ = build_decode_cache(torch, Cache, shape, 4, 8, 16384 + 2048, 0, 0, seed=777)
buf = torch.zeros(4096 + 8 * 8192, dtype=torch.int64, device="cuda")  # events + CTA timeline
LIB.hpa_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
LIB.hpa_debug_trace(cache._h, ctypes.c_void_p(buf.data_ptr()))
q = torch.randn((4 * 2048, 32, 128), device="cuda").to(torch.bfloat16)
cache.set_prefill_ctas(int(os.environ.get("PF_CTAS", "-1")))  # 0: the persistent kernel
for _ in range(3):
    cache.prefill(0, seqs, [2048] * 4, q)
torch.cuda.synchronize()
t = buf[:40 * 64].view(40, 64).cpu().long()
J = range(20, 30)
per = [int(t[7, j + 1] - t[7, j]) for j in J]
print("period (s_full0 j -> j+1):", per, "mean", sum(per) / len(per))
for s in (0, 1):
    sf, ld, h0, h1 = t[7 + s], t[9 + s], t[11 + 2 * s], t[12 + 2 * s]
    print(f"slot{s}: ldtm {[int(ld[j]-sf[j]) for j in J]}")
    print(f"slot{s}: ld->P half0 {[int(h0[j]-ld[j]) for j in J]}  half0->half1 {[int(h1[j]-h0[j]) for j in J]}")
    print(f"slot{s}: P half1 -> next s_full {[int(sf[j+1]-h1[j]) for j in J]}")
print("mma: got P0h0 after P0h0 stored:", [int(t[3, j] - t[11, j]) for j in J])
print("mma: got P1h0 after P1h0 stored:", [int(t[4, j] - t[13, j]) for j in J])
print("mma: s_full1(j) - s_full0(j):", [int(t[8, j] - t[7, j]) for j in J])
print("mma: got K(j+1) rel P0h1:", [int(t[1, j] - t[5, j]) for j in J])
print("mma: got V(j) rel s_full0(j):", [int(t[2, j] - t[7, j]) for j in J])

for s in (0, 1):
    print(f"slot{s} per-warp P half0 rel s_full{s}:", [[int(t[23 + 4 * s + w, j] - t[7 + s, j]) for w in range(4)] for j in range(20, 24)])
    print(f"slot{s} per-warp P done rel s_full{s}:", [[int(t[15 + 4 * s + w, j] - t[7 + s, j]) for w in range(4)] for j in range(20, 24)])
    print(f"slot{s} mma got half0 / half1 rel s_full{s}:", [(int(t[3 + s, j] - t[7 + s, j]), int(t[5 + s, j] - t[7 + s, j])) for j in range(20, 24)])

for s in (0, 1):
    print(f"slot{s} (warp q0): ld->opt exps done, ->max done, ->before st, exact path?:",
          [(int(t[31 + s, j] - t[9 + s, j]), int(t[33 + s, j] - t[31 + s, j]), int(t[35 + s, j] - t[33 + s, j]), int(t[37 + s, j] != 0)) for j in range(20, 26)])

for s in (0, 1):
    print(f"slot{s} (warp q0): ld -> before P st (exact path: max + exps):", [int(t[35 + s, j] - t[9 + s, j]) for j in range(20, 28)])
