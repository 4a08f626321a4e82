"""Phase trace of the HPA_PF1 prefill (needs -DHPA_PF1=1 -DHPA_TRACE=1, via HPA_LIB_PATH)."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache
from paper_2605_09100_b200 import Cache
from paper_2605_09100_b200._lib import LIB
from workloads import qwen3_8b_shape
shape = qwen3_8b_shape(16)
cache, seqs, _ = build_decode_cache(torch, Cache, shape, 4, 8, 16384 + 2048, 0, 0, seed=777)
buf = torch.zeros(40 * 64, dtype=torch.int64, device="cuda")
LIB.hpa_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
LIB.hpa_debug_trace(cache._h, ctypes.c_void_p(buf.data_ptr()))
q = torch.randn((4 * 2048, 32, 128), device="cuda").to(torch.bfloat16)
for _ in range(3):
    cache.prefill(0, seqs, [2048] * 4, q)
torch.cuda.synchronize()
t = buf.view(40, 64).cpu().long()
J = range(20, 30)
print("period s_full(j) (hc0):", [int(t[7, j + 1] - t[7, j]) for j in J])
print("softmax hc0: s_full -> P stored:", [int(t[11, j] - t[7, j]) for j in J])
print("softmax hc1: s_full -> P stored:", [int(t[12, j] - t[8, j]) for j in J])
print("mma got P half0 rel P stored hc0:", [int(t[3, j] - t[11, j]) for j in J])
print("mma got P half1 rel P stored hc1:", [int(t[4, j] - t[12, j]) for j in J])
print("s_full(j+1) - P stored(j) hc0:", [int(t[7, j + 1] - t[11, j]) for j in J])
print("K issue -> ? (ev0):", [int(t[0, j + 1] - t[0, j]) for j in J])
print("mma: iteration start (before v wait) rel s_full0(j):", [int(t[5, j] - t[7, j]) for j in J])
print("mma: v_full wait duration:", [int(t[2, j] - t[5, j]) for j in J])
print("mma: got P0 rel v done:", [int(t[3, j] - t[2, j]) for j in J])
print("mma: k_full(j+2) got rel P1 got (j):", [int(t[1, j + 2] - t[4, j]) for j in J])
print("K producer issue (ev0) j+2 rel mma wants (P1 got j):", [int(t[0, j + 2] - t[4, j]) for j in J])
print("K prod: c_empty wait:", [int(t[14, j] - t[13, j]) for j in J])
print("K prod: mask work (after c wait -> before k wait):", [int(t[15, j] - t[14, j]) for j in J])
print("K prod: k_empty wait:", [int(t[0, j] - t[15, j]) for j in J])
print("K prod: loop (issue j -> top j+1):", [int(t[13, j + 1] - t[0, j]) for j in J])
