"""Prefill phase trace (needs a -DHPA_TRACE build via HPA_LIB_PATH)."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache
from paper_2605_09100_b200 import Cache
from paper_2605_09100_b200._lib import LIB
from workloads import qwen3_8b_shape
shape = qwen3_8b_shape(16)
cache, seqs, _ = build_decode_cache(torch, Cache, shape, 4, 8, 16384 + 2048, 0, 0, seed=777)
buf = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
LIB.hpa_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
LIB.hpa_debug_trace(cache._h, ctypes.c_void_p(buf.data_ptr()))
q = torch.randn((4 * 2048, 32, 128), device="cuda").to(torch.bfloat16)
for _ in range(3):
    cache.prefill(0, seqs, [2048] * 4, q)
torch.cuda.synchronize()
t = buf.view(16, 64).cpu()
names = ["prod K issue", "mma k_full(j+1)", "mma v_full(j)", "mma p0 half0", "mma p1 half0", "mma p0 half1",
         "mma p1 half1", "sm0 s_full", "sm1 s_full", "sm0 ldtm done", "sm1 ldtm done", "sm0 p half0",
         "sm0 p half1", "sm1 p half0", "sm1 p half1"]
base = int(t[7, 0])
print("cycles relative to sm0 s_full(0)")
for j in range(20, 28):
    print(f"tile {j}: " + "  ".join(f"{names[e]}={int(t[e, j]) - base}" for e in range(15)))
print("per-tile period (sm0 s_full):", [(int(t[7, j + 1]) - int(t[7, j])) for j in range(20, 40)])
print("sm0 busy (s_full -> p half1):", [(int(t[12, j]) - int(t[7, j])) for j in range(20, 40)])
print("sm0 ldtm latency:", [(int(t[9, j]) - int(t[7, j])) for j in range(20, 40)])
print("p half1(sm0) -> s_full(sm0, j+1):", [(int(t[7, j + 1]) - int(t[12, j])) for j in range(20, 40)])
print("mma waits for p0 half0 after:", [(int(t[3, j]) - int(t[2, j])) for j in range(20, 40)])
