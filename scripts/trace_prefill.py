"""Prefill phase trace (needs a -DHPA_TRACE build via HPA_LIB_PATH)."""
import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_decode_cache
from paper_2605_09100_b200 import Cache
from paper_2605_09100_b200._lib import LIB
from workloads import qwen3_8b_shape
shape = qwen3_8b_shape(16)
cache, seqs, _ = build_decode_cache(torch, Cache, shape, 4, 8, 16384 + 2048, 0, 0, seed=777)
buf = torch.zeros(27 * 64, dtype=torch.int64, device="cuda")
LIB.hpa_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
LIB.hpa_debug_trace(cache._h, ctypes.c_void_p(buf.data_ptr()))
q = torch.randn((4 * 2048, 32, 128), device="cuda").to(torch.bfloat16)
for _ in range(3):
    cache.prefill(0, seqs, [2048] * 4, q)
torch.cuda.synchronize()
t = buf.view(27, 64).cpu()
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

print("V issue (j) rel:", [int(t[15, j]) - base for j in range(20, 30)])
print("mma before v_full wait:", [int(t[16, j]) - base for j in range(20, 30)])
print("mma after v_full wait:", [int(t[2, j]) - base for j in range(20, 30)])
print("mma end of iteration:", [int(t[17, j]) - base for j in range(20, 30)])
print("V latency issue->mma got it:", [int(t[2, j]) - int(t[15, j]) for j in range(20, 30)])
print("mma v_full wait duration:", [int(t[2, j]) - int(t[16, j]) for j in range(20, 30)])
print("mma iteration (v wait -> end):", [int(t[17, j]) - int(t[2, j]) for j in range(20, 30)])

print("sm slot0 busy (s_full0 -> p0 half0/half1):", [(int(t[11, j]) - int(t[7, j]), int(t[12, j]) - int(t[7, j])) for j in range(20, 28)])
print("sm slot1 busy (s_full1 -> p1 half0/half1):", [(int(t[13, j]) - int(t[8, j]), int(t[14, j]) - int(t[8, j])) for j in range(20, 28)])
print("s_full1 - s_full0:", [int(t[8, j]) - int(t[7, j]) for j in range(20, 28)])
print("p0 done -> s_full1 wait passed:", [int(t[8, j]) - int(t[12, j]) for j in range(20, 28)])
print("p1 done -> s_full0(j+1):", [int(t[7, j+1]) - int(t[14, j]) for j in range(20, 28)])

print("phases slot0 hs0 (from s_full0): ldtm, max-done(before bar), after bar, before rescale, exps done, st done, p arrive")
for j in range(20, 26):
    b0 = int(t[7, j])
    print(j, [int(t[e, j]) - b0 for e in (18, 19, 20, 23, 21, 22, 11)], "rescaled" if int(t[24, j]) > 0 else "")

print("K issue -> arrival:", [int(t[25, j]) - int(t[0, j]) for j in range(20, 30)])
print("V issue -> arrival:", [int(t[26, j]) - int(t[15, j]) for j in range(20, 30)])
print("K(j+1) arrival - mma wants it (p0 half1 stamp j):", [int(t[25, j + 1]) - int(t[5, j]) for j in range(20, 30)])
print("V(j) arrival - mma wants it (p0 half0 j):", [int(t[26, j]) - int(t[3, j]) for j in range(20, 30)])
print("K issue(j+1) - K release needed (k_empty: S1(j-1) issue ~ mma end of iter j-2):", [int(t[0, j + 1]) - int(t[17, j - 2]) for j in range(20, 30)])
print("warp0: busy slot0, wait S1, busy slot1, wait S0(j+1):")
for j in range(20, 28):
    print(j, int(t[11, j]) - int(t[7, j]), int(t[8, j]) - int(t[11, j]), int(t[13, j]) - int(t[8, j]), int(t[7, j + 1]) - int(t[13, j]))
print("mma: p0h0 pass -> p0h1 pass -> k -> p1h0 pass -> p1h1 pass -> end (absolute rel to s_full0(j)):")
for j in range(20, 28):
    b0 = int(t[7, j])
    print(j, [int(t[e, j]) - b0 for e in (3, 5, 1, 4, 6, 17)])
