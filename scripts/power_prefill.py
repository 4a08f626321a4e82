"""Runs configs[2] prefill (B=4) back to back for ~4 s while nvidia-smi logs SM clock, power and
throttle reasons every 50 ms (power / clock behaviour of the tensor-bound kernel)."""
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

shape = qwen3_8b_shape(16)
bp = int(os.environ.get("B", "4"))
cache, seqs, _ = bench.build_decode_cache(torch, Cache, shape, bp, 8, 16384 + 2048, 0, 0, seed=777)
q = torch.randn((bp * 2048, 32, 128), device="cuda").to(torch.bfloat16)
cache.set_prefill_ctas(int(os.environ.get("PF_CTAS", "-1")))  # 0: the persistent kernel
o = torch.empty_like(q)
for _ in range(3):
    cache.prefill(0, seqs, [2048] * bp, q, o)
torch.cuda.synchronize()
log = open(os.environ.get("OUT", "gpurun_out/power.csv"), "w")
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active",
                        "--format=csv,noheader", "-lms", "50"], stdout=log)
time.sleep(0.5)
flops = bp * bench.prefill_flops(8 * 128 + 16384, 2048, shape)
t0 = time.time()
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        cache.prefill(0, seqs, [2048] * bp, q, o)
    n += 20
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
time.sleep(0.3)
smi.terminate()
print(f"B={bp} ctas={os.environ.get('PF_CTAS', '-1')}: {n} calls, {ms * 1e3:.1f} us per call, {flops / ms / 1e9:.1f} TFLOP/s sustained")
