"""F32 fp8 decode debug: one case per invocation (CASE env), tiny shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import attend
from tests.hpa_testutil import Pair, f64
from workloads import Shape

case = os.environ.get("CASE", "t16")
scripts = {"t16": [("tokens", 16)], "t5": [("tokens", 5)], "t32": [("tokens", 32)], "t48": [("tokens", 48)],
           "t700": [("tokens", 700)], "lt": [("latent", 128), ("tokens", 40)], "tl": [("tokens", 17), ("latent", 64), ("tokens", 90)]}
shape = Shape(num_layers=1, num_q_heads=32, num_kv_heads=8, head_dim=128, page_size=16)
pr = Pair(shape, 512, 4, 160, seed=5, token_fp8=True, num_token_pages=512)
s = pr.build(scripts[case])
q = pr.queries(1)
print(case, "built", flush=True)
out = pr.cache.decode(0, [s], q.cuda())
torch.cuda.synchronize()
ref = attend(f64(q[0:1]), *pr.orc.logical_kv(s, 0), shape.scale)
print(case, "max abs err", float(np.abs(f64(out) - ref).max()), flush=True)
