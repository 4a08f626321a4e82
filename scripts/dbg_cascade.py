"""Cascade decode debug: one case per invocation (CASE env), tiny shapes; on/off vs oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import attend
from tests.hpa_testutil import Pair, f64
from workloads import Shape

case = os.environ.get("CASE", "a")
hq, hkv = (8, 2) if case in ("a", "b", "c") else (32, 8)
shape = Shape(num_layers=1, num_q_heads=hq, num_kv_heads=hkv, head_dim=128, page_size=16)
p = Pair(shape, 1024, 16, 64, seed=5)
def fork(src, n):
    d = p.cache.seq_fork(src, n); p.orc.fork(src, n, d); return d
if case == "a":    # two requests, fork with own rows
    src = p.build([("tokens", 100)]); f = fork(src, 100); p.tokens([f], [5]); seqs = [src, f]
elif case == "b":  # the failing test's shape
    src = p.build([("latent", 32), ("tokens", 40)]); f = fork(src, 67); seqs = [f, src]
    p.tokens(seqs, [1, 1])
elif case == "c":  # 4 forks, no own rows
    src = p.build([("tokens", 128)]); seqs = [src] + [fork(src, 128) for _ in range(3)]
else:              # G=4 32 heads, 10 forks with own rows
    src = p.build([("tokens", 300)]); seqs = [src] + [fork(src, 300) for _ in range(9)]
    for i, s in enumerate(seqs): p.tokens([s], [1 + i])
q = p.queries(len(seqs))
ref = np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, 0), shape.scale)[0] for i, s in enumerate(seqs)])
for on in (False, True):
    p.cache.set_decode_cascade(on)
    out = p.cache.decode(0, seqs, q.cuda())
    torch.cuda.synchronize()
    err = np.abs(f64(out) - ref).reshape(len(seqs), -1).max(axis=1)
    print(case, "cascade" if on else "plain  ", p.cache.decode_plan_info(), "err per req", np.round(err, 4), flush=True)
