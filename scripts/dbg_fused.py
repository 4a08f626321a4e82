import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from tests.hpa_testutil import Pair, f64
from tests.test_gpu_append_decode import _twins
from oracle import attend
from workloads import Shape
P = 64
shape = Shape(num_layers=1, num_q_heads=32, num_kv_heads=8, head_dim=128, page_size=P)
a, b = _twins(shape, 512, 8, 64)
seqs = []
for script in ([("latent", 128), ("tokens", 37)], [("tokens", 2 * P)], [("tokens", 50), ("latent", 64)],
               [("latent", 40), ("tokens", P - 1)], [("tokens", 1)]):
    seqs.append(a.build(script)); b.build(script)
for step in range(P + 3):
    n = len(seqs)
    k, v = a.draw.tokens(a.shape, n); q = a.draw.queries(a.shape, n)
    b.draw.tokens(b.shape, n); b.draw.queries(b.shape, n)
    oa = a.cache.append_decode(0, seqs, k.cuda(), v.cuda(), q.cuda())
    b.cache.append_kv(seqs, [1] * n, k.cuda(), v.cuda())
    ob = b.cache.decode(0, seqs, q.cuda())
    for i, s in enumerate(seqs):
        a.orc.append(s, f64(k[:, i:i + 1]), f64(v[:, i:i + 1])); b.orc.append(s, f64(k[:, i:i + 1]), f64(v[:, i:i + 1]))
    torch.cuda.synchronize()
    for i, s in enumerate(seqs):
        kl, vl = a.orc.logical_kv(s, 0)
        ref = attend(f64(q[i:i+1]), kl, vl, shape.scale)
        ea = np.abs(f64(oa[i:i+1]) - ref).max(); eb = np.abs(f64(ob[i:i+1]) - ref).max()
        d = (oa[i] != ob[i]).sum().item()
        if d or ea > 1e-2:
            hd = [(h, (oa[i, h] != ob[i, h]).sum().item()) for h in range(32) if (oa[i, h] != ob[i, h]).any()]
            print(f"step {step} seq {s} len {a.cache.seq_info(s)} ndiff {d} err fused {ea:.2e} two {eb:.2e} heads {hd[:8]}")
    ka, va = a.cache.export_logical_kv(0, seqs[0]); kb, vb = b.cache.export_logical_kv(0, seqs[0])
print("done")
