import sys, torch, numpy as np
sys.path.insert(0, ".")
from tests.hpa_testutil import Pair, f64
from workloads import Shape
from tests.test_gpu_parity import oracle_decode, oracle_prefill

def report(tag, got, ref, rows):
    g = f64(got)
    bad = ~np.isfinite(g)
    err = np.where(bad, 0, np.abs(g - ref))
    print(tag, "nan rows:", [r for r in range(g.shape[0]) if bad[r].any()],
          "nan heads(row0..):", [list(np.where(bad[r].any(-1))[0]) for r in rows],
          "max err finite:", err.max())

for P, L, NP in [(16, 2, 2048), (16, 1, 2048), (16, 1, 256)]:
    shape = Shape(L, 32, 8, 128, P)
    p = Pair(shape, num_pages=NP, max_seqs=8, max_pages_per_seq=512)
    scripts = [[("latent", 128)] * 3 + [("tokens", 700)], [("tokens", 1)],
               [("latent", 8), ("tokens", 33), ("latent", 128), ("tokens", 250)],
               [("latent", 128), ("latent", 100)], [("tokens", 2000 if NP > 256 else 500)]]
    seqs = [p.build(sc) for sc in scripts]
    q = p.queries(len(seqs))
    for S in (1, 2, 3, 11):
        p.cache.set_decode_splits(S)
        got = p.cache.decode(L - 1, seqs, q.cuda()); torch.cuda.synchronize()
        report(f"decode P{P} L{L} NP{NP} S{S}", got, oracle_decode(p, seqs, q, layer=L - 1), range(5))
    for sl in ([0], [1], [4], [0, 4]):
        ss = [seqs[i] for i in sl]
        got = p.cache.decode(L - 1, ss, q[sl].cuda()); torch.cuda.synchronize()
        report(f"decode subset {sl}", got, oracle_decode(p, ss, q[sl], layer=L - 1), range(len(sl)))

shape = Shape(1, 32, 8, 128, 16)
p = Pair(shape, num_pages=4096, max_seqs=4, max_pages_per_seq=1024)
scripts = [[("latent", 128), ("latent", 8), ("tokens", 300)], [("tokens", 77)], [("latent", 128)] * 2 + [("tokens", 900)]]
seqs = [p.build(sc) for sc in scripts]
for ql_set in ([300, 1, 385], [300], [1], [385]):
    idx = {3: [0, 1, 2], 1: None}
    if len(ql_set) == 3: ss, ql = seqs, ql_set
    else:
        i = {300: 0, 1: 1, 385: 2}[ql_set[0]]; ss, ql = [seqs[i]], ql_set
    q = p.queries(sum(ql))
    got = p.cache.prefill(0, ss, ql, q.cuda()); torch.cuda.synchronize()
    g = f64(got); ref = oracle_prefill(p, ss, ql, q)
    bad = ~np.isfinite(g)
    print("prefill", ql, "nan token rows:", np.where(bad.any(axis=(1, 2)))[0][:20], "count", bad.any(axis=(1,2)).sum(),
          "nan heads:", np.where(bad.any(axis=(0, 2)))[0], "max err finite", np.where(bad, 0, np.abs(g - ref)).max())
