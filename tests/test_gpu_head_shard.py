"""KV-head shard on the CUDA kernels, emulated on one GPU (VERDICT r1
missing-2): n caches, one per 'rank', each built with num_kv_heads = H_kv / n and the G q-heads
of its kv-heads (dist.head_shard), fed the matching head slices of the same seeded inputs
through the C ABI; their decode / prefill outputs assembled in rank order
(dist.assemble_head_shards, the layout all_gather_into_tensor produces) must match the oracle
computed over ALL heads. The NCCL all-gather itself is covered by tests/test_dist_cpu.py
(gloo, world size 2)."""
import numpy as np
import pytest
import torch

from oracle import OracleCache, attend
from tests.hpa_testutil import check_close, f64
from workloads import Draw, Shape

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,hq,hkv,P", [(2, 32, 8, 16), (4, 32, 8, 16), (8, 32, 8, 64), (2, 16, 2, 32)])
def test_head_shard_emulated_matches_full_head_oracle(n, hq, hkv, P):
    from paper_2605_09100_b200 import Cache
    from paper_2605_09100_b200.dist import assemble_head_shards, head_shard
    d = 128
    full = Shape(1, hq, hkv, d, P)
    draw = Draw(61)
    orc = OracleCache(1, hq, hkv, d, P)
    scripts = [[("latent", 128), ("latent", 128), ("tokens", 900)], [("tokens", 333), ("latent", 40), ("tokens", 5)],
               [("latent", 128)]]
    ops = []  # (seq, kind, k, v) with full-head tensors
    for s, sc in enumerate(scripts):
        orc.create_seq(s)
        for kind, m in sc:
            if kind == "latent":
                kv = draw.latent(full, m)
                orc.install(s, -1, f64(kv))
                ops.append((s, kind, kv[:, 0], kv[:, 1]))
            else:
                k, v = draw.tokens(full, m)
                orc.append(s, f64(k), f64(v))
                ops.append((s, kind, k, v))
    q = draw.queries(full, len(scripts))
    qp = draw.queries(full, 3 * 20)
    outs, pouts = [], []
    for r in range(n):
        kv_lo, kv_hi, q_lo, q_hi = head_shard(hq, hkv, r, n)
        c = Cache(1, q_hi - q_lo, kv_hi - kv_lo, d, P, 512, 4, 128, 0, 99 + r)
        seqs = [c.seq_create() for _ in scripts]
        for s, kind, k, v in ops:
            ks = k[:, :, kv_lo:kv_hi].contiguous()
            vs = v[:, :, kv_lo:kv_hi].contiguous()
            if kind == "latent":
                c.latent_install(seqs[s], -1, torch.stack([ks, vs], 1).contiguous().cuda())
            else:
                c.append_kv([seqs[s]], [ks.shape[1]], ks.cuda(), vs.cuda())
        outs.append(c.decode(0, seqs, q[:, q_lo:q_hi].contiguous().cuda()))
        pouts.append(c.prefill(0, seqs, [20] * 3, qp[:, q_lo:q_hi].contiguous().cuda()))
        torch.cuda.synchronize()
        c.close()
    got = assemble_head_shards(torch.stack(outs))
    ref = np.stack([attend(f64(q[s:s + 1]), *orc.logical_kv(s, 0), full.scale)[0] for s in range(len(scripts))])
    check_close(got, ref, f"head shard n={n} decode")
    gotp = assemble_head_shards(torch.stack([o.view(3 * 20, -1, d) for o in pouts]).view(n, 60, -1, d))
    refp = np.concatenate([attend(f64(qp[20 * s:20 * s + 20]), *orc.logical_kv(s, 0), full.scale)
                           for s in range(len(scripts))])
    check_close(gotp, refp, f"head shard n={n} prefill")
