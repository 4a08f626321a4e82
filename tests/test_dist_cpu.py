"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

Request sharding must cover every request exactly once with no collective;
KV-head shard + all-gather must reconstruct the full output (checked against
the oracle computed on all heads)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import attend


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2605_09100_b200.dist import gather_head_shards, head_shard, max_over_ranks
        rng = np.random.default_rng(7)                     # same data on every rank
        hq, hkv, d, lb, b = 8, 4, 16, 50, 3
        q = rng.standard_normal((b, hq, d))
        k = rng.standard_normal((b, hkv, lb, d))
        v = rng.standard_normal((b, hkv, lb, d))
        full = np.stack([attend(q[i:i + 1], k[i], v[i], 0.25)[0] for i in range(b)])
        kv_lo, kv_hi, q_lo, q_hi = head_shard(hq, hkv, rank, world)
        local = np.stack([attend(q[i:i + 1, q_lo:q_hi], k[i, kv_lo:kv_hi], v[i, kv_lo:kv_hi], 0.25)[0]
                          for i in range(b)])
        got = gather_head_shards(torch.from_numpy(local))
        ok = bool(np.max(np.abs(got.numpy() - full)) <= 1e-12)
        # context-parallel decode plumbing: each rank holds a row-range shard of every request
        from oracle import merge_partials, partial_attend
        from paper_2605_09100_b200.dist import gather_partials
        cut = [0, 23, lb][rank:rank + 2]
        parts = [partial_attend(q[i], k[i][:, cut[0]:cut[1]], v[i][:, cut[0]:cut[1]], 0.25) for i in range(b)]
        o_all, l_all = gather_partials(torch.from_numpy(np.stack([p[0] for p in parts])),
                                       torch.from_numpy(np.stack([p[1] for p in parts])))
        merged = merge_partials(o_all.numpy(), l_all.numpy())
        ok = ok and bool(np.max(np.abs(merged - full)) <= 1e-12)
        mx = max_over_ranks(float(rank + 1))
        ret[rank] = (ok, mx)
    finally:
        dist.destroy_process_group()


def test_head_shard_all_gather_gloo_world2():
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), ret), nprocs=2, join=True)
    assert ret[0] == (True, 2.0) and ret[1] == (True, 2.0)


@pytest.mark.parametrize("n,world", [(64, 1), (64, 2), (64, 8), (7, 4), (4096, 8), (3, 8)])
def test_shard_requests_partition(n, world):
    from paper_2605_09100_b200.dist import shard_requests
    parts = [shard_requests(n, r, world) for r in range(world)]
    flat = [i for p in parts for i in p]
    assert sorted(flat) == list(range(n)) and len(flat) == n
    sizes = [len(p) for p in parts]
    assert max(sizes) - min(sizes) <= 1


def test_head_shard_bounds():
    from paper_2605_09100_b200.dist import head_shard
    assert head_shard(32, 8, 3, 4) == (6, 8, 24, 32)
    with pytest.raises(ValueError):
        head_shard(32, 8, 0, 3)


def test_gathers_without_process_group():
    """One process (no torch.distributed group): the gathers return this process's data as the
    whole (bench.py --mode head_shard | context_parallel at N = 1)."""
    import torch

    from paper_2605_09100_b200.dist import gather_head_shards, gather_partials
    o = torch.randn(3, 8, 16)
    assert gather_head_shards(o) is o
    p, lse = torch.randn(3, 8, 16), torch.randn(3, 8)
    pa, la = gather_partials(p, lse)
    assert pa.shape == (1, 3, 8, 16) and la.shape == (1, 3, 8)
    assert torch.equal(pa[0], p) and torch.equal(la[0], lse)
