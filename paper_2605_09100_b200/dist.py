"""Multi-GPU partitioning of the HPA path.

The paper serves on one GPU (tensor_parallel_size 1). Every
request's attention depends only on its own pages, so the
default partition is by request: rank r owns a contiguous block of requests,
one cache per GPU, and there is NO collective on the data path (weak scaling).

Optional KV-head shard: rank r holds kv-heads [r*H_kv/n, (r+1)*H_kv/n) of every
request (and their G q-heads each); outputs are gathered with one NCCL
all-gather over NVLink. It exists for latency / capacity, not throughput.
"""
from __future__ import annotations

from typing import List, Tuple

import torch
import torch.distributed as dist


def shard_requests(n_requests: int, rank: int, world: int) -> List[int]:
    """Contiguous block of request indices owned by `rank` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_requests, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return list(range(lo, hi))


def head_shard(num_q_heads: int, num_kv_heads: int, rank: int, world: int) -> Tuple[int, int, int, int]:
    """(kv_lo, kv_hi, q_lo, q_hi) of the heads owned by `rank` in KV-head-shard mode.
    The GQA mapping hq -> floor(hq / G) (reading A6) keeps q-heads with their kv-head."""
    if num_kv_heads % world != 0:
        raise ValueError("num_kv_heads must be divisible by the world size")
    g = num_q_heads // num_kv_heads
    per = num_kv_heads // world
    kv_lo, kv_hi = rank * per, (rank + 1) * per
    return kv_lo, kv_hi, kv_lo * g, kv_hi * g


def assemble_head_shards(gathered: torch.Tensor) -> torch.Tensor:
    """[n][B][Hq/n][d] (rank-major, as all_gather_into_tensor leaves it) -> [B][Hq][d]: rank r's
    q-heads are [r Hq/n, (r+1) Hq/n) (head_shard), so the full output is the rank-ordered
    concatenation along the head axis."""
    n, b, hl, d = gathered.shape
    return gathered.permute(1, 0, 2, 3).reshape(b, n * hl, d)


def gather_head_shards(out_local: torch.Tensor, group=None) -> torch.Tensor:
    """out_local [B][Hq/n][d] on every rank -> full [B][Hq][d] (rank-major head order)
    with one all_gather_into_tensor (NCCL over NVLink on GPUs, gloo on CPU). The payload is
    B Hq d 2 bytes (64 KB at configs[1]), latency-bound: NCCL's all-gather is the right tool
    (a fused peer-memory kernel would save microseconds on a step that sharding already slows)."""
    if not dist.is_available() or not dist.is_initialized():  # one process: its shard is everything
        return out_local
    world = dist.get_world_size(group)
    b, hl, d = out_local.shape
    buf = torch.empty((world * b, hl, d), dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(buf, out_local.contiguous(), group=group)
    return assemble_head_shards(buf.view(world, b, hl, d))


def max_over_ranks(x: float, device=None) -> float:
    """Timing reduction for reporting (max over ranks); not on the data path."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def context_parallel_decode(cache, layer: int, seq_ids, q: torch.Tensor, group=None) -> torch.Tensor:
    """Context-parallel decode (SURVEY §8(f) NEXT-4b): this rank's cache holds a row-range
    shard of every listed sequence. Partial attention per rank (hpa_decode_partial), one
    NCCL all-gather of the fp32 partials over NVLink, LSE merge (hpa_merge_partials).
    Returns bf16 [n][Hq][d] on every rank."""
    from .cache import merge_partials
    o, lse = cache.decode_partial(layer, seq_ids, q)
    o_all, l_all = gather_partials(o, lse, group)
    return merge_partials(o_all, l_all)


def gather_partials(o: torch.Tensor, lse: torch.Tensor, group=None):
    """All-gathers every rank's partial (o [n][Hq][d], lse [n][Hq]) into rank-major
    [world][n][Hq][d] / [world][n][Hq] (two all_gather_into_tensor calls)."""
    if not dist.is_available() or not dist.is_initialized():  # one process: world of one
        return o.unsqueeze(0), lse.unsqueeze(0)
    world = dist.get_world_size(group)
    o_all = torch.empty((world,) + tuple(o.shape), dtype=o.dtype, device=o.device)
    l_all = torch.empty((world,) + tuple(lse.shape), dtype=lse.dtype, device=lse.device)
    dist.all_gather_into_tensor(o_all.view(world * o.shape[0], *o.shape[1:]), o.contiguous(), group=group)
    dist.all_gather_into_tensor(l_all.view(world * lse.shape[0], *lse.shape[1:]), lse.contiguous(), group=group)
    return o_all, l_all
