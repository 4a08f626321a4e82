"""Split-KV chunked prefill (SURVEY §8(a) a6 with the a5 LSE merge): units of an under-filled
last wave run as several key ranges whose partial (O / l, LSE) results are merged.

Parity with the fp64 oracle for forced split counts (including more pieces than key tiles,
i.e. empty pieces), the GRC span mask, ragged query lengths, G odd, D = 64, and the planner's
own choice at configs[2] B = 1 (the case it exists for)."""
import numpy as np
import pytest
import torch

from oracle import attend, attend_span
from tests.hpa_testutil import Pair, check_close, f64
from workloads import Shape

pytestmark = pytest.mark.gpu


def _oracle_prefill(pair, seqs, q_lens, q):
    out, off = [], 0
    for s, n in zip(seqs, q_lens):
        k, v = pair.orc.logical_kv(s, 0)
        out.append(attend(f64(q[off:off + n]), k, v, pair.shape.scale))
        off += n
    return np.concatenate(out)


@pytest.mark.parametrize("hq,hkv,d,P", [(32, 8, 128, 16), (6, 2, 64, 32), (16, 1, 128, 64), (4, 4, 128, 256)])
@pytest.mark.parametrize("splits", [2, 3, 8, 15, 16])
def test_prefill_forced_splits_parity(hq, hkv, d, P, splits):
    shape = Shape(1, hq, hkv, d, P)
    p = Pair(shape, num_pages=4096, max_seqs=4, max_pages_per_seq=1024)
    scripts = [[("latent", 128), ("latent", 8), ("tokens", 700)],
               [("tokens", 77)],                                   # 1 key tile: pieces >= 1 empty
               [("latent", 128)] * 2 + [("tokens", 1500)]]
    seqs = [p.build(sc) for sc in scripts]
    q_lens = [300, 1, 385]
    q = p.queries(sum(q_lens))
    ref = _oracle_prefill(p, seqs, q_lens, q)
    p.cache.set_prefill_splits(splits)
    got = p.cache.prefill(0, seqs, q_lens, q.cuda())
    torch.cuda.synchronize()
    check_close(got, ref, f"prefill split {splits} {hq}/{hkv}/{d}/P{P}")
    # the unsplit kernel on the same data agrees to bf16 output rounding
    p.cache.set_prefill_splits(1)
    one = p.cache.prefill(0, seqs, q_lens, q.cuda())
    torch.cuda.synchronize()
    assert torch.max(torch.abs(one.float() - got.float())).item() <= 1.6e-2


@pytest.mark.parametrize("splits", [0, 4])
def test_prefill_split_with_span(splits):
    """Pieces that lie entirely inside the GRC mask-out span leave span rows with nothing
    visible (LSE = -inf); the merge must weight them 0."""
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=2048, max_seqs=8, max_pages_per_seq=256)
    cases = [(900, 16, 150), (40, 128, 200), (257, 64, 1)]
    seqs, q_lens, spans = [], [], []
    for n1, m, n3 in cases:
        s = p.new_seq()
        p.tokens([s], [n1])
        p.latent(s, m)
        p.tokens([s], [n3])
        seqs.append(s)
        q_lens.append(m + n3)
        spans.append((0, n1, n1 + m))
    q = p.queries(sum(q_lens))
    p.cache.set_prefill_splits(splits)
    got = p.cache.prefill_span(0, seqs, q_lens, spans, q.cuda())
    torch.cuda.synchronize()
    ref, off = [], 0
    for s, ql, (lo, hi, qf) in zip(seqs, q_lens, spans):
        k, v = p.orc.logical_kv(s, 0)
        ref.append(attend_span(f64(q[off:off + ql]), k, v, shape.scale, lo, hi, qf))
        off += ql
    check_close(got, np.concatenate(ref), f"prefill span split {splits}")


@pytest.mark.parametrize("ctas", [-3, -1])
def test_prefill_planner_small_batch_fills_sms(ctas):
    """Planner (splits = 0) on a batch of fewer units than SMs: every unit is split -- into
    equal pieces of one CTA each (-3) or into stream-K shares of the persistent kernel (-1,
    the default under 4 waves); parity."""
    shape = Shape(1, 8, 2, 128, 16)
    p = Pair(shape, num_pages=4096, max_seqs=2, max_pages_per_seq=1024)
    s = p.build([("latent", 128), ("tokens", 6000)])
    q = p.queries(512)
    p.cache.set_prefill_ctas(ctas)
    p.cache.set_prefill_splits(1)
    p.cache.prefill(0, [s], [512], q.cuda())          # ships pending table writes
    before = p.cache.launch_count()
    p.cache.prefill(0, [s], [512], q.cuda())
    n_one = p.cache.launch_count() - before
    p.cache.set_prefill_splits(0)
    before = p.cache.launch_count()
    got = p.cache.prefill(0, [s], [512], q.cuda())
    torch.cuda.synchronize()
    assert p.cache.launch_count() - before == n_one + 1, "split plan: prefill + merge kernels"
    info = p.cache.prefill_plan_info()
    assert info["split_units"] == 16 and info["splits"] >= 2, info
    if ctas == -3:
        assert 1 <= info["ctas"] <= 16 * info["splits"], info
    check_close(got, _oracle_prefill(p, [s], [512], q), f"prefill planner small batch ctas={ctas}")


def test_prefill_split_invalid_count():
    shape = Shape(1, 8, 2, 128, 16)
    p = Pair(shape, num_pages=64, max_seqs=2, max_pages_per_seq=16)
    with pytest.raises(Exception):
        p.cache.set_prefill_splits(17)
    with pytest.raises(Exception):
        p.cache.set_prefill_splits(-1)


@pytest.mark.parametrize("hq,hkv,d,P", [(32, 8, 128, 16), (6, 2, 64, 32), (3, 1, 128, 64)])
@pytest.mark.parametrize("ctas,splits", [(1, 1), (3, 1), (5, 3), (2, 0), (-1, 0)])
def test_prefill_persistent_many_items_per_cta(hq, hkv, d, P, ctas, splits):
    """The persistent kernel with the CTA count capped so every CTA loops over many items:
    short items (1 key tile) next to long ones, G odd (a dead second slot in ragged items),
    split pieces; parity and agreement with the one-CTA-per-item kernel."""
    shape = Shape(1, hq, hkv, d, P)
    p = Pair(shape, num_pages=4096, max_seqs=4, max_pages_per_seq=1024)
    scripts = [[("latent", 128), ("latent", 8), ("tokens", 700)],
               [("tokens", 77)],
               [("latent", 128)] * 2 + [("tokens", 1500)]]
    seqs = [p.build(sc) for sc in scripts]
    q_lens = [300, 1, 385]
    q = p.queries(sum(q_lens))
    ref = _oracle_prefill(p, seqs, q_lens, q)
    p.cache.set_prefill_splits(splits)
    p.cache.set_prefill_ctas(ctas)
    got = p.cache.prefill(0, seqs, q_lens, q.cuda())
    torch.cuda.synchronize()
    info = p.cache.prefill_plan_info()
    if ctas > 0:
        assert 1 <= info["ctas"] <= ctas, info
    check_close(got, ref, f"persistent prefill ctas={ctas} splits={splits} {hq}/{hkv}/{d}/P{P}")


def test_prefill_persistent_span():
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=2048, max_seqs=8, max_pages_per_seq=256)
    cases = [(900, 16, 150), (40, 128, 200), (257, 64, 1)]
    seqs, q_lens, spans = [], [], []
    for n1, m, n3 in cases:
        s = p.new_seq()
        p.tokens([s], [n1])
        p.latent(s, m)
        p.tokens([s], [n3])
        seqs.append(s)
        q_lens.append(m + n3)
        spans.append((0, n1, n1 + m))
    q = p.queries(sum(q_lens))
    p.cache.set_prefill_ctas(2)
    p.cache.set_prefill_splits(2)
    got = p.cache.prefill_span(0, seqs, q_lens, spans, q.cuda())
    torch.cuda.synchronize()
    ref, off = [], 0
    for s, ql, (lo, hi, qf) in zip(seqs, q_lens, spans):
        k, v = p.orc.logical_kv(s, 0)
        ref.append(attend_span(f64(q[off:off + ql]), k, v, shape.scale, lo, hi, qf))
        off += ql
    check_close(got, np.concatenate(ref), "persistent prefill span")


@pytest.mark.parametrize("splits", [0, 3])
def test_prefill_plan_cache_follows_table_changes(splits):
    """The cached prefill plan (tile ranges computed on the host) must be rebuilt when the
    table changes under an identical call (same sequence ids and q_lens): after appends, after a
    latent set is replaced by one of another size, and after a latent set is removed."""
    shape = Shape(1, 8, 2, 128, 16)
    p = Pair(shape, num_pages=4096, max_seqs=4, max_pages_per_seq=1024)
    s = p.new_seq()
    set_a = p.latent(s, 128)
    p.tokens([s], [700])
    p.cache.set_prefill_splits(splits)

    def check(tag):
        q = p.queries(200)
        got = p.cache.prefill(0, [s], [200], q.cuda())
        torch.cuda.synchronize()
        check_close(got, _oracle_prefill(p, [s], [200], q), f"plan cache {tag} splits={splits}")

    check("initial")
    check("repeat")                     # plan reused
    p.tokens([s], [300])
    check("after append")
    p.latent(s, 40, set_a)              # replace the 128-row set by a 40-row one (splice)
    check("after replace")
    p.cache.latent_remove(s, set_a)
    p.orc.remove(s, set_a)
    check("after remove")


@pytest.mark.parametrize("token_fp8", [False, True])
@pytest.mark.parametrize("splits", [1, 3])
def test_prefill_upper_layer(token_fp8, splits):
    """Prefill of layer 2 of a 3-layer cache (the K/V rows of layer l live at pool rows
    l * NP * H_kv * P + ...): parity per layer, and each layer's output differs."""
    shape = Shape(3, 8, 2, 128, 16)
    p = Pair(shape, num_pages=2048, max_seqs=4, max_pages_per_seq=512, token_fp8=token_fp8,
             num_token_pages=1024 if token_fp8 else 0)
    seqs = [p.build([("latent", 128), ("tokens", 500)]), p.build([("tokens", 260), ("latent", 8), ("tokens", 40)])]
    q_lens = [300, 140]
    q = p.queries(sum(q_lens))
    p.cache.set_prefill_splits(splits)
    outs = []
    for layer in (2, 0):
        got = p.cache.prefill(layer, seqs, q_lens, q.cuda())
        torch.cuda.synchronize()
        ref, off = [], 0
        for s, n in zip(seqs, q_lens):
            k, v = p.orc.logical_kv(s, layer)
            ref.append(attend(f64(q[off:off + n]), k, v, shape.scale))
            off += n
        check_close(got, np.concatenate(ref), f"prefill layer {layer} fp8={token_fp8} splits={splits}")
        outs.append(got.float())
    assert torch.max(torch.abs(outs[0] - outs[1])).item() > 0.05


@pytest.mark.parametrize("hq,hkv,P", [(32, 8, 16), (16, 2, 64), (16, 1, 256)])
@pytest.mark.parametrize("splits", [0, 1, 3])
def test_prefill_cluster_pairs_multicast(hq, hkv, P, splits):
    """Forced 2-CTA clusters (hpa_set_prefill_ctas(c, -2); G % 4 == 0): the two head-pair units
    of a KV head share every K/V box by TMA multicast; ragged q_len, splits, parity."""
    shape = Shape(1, hq, hkv, 128, P)
    p = Pair(shape, num_pages=4096, max_seqs=4, max_pages_per_seq=1024)
    scripts = [[("latent", 128), ("latent", 8), ("tokens", 700)],
               [("tokens", 77)],
               [("latent", 128)] * 2 + [("tokens", 1500)]]
    seqs = [p.build(sc) for sc in scripts]
    q_lens = [300, 1, 385]
    q = p.queries(sum(q_lens))
    p.cache.set_prefill_splits(splits)
    p.cache.set_prefill_ctas(-2)
    got = p.cache.prefill(0, seqs, q_lens, q.cuda())
    torch.cuda.synchronize()
    check_close(got, _oracle_prefill(p, seqs, q_lens, q), f"cluster prefill {hq}/{hkv}/P{P} splits={splits}")


def test_prefill_many_short_sequences_cluster_waves():
    """200 sequences with q_len 1..5 (one ragged row tile each): enough units for >= 4 waves,
    so the default plan runs 2-CTA multicast clusters; parity on every row."""
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=8192, max_seqs=200, max_pages_per_seq=64)
    rng = np.random.default_rng(5)
    seqs = []
    for i in range(200):
        s = p.new_seq()
        if i % 3 == 0:
            p.latent(s, 128)
        p.tokens([s], [int(rng.integers(5, 300))])
        seqs.append(s)
    q_lens = [int(rng.integers(1, 6)) for _ in seqs]
    q = p.queries(sum(q_lens))
    got = p.cache.prefill(0, seqs, q_lens, q.cuda())
    torch.cuda.synchronize()
    check_close(got, _oracle_prefill(p, seqs, q_lens, q), "many short sequences")


@pytest.mark.parametrize("hq,hkv,d,P,rows,ql", [(2, 1, 128, 16, 9000, 128), (3, 1, 64, 16, 7000, 200),
                                                (4, 2, 128, 32, 6000, 300)])
def test_prefill_default_plan_few_long_units(hq, hkv, d, P, rows, ql):
    """Default plan on batches of a handful of very long units (few heads, one long sequence):
    stream-K would cut a unit into more than 15 pieces, so the planner falls back to the
    list-scheduled split plan of the persistent kernel; parity with the oracle either way."""
    shape = Shape(1, hq, hkv, d, P)
    p = Pair(shape, num_pages=rows // P + 64, max_seqs=2, max_pages_per_seq=rows // P + 32)
    s = p.build([("latent", 128), ("tokens", rows)])
    q = p.queries(ql)
    got = p.cache.prefill(0, [s], [ql], q.cuda())
    torch.cuda.synchronize()
    info = p.cache.prefill_plan_info()
    assert info["ctas"] >= 1 and info["splits"] <= 15, info
    check_close(got, _oracle_prefill(p, [s], [ql], q), f"few long units {hq}/{hkv}/{d}/P{P}")
