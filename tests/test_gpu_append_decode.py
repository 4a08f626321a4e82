"""Fused decode step (hpa_append_decode: a2 + a4 + a5 in one launch; "store ... into the
corresponding blocks", then attention over the logical sequence).

The call is defined as hpa_append_kv(1 row each) followed by hpa_decode, so it is checked three
ways on the same seeded inputs:
  * against the oracle (OracleCache.append, then attend over the logical K/V) at the north_star
    tolerance;
  * bit-exactly against a twin cache driven with the two separate calls (same placement seed,
    same ops): outputs, logical K/V (export kernel over the DEVICE table the fused kernel wrote
    back), tables and allocator counts;
  * afterwards, plain decode and prefill over the written-back device table match the oracle.
Cases: page-boundary crossings (P = 16, 64), sequences ending in a latent set (a new token
segment starts), forked prefixes with a shared partial last page (copy-on-write before the
fused kernel), 2 layers decoded at layer 1, G = 16 (non-swapped consumers), d = 64, batches on
both parameter-block variants (<= 64, <= 512) and above 512 (two-launch path), fp8 token
pages (two-launch path), and argument errors leaving the cache unchanged."""
import numpy as np
import pytest
import torch

from oracle import attend
from paper_2605_09100_b200 import HPAError
from tests.hpa_testutil import Pair, check_close, f64
from workloads import Shape

pytestmark = pytest.mark.gpu


def _twins(shape, num_pages, max_seqs, max_pages, seed=7, **kw):
    a = Pair(shape, num_pages, max_seqs, max_pages, seed=seed, **kw)   # fused
    b = Pair(shape, num_pages, max_seqs, max_pages, seed=seed, **kw)   # append_kv + decode
    return a, b


def _same_state(a, b, seqs, layers):
    torch.cuda.synchronize()
    assert a.cache.stats() == b.cache.stats()
    for s in seqs:
        assert a.cache.seq_info(s) == b.cache.seq_info(s)
        ta, tb = a.cache.export_table(s), b.cache.export_table(s)
        for x, y in zip(ta, tb):
            assert np.array_equal(np.asarray(x), np.asarray(y)), s
        for layer in layers:
            ka, va = a.cache.export_logical_kv(layer, s)
            kb, vb = b.cache.export_logical_kv(layer, s)
            assert torch.equal(ka, kb) and torch.equal(va, vb), (s, layer)
            k1, v1 = a.orc.logical_kv(s, layer)
            assert np.array_equal(f64(ka), k1) and np.array_equal(f64(va), v1), (s, layer)


def _step(a, b, seqs, layer, check_oracle=True):
    """One decode step on both twins with the same new rows and queries."""
    n = len(seqs)
    k, v = a.draw.tokens(a.shape, n)
    q = a.draw.queries(a.shape, n)
    b.draw.tokens(b.shape, n)
    b.draw.queries(b.shape, n)
    out_a = a.cache.append_decode(layer, seqs, k.cuda(), v.cuda(), q.cuda())
    b.cache.append_kv(seqs, [1] * n, k.cuda(), v.cuda())
    out_b = b.cache.decode(layer, seqs, q.cuda())
    for i, s in enumerate(seqs):
        a.orc.append(s, f64(k[:, i:i + 1]), f64(v[:, i:i + 1]))
        b.orc.append(s, f64(k[:, i:i + 1]), f64(v[:, i:i + 1]))
    torch.cuda.synchronize()
    assert torch.equal(out_a, out_b), "fused step differs from append_kv + decode"
    if check_oracle:
        for i, s in enumerate(seqs):
            kl, vl = a.orc.logical_kv(s, layer)
            ref = attend(f64(q[i:i + 1]), kl, vl, a.shape.scale)
            check_close(out_a[i:i + 1], ref, f"seq {s}")
    return out_a


@pytest.mark.parametrize("P", [16, 64])
def test_fused_step_page_crossings(P):
    shape = Shape(num_layers=1, num_q_heads=32, num_kv_heads=8, head_dim=128, page_size=P)
    a, b = _twins(shape, 512, 8, 64)
    seqs = []
    # tails: partial page, exactly full page, latent tail, one row short of a page
    for script in ([("latent", 128), ("tokens", 37)], [("tokens", 2 * P)], [("tokens", 50), ("latent", 64)],
                   [("latent", 40), ("tokens", P - 1)], [("tokens", 1)]):
        sa, sb = a.build(script), b.build(script)
        assert sa == sb
        seqs.append(sa)
    for step in range(P + 3):  # every tail crosses a page boundary at least once
        _step(a, b, seqs, 0, check_oracle=(step % 4 == 0 or step > P))
    _same_state(a, b, seqs, [0])


@pytest.mark.parametrize("hq,hkv,d", [(8, 2, 64), (32, 2, 128), (12, 4, 128)])
def test_fused_step_shapes_two_layers(hq, hkv, d):
    shape = Shape(num_layers=2, num_q_heads=hq, num_kv_heads=hkv, head_dim=d, page_size=16)
    a, b = _twins(shape, 512, 8, 80)
    seqs = []
    for n in (300, 17, 16, 1, 129):
        sa, sb = a.build([("tokens", n)]), b.build([("tokens", n)])
        seqs.append(sa)
    for step in range(20):
        _step(a, b, seqs, step % 2)
    _same_state(a, b, seqs, [0, 1])


def test_fused_step_forked_prefix_cow():
    """A fork sharing a partial last page: the first fused append on either side copies the
    page first (copy-on-write launch before the decode kernel), the other side keeps it."""
    shape = Shape(num_layers=1, num_q_heads=8, num_kv_heads=2, head_dim=128, page_size=16)
    a, b = _twins(shape, 256, 8, 32)
    src_a, src_b = a.build([("latent", 32), ("tokens", 40)]), b.build([("latent", 32), ("tokens", 40)])
    fa, fb = a.cache.seq_fork(src_a, 67), b.cache.seq_fork(src_b, 67)
    a.orc.fork(src_a, 67, fa)
    b.orc.fork(src_b, 67, fb)
    assert fa == fb
    for step in range(20):
        seqs = [fa, src_a] if step % 3 else [src_a, fa]
        _step(a, b, seqs, 0)
    _same_state(a, b, [src_a, fa], [0])


@pytest.mark.parametrize("batch", [64, 65, 300, 520])
def test_fused_step_batch_variants(batch):
    """<= 64: the 1-KB parameter variant; <= 512: the 8-KB one; 520: the two-launch path."""
    shape = Shape(num_layers=1, num_q_heads=8, num_kv_heads=2, head_dim=128, page_size=16)
    a, b = _twins(shape, 4 * batch + 64, batch, 8)
    rng = np.random.default_rng(batch)
    seqs = []
    for _ in range(batch):
        n = int(rng.integers(16, 40))  # >= 16 rows: |out| stays well below 4, where bf16 output
        # rounding alone (half an ulp = 2^-7 at [4, 8)) would exceed the 1e-2 abs bound
        seqs.append(a.build([("tokens", n)]))
        b.build([("tokens", n)])
    order = list(rng.permutation(seqs))
    l0 = a.cache.launch_count()
    _step(a, b, order, 0, check_oracle=False)
    launches = a.cache.launch_count() - l0
    if batch <= 512:
        assert launches <= 2, launches  # decode (+ combine); no scatter launch
    for _ in range(3):
        _step(a, b, order, 0, check_oracle=True)
    _same_state(a, b, seqs[:8], [0])


def test_fused_then_plain_decode_and_prefill():
    """After fused steps the device table (written back by the kernel) serves plain calls."""
    shape = Shape(num_layers=1, num_q_heads=32, num_kv_heads=8, head_dim=128, page_size=16)
    a, b = _twins(shape, 512, 4, 64)
    seqs = [a.build([("latent", 128), ("tokens", 100)]), a.build([("tokens", 15)])]
    for s in ([("latent", 128), ("tokens", 100)], [("tokens", 15)]):
        b.build(s)
    for _ in range(5):
        _step(a, b, seqs, 0)
    q = a.queries(2)
    qp = a.queries(9)
    out = a.cache.decode(0, seqs, q.cuda())
    pre = a.cache.prefill(0, seqs[:1], [9], qp.cuda())
    torch.cuda.synchronize()
    for i, s in enumerate(seqs):
        kl, vl = a.orc.logical_kv(s, 0)
        check_close(out[i:i + 1], attend(f64(q[i:i + 1]), kl, vl, shape.scale), f"decode {s}")
    kl, vl = a.orc.logical_kv(seqs[0], 0)
    check_close(pre, attend(f64(qp), kl, vl, shape.scale), "prefill")
    # a plain append after fused ones continues on the same page
    a.tokens([seqs[1]], [3])
    b.tokens([seqs[1]], [3])
    _same_state(a, b, seqs, [0])


def test_fused_step_fp8_pages_two_launch_path():
    shape = Shape(num_layers=1, num_q_heads=32, num_kv_heads=8, head_dim=128, page_size=16)
    p = Pair(shape, 128, 4, 64, token_fp8=True, num_token_pages=256)
    seqs = [p.build([("latent", 128), ("tokens", 70)]), p.build([("tokens", 31)])]
    for _ in range(4):
        k, v = p.draw.tokens(shape, 2)
        q = p.draw.queries(shape, 2)
        out = p.cache.append_decode(0, seqs, k.cuda(), v.cuda(), q.cuda())
        for i, s in enumerate(seqs):
            p.orc.append(s, f64(k[:, i:i + 1]), f64(v[:, i:i + 1]))
        torch.cuda.synchronize()
        for i, s in enumerate(seqs):
            kl, vl = p.orc.logical_kv(s, 0)
            check_close(out[i:i + 1], attend(f64(q[i:i + 1]), kl, vl, shape.scale), f"fp8 seq {s}")


def test_fused_step_errors_leave_cache_unchanged():
    shape = Shape(num_layers=1, num_q_heads=8, num_kv_heads=2, head_dim=64, page_size=16)
    p = Pair(shape, 3, 4, 4)
    s0 = p.build([("tokens", 16)])   # one full page: the next row needs a new page
    s1 = p.build([("tokens", 3)])
    k, v = p.draw.tokens(shape, 2)
    q = p.draw.queries(shape, 2)

    def expect(err, *args):
        before = (p.cache.stats(), p.cache.seq_info(s0), p.cache.seq_info(s1))
        with pytest.raises(HPAError) as e:
            p.cache.append_decode(*args)
        assert e.value.name == err
        assert (p.cache.stats(), p.cache.seq_info(s0), p.cache.seq_info(s1)) == before

    expect("HPA_ERR_INVALID_ARG", 3, [s0, s1], k.cuda(), v.cuda(), q.cuda())   # bad layer
    expect("HPA_ERR_UNKNOWN_SEQ", 0, [s0, 3], k.cuda(), v.cuda(), q.cuda())    # unknown seq
    expect("HPA_ERR_INVALID_ARG", 0, [s0, s0], k.cuda(), v.cuda(), q.cuda())   # listed twice
    p.build([("tokens", 16)])        # the last free page
    expect("HPA_ERR_OUT_OF_PAGES", 0, [s1, s0], k.cuda(), v.cuda(), q.cuda())
    # s1 alone still fits on its partial page
    out = p.cache.append_decode(0, [s1], k[:, :1].contiguous().cuda(), v[:, :1].contiguous().cuda(),
                                q[:1].cuda())
    p.orc.append(s1, f64(k[:, :1]), f64(v[:, :1]))
    torch.cuda.synchronize()
    kl, vl = p.orc.logical_kv(s1, 0)
    check_close(out, attend(f64(q[:1]), kl, vl, shape.scale), "after errors")


def test_decode_run_to_run_deterministic():
    """Units are fetched dynamically (ticket counter), so which consumer warp sees which chunk
    varies between launches; the merge goes by chunk group within the unit, so the output must
    be bitwise identical across repeated launches (and the fused step equal to the two calls)."""
    shape = Shape(num_layers=1, num_q_heads=32, num_kv_heads=8, head_dim=128, page_size=16)
    p = Pair(shape, 2048, 24, 128)
    rng = np.random.default_rng(5)
    seqs = [p.build([("latent", 128), ("tokens", int(rng.integers(200, 1800)))]) for _ in range(24)]
    q = p.queries(24).cuda()
    ref = p.cache.decode(0, seqs, q).clone()
    for r in range(30):
        order = seqs if r % 2 == 0 else seqs[::-1]
        out = p.cache.decode(0, order, q if r % 2 == 0 else q.flip(0))
        got = out if r % 2 == 0 else out.flip(0)
        assert torch.equal(got, ref), r
