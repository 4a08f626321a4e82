"""NEXT-4c: fp8 token pages with bf16 latent pages, through the C ABI.

Scheme = DESIGN.md reading A20 (per (layer, row, kv-head) e4m3 codes + fp32 scale for K
and for V). The oracle quantizes the same bf16 inputs with its own quantizer
(oracle.quantize_rows_e4m3, pinned in test_oracle_pins.py) and attends over the
dequantized rows in fp64. Checks: the stored codes and scales are bit-exact; decode over
mixed latent (bf16) + token (fp8) pages is within the north-star tolerance; export and
compression dequantize exactly as the oracle; prefill dequantizes the batch's token pages
into temporary bf16 pages and leaves the cache unchanged."""
import numpy as np
import pytest
import torch

from oracle import attend
from tests.hpa_testutil import Pair, check_close, f64
from workloads import Shape, qwen3_8b_shape

pytestmark = pytest.mark.gpu


def _shape(hq, hkv, d, P, L=1):
    return Shape(num_layers=L, num_q_heads=hq, num_kv_heads=hkv, head_dim=d, page_size=P)


def _fp8_pair(shape, pages=512, tpages=512, seqs=8, per_seq=96, seed=77):
    return Pair(shape, pages, seqs, per_seq, seed=seed, token_fp8=True, num_token_pages=tpages)


def _token_pages(pair, s):
    """(page, valid) of every TOKEN entry of seq s in table order."""
    pages, pos0, meta = pair.cache.export_table(s)
    return [(int(p), int(m) & 0x7FFF) for p, m in zip(pages, meta) if not (int(m) & 0x8000)]


@pytest.mark.parametrize("d,P", [(128, 16), (64, 32), (128, 64)])
def test_fp8_token_pool_bit_exact(d, P):
    shape = _shape(4, 2, d, P, L=2)
    pr = _fp8_pair(shape)
    s = pr.build([("latent", 2 * P), ("tokens", 3 * P + 5), ("latent", P + 3), ("tokens", 2 * P - 1)])
    pr.tokens([s], [7])                                   # extends the trailing token segment
    torch.cuda.synchronize()
    k8, v8, ks, vs, _ = pr.cache.token_pool()
    k8, v8, ks, vs = k8.cpu().numpy(), v8.cpu().numpy(), ks.cpu().numpy(), vs.cpu().numpy()
    for layer in range(shape.num_layers):
        segs = pr.orc.token_codes(s, layer)
        exp_k = np.concatenate([g[0] for g in segs])       # [rows][H][d]
        exp_ks = np.concatenate([g[1] for g in segs])
        exp_v = np.concatenate([g[2] for g in segs])
        exp_vs = np.concatenate([g[3] for g in segs])
        # walk the token entries; segment boundaries restart on a fresh page
        rows_k, rows_ks, rows_v, rows_vs = [], [], [], []
        for page, valid in _token_pages(pr, s):
            rows_k.append(k8[layer, page, :, :valid].transpose(1, 0, 2))
            rows_ks.append(ks[layer, page, :, :valid].T)
            rows_v.append(v8[layer, page, :, :valid].transpose(1, 0, 2))
            rows_vs.append(vs[layer, page, :, :valid].T)
        assert np.array_equal(np.concatenate(rows_k), exp_k)
        assert np.array_equal(np.concatenate(rows_v), exp_v)
        assert np.array_equal(np.concatenate(rows_ks), exp_ks)
        assert np.array_equal(np.concatenate(rows_vs), exp_vs)


@pytest.mark.parametrize("hq,hkv,d,P,splits", [(32, 8, 128, 16, 0), (32, 8, 128, 16, 3), (8, 1, 128, 64, 0),
                                                (16, 1, 64, 32, 2), (4, 4, 128, 256, 0)])
def test_fp8_decode_parity_mixed_pages(hq, hkv, d, P, splits):
    shape = _shape(hq, hkv, d, P, L=2)
    pr = _fp8_pair(shape, pages=2048, tpages=2048, seqs=6, per_seq=160)
    scripts = [[("latent", 128), ("tokens", 700)], [("tokens", 333)], [("latent", 37), ("tokens", 1), ("latent", 128)],
               [("latent", 256), ("tokens", 1100)], [("tokens", 17), ("latent", 64), ("tokens", 90)]]
    seqs = [pr.build(sc) for sc in scripts]
    if splits:
        pr.cache.set_decode_splits(splits)
    q = pr.queries(len(seqs))
    for layer in (0, 1):
        out = pr.cache.decode(layer, seqs, q.cuda())
        torch.cuda.synchronize()
        ref = np.stack([attend(f64(q[i:i + 1]), *pr.orc.logical_kv(s, layer), shape.scale)[0]
                        for i, s in enumerate(seqs)])
        check_close(out, ref, f"fp8 decode hq={hq} hkv={hkv} d={d} P={P} S={splits} layer={layer}")


def test_fp8_latent_only_and_token_only_sequences_and_errors():
    from paper_2605_09100_b200 import HPAError
    shape = _shape(8, 2, 128, 16)
    pr = _fp8_pair(shape)
    a = pr.build([("latent", 100)])                       # bf16 pages only
    b = pr.build([("tokens", 250)])                       # fp8 pages only
    q = pr.queries(2)
    out = pr.cache.decode(0, [a, b], q.cuda())
    ref = np.stack([attend(f64(q[i:i + 1]), *pr.orc.logical_kv(s, 0), shape.scale)[0] for i, s in enumerate([a, b])])
    check_close(out, ref, "fp8 latent-only / token-only")
    with pytest.raises(HPAError):
        pr.cache.prefill(0, [b], [251], pr.queries(251).cuda())   # q_len > seq_len
    out2 = pr.cache.prefill(0, [a], [10], pr.queries(10).cuda())   # latent-only rows
    assert torch.isfinite(out2.float()).all()


@pytest.mark.parametrize("hq,hkv,d,P", [(32, 8, 128, 16), (8, 1, 128, 64), (16, 2, 64, 32)])
def test_fp8_prefill_parity_and_cache_unchanged(hq, hkv, d, P):
    """Prefill over fp8 token pages (dequantized into temporary bf16 pages for the call):
    parity with the oracle over the dequantized rows; afterwards the table, the token pool,
    the free-page counts and decode are unchanged."""
    shape = _shape(hq, hkv, d, P, L=2)
    pr = _fp8_pair(shape, pages=1024, tpages=1024, seqs=4, per_seq=200)
    seqs = [pr.build([("latent", 128), ("tokens", 500)]), pr.build([("tokens", 300), ("latent", 64), ("tokens", 77)])]
    qd = pr.queries(1)
    before = pr.cache.decode(1, [seqs[0]], qd.cuda()).clone()
    tables = [pr.cache.export_table(s) for s in seqs]
    free0, tfree0 = pr.cache.stats()[0], pr.cache.token_pool()[4]
    k8a = pr.cache.token_pool()[0].clone()
    q_lens = [200, 77]
    q = pr.queries(sum(q_lens))
    for layer in (0, 1):
        out = pr.cache.prefill(layer, seqs, q_lens, q.cuda())
        torch.cuda.synchronize()
        off = 0
        for s, n in zip(seqs, q_lens):
            k, v = pr.orc.logical_kv(s, layer, fp8_staged=True)
            lb = k.shape[1]
            ref = np.stack([attend(f64(q[off + t:off + t + 1]), k[:, :lb - n + t + 1], v[:, :lb - n + t + 1],
                                   shape.scale)[0] for t in range(n)])
            check_close(out[off:off + n], ref, f"fp8 prefill layer {layer} seq {s}")
            off += n
    assert pr.cache.stats()[0] == free0 and pr.cache.token_pool()[4] == tfree0
    for s, t in zip(seqs, tables):
        t2 = pr.cache.export_table(s)
        assert all(np.array_equal(x, y) for x, y in zip(t, t2))
    assert torch.equal(pr.cache.token_pool()[0], k8a)
    after = pr.cache.decode(1, [seqs[0]], qd.cuda())
    assert torch.equal(before, after)


def test_fp8_export_and_compress_dequantize_like_the_oracle():
    shape = _shape(8, 2, 128, 16, L=2)
    pr = _fp8_pair(shape)
    s = pr.build([("latent", 64), ("tokens", 4096 // 16 + 128 + 40)])
    for layer in range(2):
        k, v = pr.cache.export_logical_kv(layer, s)
        ek, ev = pr.orc.logical_kv(s, layer)
        # latent rows are exact bf16; fp8 rows export as bf16(code * scale) -> within bf16 rounding
        assert np.array_equal(f64(k)[:, :64], ek[:, :64])
        np.testing.assert_allclose(f64(k)[:, 64:], ek[:, 64:], rtol=2 ** -8, atol=0)
        np.testing.assert_allclose(f64(v)[:, 64:], ev[:, 64:], rtol=2 ** -8, atol=0)
        # ... and bit-exactly the staged rows of reading A20 (bf16(fp32(code) * scale))
        sk, sv = pr.orc.logical_kv(s, layer, fp8_staged=True)
        assert np.array_equal(f64(k), sk) and np.array_equal(f64(v), sv)
    free0 = pr.cache.token_pool()[4]
    got = pr.cache.compress(s, 4096 // 16, 128)          # document rows -> 128 bf16 latent rows
    exp = pr.orc.compress(s, 4096 // 16, 128)
    assert got == exp
    assert pr.cache.token_pool()[4] > free0               # token pages were returned to the fp8 pool
    for layer in range(2):
        k, v = pr.cache.export_logical_kv(layer, s)
        ek, ev = pr.orc.logical_kv(s, layer)
        assert k.shape[1] == ek.shape[1] == 64 + 40 + 128
        # the compressed set is bit-exact bf16(fp32(code) * scale) (A20), after the 40 kept tokens
        assert np.array_equal(f64(k)[:, 64 + 40:], ek[:, 64 + 40:])
        assert np.array_equal(f64(v)[:, 64 + 40:], ev[:, 64 + 40:])
    q = pr.queries(1)
    out = pr.cache.decode(0, [s], q.cuda())
    check_close(out, attend(f64(q), *pr.orc.logical_kv(s, 0), shape.scale), "fp8 decode after compress")


def test_fp8_full_size_configs1_sampled():
    from tests.test_gpu_fullsize import _build
    from oracle import OracleCache
    from paper_2605_09100_b200 import Cache
    from workloads import Draw
    shape = qwen3_8b_shape(16)
    B, sampled = 64, [0, 21, 63]
    cache = Cache(1, 32, 8, 128, 16, B * 66, B, 330, 0, 99, "fp8", B * 260)
    orc = OracleCache(1, 32, 8, 128, 16, token_fp8=True)
    seqs, _ = _build(cache, orc, shape, B, sampled, 8, 4096, 2025)
    q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
    qs = Draw(9).queries(shape, len(sampled))
    for i, s in enumerate(sampled):
        q[s] = qs[i].cuda()
    out = cache.decode(0, seqs, q)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    ref = np.stack([attend(f64(qs[i:i + 1]), *orc.logical_kv(seqs[s], 0), shape.scale)[0]
                    for i, s in enumerate(sampled)])
    check_close(out[sampled], ref, "configs[1] fp8 token pages, sampled")
    cache.close()


def test_fp8_page256_and_partial_pages():
    shape = _shape(8, 2, 128, 256)
    pr = _fp8_pair(shape, pages=64, tpages=64, seqs=3, per_seq=16)
    s1 = pr.build([("tokens", 300), ("latent", 40), ("tokens", 700)])
    s2 = pr.build([("latent", 300), ("tokens", 3)])
    q = pr.queries(2)
    out = pr.cache.decode(0, [s1, s2], q.cuda())
    ref = np.stack([attend(f64(q[i:i + 1]), *pr.orc.logical_kv(s, 0), shape.scale)[0] for i, s in enumerate([s1, s2])])
    check_close(out, ref, "fp8 P=256")
    qp = pr.queries(64)
    outp = pr.cache.prefill(0, [s1], [64], qp.cuda())
    k, v = pr.orc.logical_kv(s1, 0, fp8_staged=True)
    lb = k.shape[1]
    refp = np.stack([attend(f64(qp[t:t + 1]), k[:, :lb - 64 + t + 1], v[:, :lb - 64 + t + 1], shape.scale)[0]
                     for t in range(64)])
    check_close(outp, refp, "fp8 P=256 prefill")


def test_fp8_prefill_config2_b4_full_size_sampled():
    """configs[2] at B_p = 4 with fp8 token pages, as bench.py's next.fp8_prefill times it: the
    batch's token pages dequantized into temporary bf16 pages, then the 1024-CTA cluster
    launch. Two CPU-drawn requests mirrored in the oracle (prefill attends over the staged rows,
    reading A20); 24 sampled query rows each, all 32 heads; the cache (fp8 codes, table, free
    pages) unchanged afterwards is covered by test_fp8_prefill_parity_and_cache_unchanged."""
    from tests.test_gpu_fullsize import _build
    from oracle import OracleCache
    from paper_2605_09100_b200 import Cache
    from workloads import Draw
    shape = qwen3_8b_shape(16)
    C, prior, B, sampled = 2048, 16384, 4, [0, 2]
    tok_pages = (prior + C) // 16
    cache = Cache(1, 32, 8, 128, 16, B * (64 + tok_pages) + 64, B, 64 + tok_pages, 0, 99, "fp8", B * tok_pages + 64)
    orc = OracleCache(1, 32, 8, 128, 16, token_fp8=True)
    seqs, _ = _build(cache, orc, shape, B, sampled, 8, prior + C, 79)
    q = torch.randn((B * C, 32, 128), device="cuda").to(torch.bfloat16)
    qs = {s: Draw(30 + s).queries(shape, C) for s in sampled}
    for s in sampled:
        q[s * C:(s + 1) * C] = qs[s].cuda()
    out = cache.prefill(0, seqs, [C] * B, q)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    for s in sampled:
        k, v = orc.logical_kv(seqs[s], 0, fp8_staged=True)
        lb = k.shape[1]
        rows = sorted(set([0, 127, 128, 2047] + list(np.random.default_rng(s).integers(0, C, 20))))
        ref = np.stack([attend(f64(qs[s][t:t + 1]), k[:, :lb - C + t + 1], v[:, :lb - C + t + 1], shape.scale)[0]
                        for t in rows])
        check_close(out[s * C:(s + 1) * C][rows], ref, f"configs[2] B=4 fp8 prefill request {s} sampled rows")
    cache.close()
