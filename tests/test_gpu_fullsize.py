"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times, on sampled outputs the oracle computes one by one.

configs[1]: B=64 decode, 8 x 128 latent rows + 4096 token rows (Lb = 5120),
            split planner as in the bench; 4 sampled requests, all 32 heads.
configs[2]: chunked prefill C=2048 over 1024 latent + 16384 cached token rows;
            48 sampled query rows (first/last/ragged positions), all 32 heads.
configs[3]: B=256 LMAG step (batched latent replacement + append + decode);
            4 sampled requests.
configs[1] ragged variant: reasoning rows ~ U[1K, 8K] per request.
configs[4]: per-GPU shard of the 8-GPU sweep (B=512/8=64 requests) at ctx=64K
            with latent ratios 0.1 and 0.9; 2 sampled requests.
NEXT rows as bench.py times them: the GRC span prefill (configs[2] B=1, 8192 masked rows)
the B=64 compress batch (4096-row documents -> 128-row latent sets) and the B=256
host-staged install; fp8 prefill at
B=4 is in test_gpu_fp8.py, the full-size prefix cascade and shared sets in test_gpu_cascade.py.
Sampled requests are drawn on the CPU (workloads.Draw); the rest of the batch
is filled with GPU-drawn data of the same distribution (it only shapes the
launch; its outputs are checked for finiteness)."""
import numpy as np
import pytest
import torch

from oracle import OracleCache, attend
from tests.hpa_testutil import check_close, f64
from workloads import LATENT_ROWS, Draw, qwen3_8b_shape

pytestmark = pytest.mark.gpu


def _build(cache, orc, shape, n_req, sampled, docs, tokens, seed):
    """Builds n_req requests; the `sampled` ones with CPU draws mirrored in the oracle.
    `tokens` is one row count for all requests or a list (ragged)."""
    tok = [tokens] * n_req if isinstance(tokens, int) else list(tokens)
    g = torch.Generator(device="cuda").manual_seed(seed)
    seqs = [cache.seq_create() for _ in range(n_req)]
    draws = {}
    for s in sampled:
        orc.create_seq(seqs[s])
        draws[s] = Draw(seed + 100 + s)
    for _ in range(docs):
        kvs = []
        for s in range(n_req):
            if s in draws:
                kv = draws[s].latent(shape, LATENT_ROWS)
                orc.install(seqs[s], -1, f64(kv))
                kvs.append(kv.cuda())
            else:
                kvs.append(torch.randn((1, 2, LATENT_ROWS, 8, 128), generator=g, device="cuda").to(torch.bfloat16))
        cache.latent_install_batch(seqs, [-1] * n_req, kvs)
    ks, vs = [], []
    for s in range(n_req):
        if s in draws:
            k, v = draws[s].tokens(shape, tok[s])
            orc.append(seqs[s], f64(k), f64(v))
            ks.append(k.cuda())
            vs.append(v.cuda())
        else:
            ks.append(torch.randn((1, tok[s], 8, 128), generator=g, device="cuda").to(torch.bfloat16))
            vs.append(torch.randn((1, tok[s], 8, 128), generator=g, device="cuda").to(torch.bfloat16))
    cache.append_kv(seqs, tok, torch.cat(ks, 1), torch.cat(vs, 1))
    return seqs, draws


def test_decode_config1_full_size_sampled():
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    B, sampled = 64, [0, 17, 42, 63]
    cache = Cache(1, 32, 8, 128, 16, B * 330, B, 330, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    seqs, draws = _build(cache, orc, shape, B, sampled, 8, 4096, 2024)
    q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
    qs = Draw(7).queries(shape, len(sampled))
    for i, s in enumerate(sampled):
        q[s] = qs[i].cuda()
    out = cache.decode(0, seqs, q)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    ref = np.stack([attend(f64(qs[i:i + 1]), *orc.logical_kv(seqs[s], 0), shape.scale)[0]
                    for i, s in enumerate(sampled)])
    check_close(out[sampled], ref, "configs[1] decode sampled")
    cache.close()


def test_prefill_config2_full_size_sampled():
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    C, prior = 2048, 16384
    cache = Cache(1, 32, 8, 128, 16, 1300, 1, 1300, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    seqs, draws = _build(cache, orc, shape, 1, [0], 8, prior + C, 77)
    q = Draw(8).queries(shape, C)
    out = cache.prefill(0, seqs, [C], q.cuda())
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    k, v = orc.logical_kv(seqs[0], 0)
    lb = k.shape[1]
    rows = sorted(set([0, 1, 127, 128, 255, 1000, 1023, 1024, 2046, 2047] +
                      list(np.random.default_rng(3).integers(0, C, 38))))
    ref = np.stack([attend(f64(q[t:t + 1]), k[:, :lb - C + t + 1], v[:, :lb - C + t + 1], shape.scale)[0]
                    for t in rows])
    check_close(out[rows], ref, "configs[2] prefill sampled rows")
    # the bench's B=1 launch: stream-K shares on the persistent kernel (256 units, 1.73 waves);
    # the one-CTA-per-item plan (-3) must agree everywhere up to fp32 summation order
    info = cache.prefill_plan_info()
    assert info["split_units"] > 0 and info["splits"] <= 15 and info["cluster"] == 1, info
    cache.set_prefill_ctas(-3)
    out2 = cache.prefill(0, seqs, [C], q.cuda())
    torch.cuda.synchronize()
    check_close(out2[rows], ref, "configs[2] prefill sampled rows, one CTA per item")
    d = (out.float() - out2.float()).abs().max().item()
    assert d <= 2.0 ** -7 * (1.0 + out2.float().abs().max().item()), d
    cache.close()


def test_lmag_config3_full_size_sampled():
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    B, sampled = 256, [0, 100, 200, 255]
    cache = Cache(1, 32, 8, 128, 16, B * 330, B, 330, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    seqs, draws = _build(cache, orc, shape, B, sampled, 8, 4095, 555)
    g = torch.Generator(device="cuda").manual_seed(9)
    for step in range(2):
        sid = step % 8
        kvs = []
        for s in range(B):
            if s in draws:
                kv = draws[s].latent(shape, LATENT_ROWS)
                orc.install(seqs[s], sid, f64(kv))
                kvs.append(kv.cuda())
            else:
                kvs.append(torch.randn((1, 2, LATENT_ROWS, 8, 128), generator=g, device="cuda").to(torch.bfloat16))
        cache.latent_install_batch(seqs, [sid] * B, kvs)
        step_draw = Draw(900 + step)                   # CPU draws for everything the oracle sees
        kn, vn = step_draw.tokens(shape, B)            # [1][B][8][128]: one new row per request
        cache.append_kv(seqs, [1] * B, kn.cuda(), vn.cuda())
        for s in sampled:
            orc.append(seqs[s], f64(kn[:, s:s + 1]), f64(vn[:, s:s + 1]))
        q = step_draw.queries(shape, B)
        out = cache.decode(0, seqs, q.cuda())
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all()
        ref = np.stack([attend(f64(q[s:s + 1]), *orc.logical_kv(seqs[s], 0), shape.scale)[0] for s in sampled])
        check_close(out[sampled], ref, f"configs[3] LMAG step {step}")
    cache.close()


def _decode_sampled(cache, orc, shape, seqs, sampled, what, qseed=7):
    B = len(seqs)
    q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
    qs = Draw(qseed).queries(shape, len(sampled))
    for i, s in enumerate(sampled):
        q[s] = qs[i].cuda()
    out = cache.decode(0, seqs, q)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    ref = np.stack([attend(f64(qs[i:i + 1]), *orc.logical_kv(seqs[s], 0), shape.scale)[0]
                    for i, s in enumerate(sampled)])
    check_close(out[sampled], ref, what)


def test_decode_config1_ragged_sampled():
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    B, sampled = 64, [0, 5, 33, 63]
    g = torch.Generator().manual_seed(1234 + 7)
    toks = [int(torch.randint(1024, 8193, (1,), generator=g).item()) for _ in range(B)]
    toks[5], toks[33] = 1024, 8192                     # both ends of the range among the sampled
    pages = 64 + 8192 // 16 + 2
    cache = Cache(1, 32, 8, 128, 16, B * pages, B, pages, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    seqs, _ = _build(cache, orc, shape, B, sampled, 8, toks, 4242)
    _decode_sampled(cache, orc, shape, seqs, sampled, "configs[1] ragged decode sampled")
    cache.close()


@pytest.mark.parametrize("ratio", [0.1, 0.9])
def test_decode_config4_sweep_shard_64k_sampled(ratio):
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    ctx, B, sampled = 65536, 64, [0, 63]
    sets = int(ratio * ctx) // LATENT_ROWS
    tok = ctx - sets * LATENT_ROWS
    pages = sets * (LATENT_ROWS // 16) + tok // 16 + 1
    cache = Cache(1, 32, 8, 128, 16, B * pages, B, pages, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    seqs, _ = _build(cache, orc, shape, B, sampled, sets, tok, 31)
    _decode_sampled(cache, orc, shape, seqs, sampled, f"configs[4] shard ctx=64K r={ratio}")
    cache.close()


def test_prefill_config2_b4_full_size_sampled_clusters():
    """configs[2] at B_p = 4 in the launch configuration bench.py times:
    1024 CTAs as 2-CTA TMA-multicast clusters with no split. Two of the four requests are
    CPU-drawn and mirrored in the oracle; 24 sampled query rows each, all 32 heads."""
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    C, prior, B, sampled = 2048, 16384, 4, [1, 3]
    pages = 64 + (prior + C) // 16
    cache = Cache(1, 32, 8, 128, 16, B * pages, B, pages, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    seqs, draws = _build(cache, orc, shape, B, sampled, 8, prior + C, 78)
    q = torch.randn((B * C, 32, 128), device="cuda").to(torch.bfloat16)
    qs = {s: Draw(20 + s).queries(shape, C) for s in sampled}
    for s in sampled:
        q[s * C:(s + 1) * C] = qs[s].cuda()
    out = cache.prefill(0, seqs, [C] * B, q)
    torch.cuda.synchronize()
    info = cache.prefill_plan_info()
    assert info["cluster"] == 2 and info["split_units"] == 0 and info["ctas"] == B * 32 * C // 256, info
    assert torch.isfinite(out.float()).all()
    for s in sampled:
        k, v = orc.logical_kv(seqs[s], 0)
        lb = k.shape[1]
        rows = sorted(set([0, 127, 128, 1023, 1024, 2047] + list(np.random.default_rng(s).integers(0, C, 18))))
        ref = np.stack([attend(f64(qs[s][t:t + 1]), k[:, :lb - C + t + 1], v[:, :lb - C + t + 1], shape.scale)[0]
                        for t in rows])
        check_close(out[s * C:(s + 1) * C][rows], ref, f"configs[2] B=4 prefill request {s} sampled rows")
    cache.close()


def test_span_prefill_config2_full_size_sampled():
    """bench.py's next.span_prefill at full size: configs[2] B = 1 (the default stream-K plan on
    the persistent kernel) with the GRC mask-out span over the first 8192 token rows (all C
    queries are segment-3 rows); 12 sampled query rows, all 32 heads, against oracle.attend_span."""
    from oracle import attend_span
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    C, prior, n1 = 2048, 16384, 8192
    cache = Cache(1, 32, 8, 128, 16, 1300, 1, 1300, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    seqs, _ = _build(cache, orc, shape, 1, [0], 8, prior + C, 46)
    q = Draw(47).queries(shape, C)
    span = (1024, 1024 + n1, 1024 + prior)
    out = cache.prefill_span(0, seqs, [C], [span], q.cuda())
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    k, v = orc.logical_kv(seqs[0], 0)
    lb = k.shape[1]
    rows = sorted(set([0, 127, 1024, 2047] + list(np.random.default_rng(5).integers(0, C, 8))))
    ref = np.stack([attend_span(f64(q[t:t + 1]), k[:, :lb - C + t + 1], v[:, :lb - C + t + 1], shape.scale,
                                *span)[0] for t in rows])
    check_close(out[rows], ref, "configs[2] span prefill sampled rows")
    cache.close()


def test_compress_batch_full_size_sampled():
    """bench.py's next.compress at full size: B = 64 requests of 8 latent sets + a 4096-row
    document + 128 meta-latent rows, one hpa_seq_compress_batch call turning the last 128 rows
    of each into a latent set and dropping the document. Two requests mirrored in the oracle:
    their logical K/V after the call is bit-exact, their decode matches; every request freed
    its document pages (4096 / 16 - its kept partial page) and decodes finitely."""
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    B, n_doc, m, sampled = 64, 4096, LATENT_ROWS, [3, 60]
    pages = 64 + (n_doc + m) // 16 + 2
    cache = Cache(1, 32, 8, 128, 16, B * pages + 64, B, pages, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    seqs, _ = _build(cache, orc, shape, B, sampled, 8, n_doc + m, 80)
    free0 = cache.stats()[0]
    sets = cache.compress_batch(seqs, [n_doc] * B, [m] * B)
    torch.cuda.synchronize()
    for s in sampled:
        assert sets[s] == orc.compress(seqs[s], n_doc, m)
        k1, v1 = orc.logical_kv(seqs[s], 0)
        k2, v2 = cache.export_logical_kv(0, seqs[s])
        assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2)), s
    assert cache.stats()[0] - free0 == B * (n_doc // 16), (cache.stats()[0], free0)
    q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
    qs = Draw(81).queries(shape, len(sampled))
    for i, s in enumerate(sampled):
        q[s] = qs[i].cuda()
    out = cache.decode(0, seqs, q)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    ref = np.stack([attend(f64(qs[i:i + 1]), *orc.logical_kv(seqs[s], 0), shape.scale)[0]
                    for i, s in enumerate(sampled)])
    check_close(out[sampled], ref, "decode after full-size compress batch")
    cache.close()


def test_host_staged_install_full_size_sampled():
    """bench.py's next.host_staged_install at full size: B = 256 configs[1]-shaped requests, one
    128-row latent set of each replaced from a pinned host payload in one
    hpa_latent_set_install_host call (copy stream + scatter). Two requests mirrored in the
    oracle: bit-exact logical views and decode parity afterwards."""
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    B, sampled, tokens = 256, [7, 200], 4096
    pages = 64 + tokens // 16 + 2
    cache = Cache(1, 32, 8, 128, 16, B * pages + 64, B, pages, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    seqs, _ = _build(cache, orc, shape, B, sampled, 8, tokens, 90)
    d = Draw(91)
    kv = torch.randn((B, 1, 2, LATENT_ROWS, 8, 128)).to(torch.bfloat16)
    for s in sampled:
        kv[s] = d.latent(shape, LATENT_ROWS)
    kv = kv.pin_memory()
    got = cache.latent_install_host(seqs, [3] * B, kv)
    torch.cuda.synchronize()
    for s in sampled:
        assert got[s] == orc.install(seqs[s], 3, f64(kv[s]))
        k1, v1 = orc.logical_kv(seqs[s], 0)
        k2, v2 = cache.export_logical_kv(0, seqs[s])
        assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2)), s
    q = torch.randn((B, 32, 128), device="cuda").to(torch.bfloat16)
    qs = Draw(92).queries(shape, len(sampled))
    for i, s in enumerate(sampled):
        q[s] = qs[i].cuda()
    out = cache.decode(0, seqs, q)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    ref = np.stack([attend(f64(qs[i:i + 1]), *orc.logical_kv(seqs[s], 0), shape.scale)[0]
                    for i, s in enumerate(sampled)])
    check_close(out[sampled], ref, "decode after full-size host-staged install")
    cache.close()
