"""GPU parity: CUDA path (through the C ABI) vs the fp64 oracle, element by element.

Tolerance (BASELINE.json north_star): max abs <= 1e-2, relative L2 <= 5e-3.
Gathers / tables: bit-exact.
"""
import hashlib

import numpy as np
import pytest
import torch

from oracle import attend, expected_table, gather_physical
from oracle.hpa_oracle import META_LATENT_BIT
from tests.hpa_testutil import Pair, check_close, f64
from workloads import Draw, Shape, tiny_decode

pytestmark = pytest.mark.gpu


def oracle_decode(pair, seqs, q, layer=0):
    out = []
    for i, s in enumerate(seqs):
        k, v = pair.orc.logical_kv(s, layer)
        out.append(attend(f64(q[i:i + 1]), k, v, pair.shape.scale)[0])
    return np.stack(out)


def oracle_prefill(pair, seqs, q_lens, q, layer=0):
    out, off = [], 0
    for s, n in zip(seqs, q_lens):
        k, v = pair.orc.logical_kv(s, layer)
        out.append(attend(f64(q[off:off + n]), k, v, pair.shape.scale))
        off += n
    return np.concatenate(out)


# ----------------------------------------------------------------------------- tiny config
@pytest.mark.parametrize("variant", ["a", "b", "c"])
def test_tiny_config(variant):
    """BASELINE.json configs[0]: 1 latent page + 3 token pages (b: m=8, c: prefill 16)."""
    w = tiny_decode(variant)
    p = Pair(w.shape, num_pages=8, max_seqs=1, max_pages_per_seq=8)
    s = p.build(w.seqs[0].segments)
    q = p.queries(w.seqs[0].q_len)
    if w.mode == "decode":
        got = p.cache.decode(0, [s], q.cuda())
        ref = oracle_decode(p, [s], q)
    else:
        got = p.cache.prefill(0, [s], [w.seqs[0].q_len], q.cuda())
        ref = oracle_prefill(p, [s], [w.seqs[0].q_len], q)
    torch.cuda.synchronize()
    check_close(got, ref, w.name)


# ----------------------------------------------------------------------------- gathers
def test_gather_and_table_bit_exact():
    """Route 1 (oracle model) == hpa_export_logical_kv == route 2 (pool dump +
    exported table), bitwise; table == expected_table (kinds, valid rows, pos0)."""
    shape = Shape(2, 4, 2, 128, 16)
    p = Pair(shape, num_pages=256, max_seqs=4, max_pages_per_seq=64)
    scripts = [[("latent", 128), ("latent", 8), ("tokens", 37), ("latent", 20), ("tokens", 5)],
               [("tokens", 1)], [("latent", 128), ("tokens", 300)]]
    seqs = [p.build(sc) for sc in scripts]
    p.tokens(seqs, [3, 17, 16])  # cross-boundary / exact-multiple appends in one call
    torch.cuda.synchronize()
    kpool, vpool = (f64(t) for t in p.cache.pools())
    for s in seqs:
        pages, pos0, meta = p.cache.export_table(s)
        exp = p.orc.expected_table(s)
        assert [(("latent" if m & META_LATENT_BIT else "token"), int(m & 0x7fff), int(p0))
                for m, p0 in zip(meta, pos0)] == exp
        assert p.cache.seq_info(s)[0] == p.orc.seq_len(s)
        for layer in range(2):
            k1, v1 = p.orc.logical_kv(s, layer)
            k2, v2 = p.cache.export_logical_kv(layer, s)
            assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2))
            k3, v3 = gather_physical(kpool, vpool, pages.tolist(), meta.tolist(), layer)
            assert np.array_equal(k1, k3) and np.array_equal(v1, v3)


# ----------------------------------------------------------------------------- decode grid
DECODE_GRID = [
    # (Hq, Hkv, d, P)
    (32, 8, 128, 16),
    (32, 8, 128, 64),
    (8, 1, 128, 16),    # G = 8
    (16, 1, 64, 32),    # G = 16, d = 64
    (2, 1, 64, 16),     # tiny shape
    (4, 4, 128, 256),   # G = 1, P = 256
]


@pytest.mark.parametrize("hq,hkv,d,P", DECODE_GRID)
@pytest.mark.parametrize("splits", [0, 1, 3])
def test_decode_parity_grid(hq, hkv, d, P, splits):
    shape = Shape(2, hq, hkv, d, P)
    p = Pair(shape, num_pages=2048, max_seqs=8, max_pages_per_seq=512)
    scripts = [
        [("latent", 128)] * 3 + [("tokens", 700)],
        [("tokens", 1)],
        [("latent", 8), ("tokens", 33), ("latent", 128), ("tokens", 250)],  # partial pages mid-table
        [("latent", 128), ("latent", 100)],
        [("tokens", 2000)],
    ]
    seqs = [p.build(sc) for sc in scripts]
    p.cache.set_decode_splits(splits)
    q = p.queries(len(seqs))
    got = p.cache.decode(1, seqs, q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_decode(p, seqs, q, layer=1), f"decode {hq}/{hkv}/{d}/P{P}/S{splits}")


def test_decode_peaked_softmax():
    """K x 3 stress: peaked softmax, V x 0.5 keeps |o| < 4."""
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=4096, max_seqs=4, max_pages_per_seq=1024, v_scale=0.5)
    seqs = []
    for _ in range(3):
        s = p.new_seq()
        kv = p.draw.latent(shape, 128)
        kv[:, 0] *= 3
        kv[:, 1] *= 0.5
        p.cache.latent_install(s, -1, kv.cuda())
        p.orc.install(s, -1, f64(kv))
        k, v = p.draw.tokens(shape, 3000, 0.5)
        k = (k.float() * 3).to(torch.bfloat16)
        p.cache.append_kv([s], [3000], k.cuda(), v.cuda())
        p.orc.append(s, f64(k), f64(v))
        seqs.append(s)
    q = p.queries(3)
    got = p.cache.decode(0, seqs, q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_decode(p, seqs, q), "peaked")


# ----------------------------------------------------------------------------- invariants
def _decode_once(placement_seed, as_latent, splits=0):
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=1024, max_seqs=2, max_pages_per_seq=512, placement_seed=placement_seed)
    s = p.new_seq()
    kv = p.draw.latent(shape, 128)
    if as_latent:
        p.cache.latent_install(s, -1, kv.cuda())
    else:  # the same rows appended as token KV (kind flip)
        p.cache.append_kv([s], [128], kv[:, 0].contiguous().cuda(), kv[:, 1].contiguous().cuda())
    s2 = p.new_seq()  # keeps the token segment of `s` a separate segment either way
    p.cache.latent_install(s2, -1, kv.cuda())
    if not as_latent:
        p.cache.latent_install(s, -1, p.draw.latent(shape, 128).cuda())
    else:
        p.cache.latent_install(s, -1, p.draw.latent(shape, 128).cuda())
    k, v = p.draw.tokens(shape, 1000)
    p.cache.append_kv([s], [1000], k.cuda(), v.cuda())
    p.cache.set_decode_splits(splits)
    q = p.queries(1).cuda()
    out = p.cache.decode(0, [s], q)
    torch.cuda.synchronize()
    return out.cpu()


def test_physical_placement_invariance_bitwise():
    a = _decode_once(1, True)
    for seed in (2, 77, 0):
        assert torch.equal(a, _decode_once(seed, True))


def test_kind_flip_bitwise():
    """Latent page = just KV: the same rows stored as a latent set or as tokens."""
    assert torch.equal(_decode_once(5, True), _decode_once(5, False))


def test_split_invariance():
    a = _decode_once(3, True, splits=1).float()
    for s in (2, 5, 16):
        b = _decode_once(3, True, splits=s).float()
        assert torch.max(torch.abs(a - b)) <= 2 ** -7 * (1 + torch.max(torch.abs(a)))


def test_split_invariance_fp32_partials():
    """SURVEY §8(c) "Split invariance", on the fp32 result of the split combine
    (hpa_decode_partial writes fp32 O and the LSE: no bf16 output rounding hides an error).
    (a) q = 0: every score is 0, so every P weight is exactly 1 in every split and the only
        difference between split counts is fp32 summation order and the combine's weights
        2^(lse_s - LSE) over ragged split lengths -> <= 1e-5 relative.
    (b) random q: each split (and each consumer warp) rounds its P weights to bf16 relative to
        its own running max (reading A9), a relative perturbation <= 2^-9 per weight, so S = 1
        and S = k may differ by that much: rel-L2 <= 2^-9."""
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=2048, max_seqs=4, max_pages_per_seq=512)
    seqs = [p.build([("latent", 128), ("tokens", n)]) for n in (1000, 3333, 77)]
    for q, tol in ((torch.zeros((len(seqs), 32, 128), dtype=torch.bfloat16), 1e-5),
                   (p.queries(len(seqs)), 2.0 ** -9)):
        q = q.cuda()
        p.cache.set_decode_splits(1)
        o1, l1 = p.cache.decode_partial(0, seqs, q)
        for splits in (0, 2, 3, 5, 16):
            p.cache.set_decode_splits(splits)
            o, l = p.cache.decode_partial(0, seqs, q)
            torch.cuda.synchronize()
            rel = (torch.linalg.vector_norm(o - o1) / torch.linalg.vector_norm(o1)).item()
            assert rel <= tol, (splits, rel, tol)
            assert torch.allclose(l, l1, rtol=0, atol=1e-5 * (1 + l1.abs().max().item())), splits
    p.cache.set_decode_splits(0)


def test_rows_beyond_valid_are_masked():
    """Junk written into pool rows >= valid_rows (partial pages) changes nothing."""
    shape = Shape(1, 8, 2, 128, 16)
    p = Pair(shape, num_pages=256, max_seqs=2, max_pages_per_seq=64)
    s = p.build([("latent", 8), ("tokens", 21), ("latent", 100), ("tokens", 3)])
    q = p.queries(3)
    out1 = p.cache.decode(0, [s], q[:1].cuda()).clone()
    pre1 = p.cache.prefill(0, [s], [3], q.cuda()).clone()
    pages, pos0, meta = p.cache.export_table(s)
    kp, vp = p.cache.pools()
    for pg, m in zip(pages, meta):
        valid = int(m & 0x7fff)
        kp[0, pg, :, valid:] = 1000.0
        vp[0, pg, :, valid:] = -777.0
    out2 = p.cache.decode(0, [s], q[:1].cuda())
    pre2 = p.cache.prefill(0, [s], [3], q.cuda())
    torch.cuda.synchronize()
    assert torch.equal(out1, out2)
    assert torch.equal(pre1, pre2)


def test_gqa_mapping_constant_v():
    """kv-head h holds V == h+1 everywhere -> q-head hq returns floor(hq/G)+1."""
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=256, max_seqs=1, max_pages_per_seq=64)
    s = p.new_seq()
    k, _ = p.draw.tokens(shape, 300)
    v = torch.arange(1, 9, dtype=torch.bfloat16)[None, None, :, None].expand(1, 300, 8, 128).contiguous()
    p.cache.append_kv([s], [300], k.cuda(), v.cuda())
    out = p.cache.decode(0, [s], p.queries(1).cuda()).float().cpu()
    exp = (torch.arange(32) // 4 + 1).float()[:, None].expand(32, 128)
    assert torch.equal(out[0], exp)


# ----------------------------------------------------------------------------- prefill
PREFILL_GRID = [(32, 8, 128, 16), (32, 8, 128, 64), (8, 2, 64, 16), (4, 4, 128, 256), (16, 1, 128, 32)]


@pytest.mark.parametrize("hq,hkv,d,P", PREFILL_GRID)
def test_prefill_parity_grid(hq, hkv, d, P):
    shape = Shape(1, hq, hkv, d, P)
    p = Pair(shape, num_pages=4096, max_seqs=4, max_pages_per_seq=1024)
    scripts = [[("latent", 128), ("latent", 8), ("tokens", 300)],
               [("tokens", 77)],
               [("latent", 128)] * 2 + [("tokens", 900)]]
    seqs = [p.build(sc) for sc in scripts]
    q_lens = [300, 1, 385]          # several 128-row tiles + ragged tails; q_len 1
    q = p.queries(sum(q_lens))
    got = p.cache.prefill(0, seqs, q_lens, q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_prefill(p, seqs, q_lens, q), f"prefill {hq}/{hkv}/{d}/P{P}")


def test_prefill_queries_spanning_latent_rows():
    """q_len = seq_len: queries cover latent rows too (latent<->latent causal, A3)."""
    shape = Shape(1, 8, 2, 128, 16)
    p = Pair(shape, num_pages=512, max_seqs=2, max_pages_per_seq=128)
    s = p.build([("latent", 128), ("tokens", 100), ("latent", 8)])
    q = p.queries(236)
    got = p.cache.prefill(0, [s], [236], q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_prefill(p, [s], [236], q), "prefill full")


def test_chunk_equals_decodes():
    """Causal consistency: row t of a prefill == decode of the prefix ending at t."""
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=1024, max_seqs=8, max_pages_per_seq=256)
    s = p.build([("latent", 128), ("tokens", 500)])
    q = p.queries(4)
    pre = p.cache.prefill(0, [s], [4], q.cuda()).float()
    dec = p.cache.decode(0, [s], q[3:4].cuda()).float()
    torch.cuda.synchronize()
    assert torch.max(torch.abs(pre[3] - dec[0])) <= 2e-2
    check_close(pre, oracle_prefill(p, [s], [4], q), "chunk")


# ----------------------------------------------------------------------------- O(1) latent update
def _page_hash(cache, pages):
    kp, vp = cache.pools()
    h = hashlib.sha256()
    for pg in pages:
        h.update(kp[:, pg].contiguous().view(torch.int16).cpu().numpy().tobytes())
        h.update(vp[:, pg].contiguous().view(torch.int16).cpu().numpy().tobytes())
    return h.hexdigest()


def test_latent_replace_same_size_and_splice():
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=2048, max_seqs=4, max_pages_per_seq=512)
    seqs = [p.build([("latent", 128)] * 4 + [("tokens", 600)]) for _ in range(3)]
    pages, _, meta = p.cache.export_table(seqs[0])
    tok_pages = [int(pg) for pg, m in zip(pages, meta) if not m & META_LATENT_BIT]
    lat_pages = [int(pg) for pg, m in zip(pages, meta) if m & META_LATENT_BIT]
    h0 = _page_hash(p.cache, tok_pages)
    # same size: batched in-place rewrite of set `1` for every sequence
    kvs = [p.draw.latent(shape, 128) for _ in seqs]
    p.cache.latent_install_batch(seqs, [1] * 3, [kv.cuda() for kv in kvs])
    for s, kv in zip(seqs, kvs):
        p.orc.install(s, 1, f64(kv))
    pages2, _, meta2 = p.cache.export_table(seqs[0])
    assert list(pages2) == list(pages) and list(meta2) == list(meta)  # same pages, no splice
    assert _page_hash(p.cache, tok_pages) == h0                      # token pages untouched
    q = p.queries(3)
    got = p.cache.decode(0, seqs, q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_decode(p, seqs, q), "replace same size")
    # different size: splice (set 2 of seq 1 -> 40 rows; set 0 of seq 2 -> 300 rows)
    for s, sid, m in ((seqs[1], 2, 40), (seqs[2], 0, 300)):
        p.latent(s, m, set_id=sid)
    p.cache.latent_remove(seqs[0], 3)
    p.orc.remove(seqs[0], 3)
    for s in seqs:
        pages, pos0, meta = p.cache.export_table(s)
        assert [(("latent" if m & META_LATENT_BIT else "token"), int(m & 0x7fff), int(p0))
                for m, p0 in zip(meta, pos0)] == p.orc.expected_table(s)
    q = p.queries(3)
    got = p.cache.decode(0, seqs, q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_decode(p, seqs, q), "replace splice")
    assert len(lat_pages) == 32


# ----------------------------------------------------------------------------- errors
def test_errors_leave_cache_unchanged():
    from paper_2605_09100_b200 import HPAError
    shape = Shape(1, 4, 2, 64, 16)
    p = Pair(shape, num_pages=10, max_seqs=2, max_pages_per_seq=8)
    s = p.build([("latent", 16), ("tokens", 40)])  # 1 + 3 pages
    before = (p.cache.stats(), p.cache.export_table(s)[0].tolist())
    k, v = p.draw.tokens(shape, 200)
    with pytest.raises(HPAError) as e:
        p.cache.append_kv([s], [200], k.cuda(), v.cuda())
    assert e.value.name in ("HPA_ERR_OUT_OF_PAGES", "HPA_ERR_SEQ_CAPACITY")
    s2 = p.cache.seq_create()
    k, v = p.draw.tokens(shape, 120)
    with pytest.raises(HPAError) as e:
        p.cache.append_kv([s2], [120], k.cuda(), v.cuda())  # 8 pages needed, 6 free
    assert e.value.name == "HPA_ERR_OUT_OF_PAGES"
    assert (p.cache.stats()[0], p.cache.export_table(s)[0].tolist()) == (6, before[1])
    with pytest.raises(HPAError) as e:
        p.cache.decode(0, [s2], torch.zeros(1, 4, 64, dtype=torch.bfloat16, device="cuda"))
    assert e.value.name == "HPA_ERR_INVALID_ARG"  # empty sequence
    with pytest.raises(HPAError) as e:
        p.cache.prefill(0, [s], [57], torch.zeros(57, 4, 64, dtype=torch.bfloat16, device="cuda"))
    assert e.value.name == "HPA_ERR_INVALID_ARG"  # q_len > seq_len
    with pytest.raises(HPAError) as e:
        p.cache.latent_remove(s, 9)
    assert e.value.name == "HPA_ERR_UNKNOWN_SET"
    with pytest.raises(HPAError) as e:
        p.cache.decode(0, [1 - s + 5], torch.zeros(1, 4, 64, dtype=torch.bfloat16, device="cuda"))
    assert e.value.name == "HPA_ERR_UNKNOWN_SEQ"
    p.cache.seq_release(s)
    assert p.cache.stats() == (10, 0, 1)


def test_allocator_fuzz_against_model():
    """1000 random append / install / replace / remove / release ops keep
    free + used == NP, used == pages referenced by live tables, and every
    table equal to the model's expected table."""
    import random
    from paper_2605_09100_b200 import HPAError
    rng = random.Random(0)
    shape = Shape(1, 2, 1, 64, 16)
    p = Pair(shape, num_pages=300, max_seqs=6, max_pages_per_seq=64)
    live = []
    for step in range(1000):
        op = rng.random()
        try:
            if op < 0.15 and len(live) < 6:
                live.append(p.new_seq())
            elif op < 0.45 and live:
                s = rng.choice(live)
                p.tokens([s], [rng.randint(0, 40)])
            elif op < 0.65 and live:
                s = rng.choice(live)
                ids = [sg.set_id for sg in p.orc.seqs[s] if sg.kind == "latent"]
                sid = rng.choice(ids) if ids and rng.random() < 0.5 else -1
                p.latent(s, rng.randint(1, 70), set_id=sid)
            elif op < 0.75 and live:
                s = rng.choice(live)
                ids = [sg.set_id for sg in p.orc.seqs[s] if sg.kind == "latent"]
                if ids:
                    sid = rng.choice(ids)
                    p.cache.latent_remove(s, sid)
                    p.orc.remove(s, sid)
            elif op < 0.85 and live:
                s = live.pop(rng.randrange(len(live)))
                p.cache.seq_release(s)
                p.orc.release(s)
        except HPAError as e:
            assert e.name in ("HPA_ERR_OUT_OF_PAGES", "HPA_ERR_SEQ_CAPACITY")
            # the oracle op was not applied either (the GPU call raised first)
        free, used, nlive = p.cache.stats()
        assert free + used == 300 and nlive == len(live)
        assert used == sum(p.cache.seq_info(s)[1] for s in live)
        if step % 50 == 0:
            for s in live:
                _, pos0, meta = p.cache.export_table(s)
                assert [(("latent" if m & META_LATENT_BIT else "token"), int(m & 0x7fff), int(x))
                        for m, x in zip(meta, pos0)] == p.orc.expected_table(s)
    torch.cuda.synchronize()
    for s in live:
        k1, v1 = p.orc.logical_kv(s, 0)
        k2, v2 = p.cache.export_logical_kv(0, s)
        assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2))


# ----------------------------------------------------------------------------- NEXT-1: compression
@pytest.mark.parametrize("P", [16, 64])
def test_compress_in_cache(P):
    """In-cache compression (hpa_seq_compress): [latents 128 | tokens 21 | doc n | meta-latent m]
    -> [latents 128 | tokens 21 | LATENT m]; bit-exact table/gather vs the oracle model, decode and
    prefill parity after compression, document pages returned to the pool."""
    shape = Shape(1, 8, 2, 128, P)
    p = Pair(shape, num_pages=2048, max_seqs=4, max_pages_per_seq=256)
    seqs = []
    for n_doc, m in ((300, 128), (5, 40), (0, 16)):
        s = p.build([("latent", 128), ("tokens", 21 + n_doc + m)])
        seqs.append(s)
        free0 = p.cache.stats()[0]
        got = p.cache.compress(s, n_doc, m)
        assert got == p.orc.compress(s, n_doc, m)
        pages_before = -(-(21 + n_doc + m) // P)
        pages_after = -(-21 // P) + -(-m // P)
        assert p.cache.stats()[0] == free0 + pages_before - pages_after
    p.tokens(seqs, [3, 17, 1])          # appending after a compressed set opens a token segment
    torch.cuda.synchronize()
    for s in seqs:
        pages, pos0, meta = p.cache.export_table(s)
        assert [(("latent" if m & META_LATENT_BIT else "token"), int(m & 0x7fff), int(x))
                for m, x in zip(meta, pos0)] == p.orc.expected_table(s)
        k1, v1 = p.orc.logical_kv(s, 0)
        k2, v2 = p.cache.export_logical_kv(0, s)
        assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2))
    q = p.queries(3)
    got = p.cache.decode(0, seqs, q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_decode(p, seqs, q), "decode after compress")
    q = p.queries(20)
    got = p.cache.prefill(0, [seqs[0]], [20], q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_prefill(p, [seqs[0]], [20], q), "prefill after compress")


@pytest.mark.parametrize("P,fp8", [(16, False), (32, False), (16, True)])
def test_compress_batch(P, fp8):
    """hpa_seq_compress_batch: five requests (including a fork sharing the documents' prefix)
    compressed in one call == the oracle's sequential compressions; bit-exact views and tables,
    exact page accounting, decode parity; a bad request or a repeated sequence changes nothing."""
    from paper_2605_09100_b200 import HPAError
    shape = Shape(2, 8, 2, 128, P)
    p = Pair(shape, num_pages=3000, max_seqs=8, max_pages_per_seq=256, token_fp8=fp8,
             num_token_pages=3000 if fp8 else 0)
    jobs = [(300, 128), (5, 40), (0, 16), (77, 128), (10, 24)]
    seqs = [p.build([("latent", 128), ("tokens", 21 + n_doc + m)]) for n_doc, m in jobs]
    fork = p.cache.seq_fork(seqs[0], 128 + 21)
    p.orc.fork(seqs[0], 128 + 21, fork)
    state0 = (p.cache.stats(), [p.cache.export_table(s)[0].tolist() for s in seqs])
    with pytest.raises(HPAError) as e:                       # request 3 asks for too many rows
        p.cache.compress_batch(seqs, [n for n, _ in jobs[:3]] + [10 ** 4] + [jobs[4][0]], [m for _, m in jobs])
    assert e.value.name == "HPA_ERR_INVALID_ARG"
    with pytest.raises(HPAError) as e:                       # a sequence twice
        p.cache.compress_batch([seqs[0], seqs[0]], [1, 1], [8, 8])
    assert e.value.name == "HPA_ERR_INVALID_ARG"
    assert (p.cache.stats(), [p.cache.export_table(s)[0].tolist() for s in seqs]) == state0
    got = p.cache.compress_batch(seqs, [n for n, _ in jobs], [m for _, m in jobs])
    for i, (s, (n_doc, m)) in enumerate(zip(seqs, jobs)):
        assert got[i] == p.orc.compress(s, n_doc, m)
    torch.cuda.synchronize()
    live = seqs + [fork]
    for layer in (0, 1):
        for s in live:
            pages, pos0, meta = p.cache.export_table(s)
            assert [(("latent" if mm & META_LATENT_BIT else "token"), int(mm & 0x7fff), int(x))
                    for mm, x in zip(meta, pos0)] == p.orc.expected_table(s)
            k1, v1 = p.orc.logical_kv(s, layer, fp8_staged=fp8)  # export gives fp8 rows as bf16 (A20)
            k2, v2 = p.cache.export_logical_kv(layer, s)
            assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2))
    q = p.queries(len(live))
    out = p.cache.decode(1, live, q.cuda())
    torch.cuda.synchronize()
    ref = np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, 1), shape.scale)[0] for i, s in enumerate(live)])
    check_close(out, ref, "decode after batched compress")


def test_compress_errors_leave_cache_unchanged():
    from paper_2605_09100_b200 import HPAError
    shape = Shape(1, 4, 2, 64, 16)
    p = Pair(shape, num_pages=64, max_seqs=2, max_pages_per_seq=32)
    s = p.build([("tokens", 40), ("latent", 16)])
    before = (p.cache.stats(), p.cache.export_table(s)[0].tolist())
    with pytest.raises(HPAError) as e:
        p.cache.compress(s, 4, 8)              # trailing segment is LATENT
    assert e.value.name == "HPA_ERR_INVALID_ARG"
    p.tokens([s], [10])
    with pytest.raises(HPAError) as e:
        p.cache.compress(s, 5, 6)              # 11 > 10 rows in the trailing token segment
    assert e.value.name == "HPA_ERR_INVALID_ARG"
    assert p.cache.stats()[0] == before[0][0] - 1


# ----------------------------------------------------------------------------- NEXT-2: sharing
def test_shared_latent_sets_refcount_and_copy_on_write():
    """A document's latent set installed once and shared by 3 other requests: pages are
    stored once (stats), decode parity for all, replacement in one request copies on
    write (others unchanged, bitwise), removal/release drop only references."""
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=1024, max_seqs=8, max_pages_per_seq=256)
    owner = p.build([("latent", 128), ("latent", 40)])     # 8 + 3 pages
    readers = [p.build([("tokens", 30 + 7 * i)]) for i in range(3)]
    used0 = p.cache.stats()[1]
    for r in readers:
        assert p.cache.latent_share(r, owner, 0) == p.orc.share(r, owner, 0)
        p.tokens([r], [5])
    assert p.cache.stats()[1] == used0 + 3                 # only the 3 new token pages
    seqs = [owner] + readers
    q = p.queries(4)
    got = p.cache.decode(0, seqs, q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_decode(p, seqs, q), "decode with shared sets")
    before = [p.cache.export_logical_kv(0, s) for s in readers]
    p.latent(readers[0], 128, set_id=0)                    # copy-on-write replacement
    assert p.cache.stats()[1] == used0 + 3 + 8
    p.latent(owner, 128, set_id=0)                         # owner also replaces: shared still by 2
    torch.cuda.synchronize()
    for r, (k0, v0) in zip(readers[1:], before[1:]):
        k1, v1 = p.cache.export_logical_kv(0, r)
        assert torch.equal(k0, k1) and torch.equal(v0, v1)
    for s in seqs:
        k1, v1 = p.orc.logical_kv(s, 0)
        k2, v2 = p.cache.export_logical_kv(0, s)
        assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2))
    q = p.queries(4)
    got = p.cache.decode(0, seqs, q.cuda())
    torch.cuda.synchronize()
    check_close(got, oracle_decode(p, seqs, q), "decode after copy-on-write")
    for r in readers:
        p.cache.seq_release(r)
    p.cache.seq_release(owner)
    assert p.cache.stats() == (1024, 0, 0)


# ----------------------------------------------------------------------------- NEXT-3: host staging
def test_install_from_host_payloads_scattered():
    """hpa_latent_set_install_host with payloads of different sizes, some back to back in one
    host buffer (coalesced into one copy) and some in separate buffers, in any order."""
    import ctypes

    from paper_2605_09100_b200._lib import LIB, check
    shape = Shape(2, 32, 8, 128, 16)
    p = Pair(shape, num_pages=2048, max_seqs=8, max_pages_per_seq=256)
    seqs = [p.build([("latent", 128), ("tokens", 100 + 30 * i)]) for i in range(5)]
    ms = [128, 40, 128, 16, 72]
    kvs = [p.draw.latent(shape, m) for m in ms]                    # [L][2][m][Hkv][d]
    joint = torch.cat([kvs[0].reshape(-1), kvs[1].reshape(-1)]).pin_memory()  # payloads 0, 1 back to back
    sep = [kvs[i].contiguous().pin_memory() for i in (2, 3, 4)]
    ptrs = [joint.data_ptr(), joint.data_ptr() + kvs[0].numel() * 2] + [t.data_ptr() for t in sep]
    order = [3, 0, 1, 4, 2]                                         # request order != buffer order
    ids = np.array([seqs[i] for i in order], np.int32)
    sids = np.full(5, -1, np.int32)
    mrows = np.array([ms[i] for i in order], np.int32)
    hp = (ctypes.c_void_p * 5)(*[ptrs[i] for i in order])
    out = np.zeros(5, np.int32)
    i32p = ctypes.POINTER(ctypes.c_int32)
    check(LIB.hpa_latent_set_install_host(p.cache._h, 5, ids.ctypes.data_as(i32p), sids.ctypes.data_as(i32p),
                                          mrows.ctypes.data_as(i32p), hp,
                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream),
                                          out.ctypes.data_as(i32p)))
    for k, i in enumerate(order):
        assert out[k] == p.orc.install(seqs[i], -1, f64(kvs[i]))
    torch.cuda.synchronize()
    for layer in (0, 1):
        for s in seqs:
            k1, v1 = p.orc.logical_kv(s, layer)
            k2, v2 = p.cache.export_logical_kv(layer, s)
            assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2))


def test_install_from_host_payloads():
    """hpa_latent_set_install_host (pinned host payloads, internal copy stream) installs the
    same bits as the device-payload path; repeated calls reuse the staging buffer while
    decodes are queued in between."""
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=2048, max_seqs=8, max_pages_per_seq=256)
    seqs = [p.build([("latent", 128), ("tokens", 200 + 50 * i)]) for i in range(4)]
    for step in range(3):
        kv = torch.stack([p.draw.latent(shape, 128) for _ in seqs]).pin_memory()   # [n][L][2][m][Hkv][d]
        sid = [0] * 4 if step else [-1] * 4
        got = p.cache.latent_install_host(seqs, sid, kv)
        for i, s in enumerate(seqs):
            assert got[i] == p.orc.install(s, sid[i], f64(kv[i]))
        q = p.queries(4)
        out = p.cache.decode(0, seqs, q.cuda())
        torch.cuda.synchronize()
        check_close(out, oracle_decode(p, seqs, q), f"decode after host install {step}")
    for s in seqs:
        k1, v1 = p.orc.logical_kv(s, 0)
        k2, v2 = p.cache.export_logical_kv(0, s)
        assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2))


# ----------------------------------------------------------------------------- NEXT-4a: mask-out span
@pytest.mark.parametrize("hq,hkv,P", [(32, 8, 16), (8, 8, 64), (6, 2, 32)])
def test_prefill_span_grc_mask(hq, hkv, P):
    """Eq. (1) layout [segment 1 (n1) | latents (m) | segment 3 (n3)]: the m + n3 queries run
    with span (0, n1, n1 + m); parity with oracle.attend_span; rows of segment 3 equal plain
    prefill over a cache without segment 1."""
    from oracle import attend_span
    shape = Shape(1, hq, hkv, 128, P)
    p = Pair(shape, num_pages=2048, max_seqs=8, max_pages_per_seq=256)
    cases = [(300, 16, 150), (40, 128, 200), (0, 8, 50), (257, 64, 1)]
    seqs, q_lens, spans = [], [], []
    for n1, m, n3 in cases:
        s = p.new_seq()
        p.tokens([s], [n1]) if n1 else None
        p.latent(s, m)
        p.tokens([s], [n3])
        seqs.append(s)
        q_lens.append(m + n3)
        spans.append((0, n1, n1 + m))
    q = p.queries(sum(q_lens))
    got = p.cache.prefill_span(0, seqs, q_lens, spans, q.cuda())
    torch.cuda.synchronize()
    ref, off = [], 0
    for s, ql, (lo, hi, qf) in zip(seqs, q_lens, spans):
        k, v = p.orc.logical_kv(s, 0)
        ref.append(attend_span(f64(q[off:off + ql]), k, v, shape.scale, lo, hi, qf))
        off += ql
    ref = np.concatenate(ref)
    check_close(got, ref, "prefill span")
    # segment-3 rows == a cache whose segment-1 pages are absent (reading A4)
    p2 = Pair(shape, num_pages=2048, max_seqs=8, max_pages_per_seq=256)
    n1, m, n3 = cases[0]
    s2 = p2.new_seq()
    k, v = p.orc.logical_kv(seqs[0], 0)
    kk = torch.from_numpy(k[:, n1:]).to(torch.bfloat16).permute(1, 0, 2).unsqueeze(0).contiguous()
    vv = torch.from_numpy(v[:, n1:]).to(torch.bfloat16).permute(1, 0, 2).unsqueeze(0).contiguous()
    p2.cache.append_kv([s2], [m + n3], kk.cuda(), vv.cuda())
    plain = p2.cache.prefill(0, [s2], [m + n3], q[:m + n3].cuda())
    torch.cuda.synchronize()
    assert torch.max(torch.abs(plain[m:].float() - got[m:m + n3].float())) <= 2e-2


# ----------------------------------------------------------------------------- NEXT-4b: context parallel
@pytest.mark.parametrize("n_shards", [1, 2, 3])
def test_context_parallel_decode_shards_merge(n_shards):
    """A long sequence split by row ranges over n shards (one 'rank' per shard, emulated as
    sequences of one cache): hpa_decode_partial per shard + hpa_merge_partials == the oracle
    over the full sequence; the fp32 partials match oracle.partial_attend per shard."""
    from oracle import partial_attend
    from paper_2605_09100_b200 import merge_partials
    shape = Shape(1, 32, 8, 128, 16)
    p = Pair(shape, num_pages=4096, max_seqs=16, max_pages_per_seq=1024)
    full = [("latent", 128)] * 4 + [("tokens", 3001)]
    n_req = 3
    d = Draw(77)
    # draw each request's rows once (CPU), then split them over the shards
    req_rows = []
    for _ in range(n_req):
        rows = []
        for kind, n in full:
            if kind == "latent":
                kv = d.latent(shape, n)
                rows.append((kind, kv[:, 0], kv[:, 1]))
            else:
                k, v = d.tokens(shape, n)
                rows.append((kind, k, v))
        req_rows.append(rows)
    shard_seqs = [[None] * n_req for _ in range(n_shards)]
    for r, rows in enumerate(req_rows):
        k_all = torch.cat([k for _, k, _ in rows], 1)
        v_all = torch.cat([v for _, _, v in rows], 1)
        lb = k_all.shape[1]
        cuts = [lb * i // n_shards for i in range(n_shards + 1)]
        for sh in range(n_shards):
            s = p.new_seq()
            a, b = cuts[sh], cuts[sh + 1]
            p.cache.append_kv([s], [b - a], k_all[:, a:b].contiguous().cuda(), v_all[:, a:b].contiguous().cuda())
            p.orc.append(s, f64(k_all[:, a:b]), f64(v_all[:, a:b]))
            shard_seqs[sh][r] = s
    q = p.queries(n_req)
    parts = [p.cache.decode_partial(0, shard_seqs[sh], q.cuda()) for sh in range(n_shards)]
    out = merge_partials(torch.stack([o for o, _ in parts]), torch.stack([l for _, l in parts]))
    torch.cuda.synchronize()
    ref_parts = []
    for sh in range(n_shards):
        o_sh, l_sh = [], []
        for r in range(n_req):
            k, v = p.orc.logical_kv(shard_seqs[sh][r], 0)
            o1, l1 = partial_attend(f64(q[r]), k, v, shape.scale)
            o_sh.append(o1)
            l_sh.append(l1)
        ref_parts.append((np.stack(o_sh), np.stack(l_sh)))
        assert np.max(np.abs(f64(parts[sh][1]) - ref_parts[-1][1])) <= 1e-3       # LSE (log2)
        assert np.max(np.abs(f64(parts[sh][0]) - ref_parts[-1][0])) <= 1e-2
    ref = []
    for r in range(n_req):
        k = np.concatenate([p.orc.logical_kv(shard_seqs[sh][r], 0)[0] for sh in range(n_shards)], 1)
        v = np.concatenate([p.orc.logical_kv(shard_seqs[sh][r], 0)[1] for sh in range(n_shards)], 1)
        ref.append(attend(f64(q[r:r + 1]), k, v, shape.scale)[0])
    check_close(out, np.stack(ref), f"context-parallel decode over {n_shards} shards")


# ----------------------------------------------------------------------------- planner edge cases
def test_decode_many_tiny_requests_and_more_ctas_than_units():
    """4096 one-row requests (units << CTA slots is false: units >> slots, S_b = 1 everywhere)
    and a 3-request batch (fewer units than resident CTAs): both through the persistent kernel."""
    from tests.hpa_testutil import Pair
    shape = Shape(num_layers=1, num_q_heads=8, num_kv_heads=2, head_dim=128, page_size=16)
    pr = Pair(shape, num_pages=4200, max_seqs=4100, max_pages_per_seq=4)
    seqs = [pr.new_seq() for _ in range(4096)]
    pr.tokens(seqs, [1] * 4096)
    q = pr.queries(4096)
    out = pr.cache.decode(0, seqs, q.cuda())
    torch.cuda.synchronize()
    for i in (0, 1, 777, 2048, 4095):
        ref = attend(f64(q[i:i + 1]), *pr.orc.logical_kv(seqs[i], 0), shape.scale)
        check_close(out[i:i + 1], ref, f"tiny request {i}")
    few = seqs[:3]
    out3 = pr.cache.decode(0, few, q[:3].cuda())
    assert torch.equal(out3, out[:3])              # same per-request result, different grid / plan


def test_decode_one_long_request_many_splits():
    """A single 40K-row request (1 request x H_kv units: the planner splits it up to 64 ways)
    next to a short one: parity and equality with a forced single split."""
    from tests.hpa_testutil import Pair
    shape = Shape(num_layers=1, num_q_heads=16, num_kv_heads=2, head_dim=64, page_size=64)
    pr = Pair(shape, num_pages=800, max_seqs=4, max_pages_per_seq=700)
    a = pr.build([("latent", 128), ("tokens", 40000)])
    b = pr.build([("tokens", 50)])
    q = pr.queries(2)
    out = pr.cache.decode(0, [a, b], q.cuda())
    for i, s in enumerate([a, b]):
        check_close(out[i:i + 1], attend(f64(q[i:i + 1]), *pr.orc.logical_kv(s, 0), shape.scale), f"long req {i}")
    pr.cache.set_decode_splits(1)
    out1 = pr.cache.decode(0, [a, b], q.cuda())
    rel = float((out1.float() - out.float()).norm() / out.float().norm())
    assert rel < 1e-2
