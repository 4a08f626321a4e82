"""Pins for the CPU oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a number printed by the paper,
a closed form, a library routine (torch SDPA) with an explicit mask, or a
pure-Python brute force written independently of oracle/hpa_oracle.py.
"""
import math
import os
import random

import numpy as np
import pytest
import torch

from oracle import OracleCache, attend, expected_table, gather_physical, kv_cache_bytes
from oracle.hpa_oracle import META_LATENT_BIT
from workloads import Draw, Shape, tiny_decode

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def f64(t):
    return t.to(torch.float64).numpy()


def build_cache(shape: Shape, script, seed=0, v_scale=1.0):
    """Drive an OracleCache with a list of ("latent", m) / ("tokens", n) segments."""
    c = OracleCache(shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim,
                    shape.page_size)
    c.create_seq(0)
    d = Draw(seed)
    for kind, n in script:
        if kind == "latent":
            c.install(0, -1, f64(d.latent(shape, n, v_scale)))
        else:
            k, v = d.tokens(shape, n, v_scale)
            c.append(0, f64(k), f64(v))
    return c, d


# --------------------------------------------------------------------------- paper numbers
def test_kv_bytes_matches_paper_golden():
    """P:L232-240 (§3 KV cache cost): 114688 B/token for Qwen3-1.7B, 14 MiB for m=128."""
    rows = 0
    with open(os.path.join(GOLDEN, "kv_bytes_paper.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            L, h, d, n, b, exp = map(int, line.split())
            assert kv_cache_bytes(L, h, d, n, b) == exp
            rows += 1
    assert rows == 5
    assert kv_cache_bytes(28, 8, 128, 1024, 2) == 112 * 1024 * 1024
    assert kv_cache_bytes(28, 8, 128, 128, 2) == 14 * 1024 * 1024


# --------------------------------------------------------------------------- brute force
def _brute_force(q, k, v, scale):
    """Pure-Python triple loop (no numpy), bottom-right causal, hq -> hq // G."""
    tq, hq_n, d = len(q), len(q[0]), len(q[0][0])
    hkv, lb = len(k), len(k[0])
    g = hq_n // hkv
    out = [[[0.0] * d for _ in range(hq_n)] for _ in range(tq)]
    for t in range(tq):
        last = lb - tq + t
        for hq in range(hq_n):
            h = hq // g
            scores = []
            for j in range(last + 1):
                acc = 0.0
                for x in range(d):
                    acc += q[t][hq][x] * k[h][j][x]
                scores.append(acc * scale)
            mx = max(scores)
            w = [math.exp(s - mx) for s in scores]
            tot = sum(w)
            for x in range(d):
                out[t][hq][x] = sum(w[j] * v[h][j][x] for j in range(last + 1)) / tot
    return out


@pytest.mark.parametrize("variant", ["a", "b", "c"])
def test_tiny_config_vs_bruteforce(variant):
    """BASELINE.json configs[0] (tiny decode; b: partial latent page; c: prefill)."""
    w = tiny_decode(variant)
    c, d = build_cache(w.shape, w.seqs[0].segments)
    q = f64(d.queries(w.shape, w.seqs[0].q_len))
    k, v = c.logical_kv(0, 0)
    got = attend(q, k, v, w.shape.scale)
    ref = np.array(_brute_force(q.tolist(), k.tolist(), v.tolist(), w.shape.scale))
    assert np.max(np.abs(got - ref)) <= 1e-12


# --------------------------------------------------------------------------- library routine
@pytest.mark.parametrize("tq,lb,hq,hkv,d", [(1, 64, 2, 1, 64), (16, 64, 2, 1, 64),
                                            (7, 300, 8, 2, 32), (33, 100, 4, 4, 16)])
def test_vs_torch_sdpa_explicit_bottom_right_mask(tq, lb, hq, hkv, d):
    """torch SDPA in fp64 with an explicit boolean bottom-right mask (is_causal is
    top-left aligned when Lq != Lk) and repeat_kv GQA."""
    g = torch.Generator().manual_seed(tq * 1000 + lb)
    q = torch.randn(tq, hq, d, generator=g, dtype=torch.float64)
    k = torch.randn(hkv, lb, d, generator=g, dtype=torch.float64)
    v = torch.randn(hkv, lb, d, generator=g, dtype=torch.float64)
    scale = 1.0 / math.sqrt(d)
    got = attend(q.numpy(), k.numpy(), v.numpy(), scale)
    rows = torch.arange(tq)[:, None] + (lb - tq)
    mask = torch.arange(lb)[None, :] <= rows                       # [tq][lb]
    kk = k.repeat_interleave(hq // hkv, dim=0)                      # [hq][lb][d]
    vv = v.repeat_interleave(hq // hkv, dim=0)
    ref = torch.nn.functional.scaled_dot_product_attention(
        q.transpose(0, 1), kk, vv, attn_mask=mask, scale=scale).transpose(0, 1)
    assert np.max(np.abs(got - ref.numpy())) <= 1e-12


# --------------------------------------------------------------------------- closed forms
def test_uniform_v_gives_v():
    """All visible V rows equal v -> o = v."""
    rng = np.random.default_rng(0)
    k = rng.standard_normal((2, 50, 16))
    v = np.broadcast_to(rng.standard_normal((2, 1, 16)), (2, 50, 16)).copy()
    q = rng.standard_normal((5, 4, 16))
    o = attend(q, k, v, 0.25)
    for hq in range(4):
        assert np.max(np.abs(o[:, hq] - v[hq // 2, 0])) <= 1e-12


def test_equal_keys_give_mean_of_visible_v():
    """All visible K rows equal -> uniform weights -> o = mean of the visible V rows."""
    rng = np.random.default_rng(1)
    k = np.broadcast_to(rng.standard_normal((1, 1, 8)), (1, 40, 8)).copy()
    v = rng.standard_normal((1, 40, 8))
    q = rng.standard_normal((3, 2, 8))
    o = attend(q, k, v, 0.3)
    for t in range(3):
        i = 40 - 3 + t
        assert np.max(np.abs(o[t, 0] - v[0, : i + 1].mean(axis=0))) <= 1e-12


def test_single_row_and_zero_query():
    rng = np.random.default_rng(2)
    k = rng.standard_normal((1, 1, 8))
    v = rng.standard_normal((1, 1, 8))
    assert np.max(np.abs(attend(rng.standard_normal((1, 1, 8)), k, v, 1.0)[0, 0] - v[0, 0])) == 0
    k = rng.standard_normal((1, 30, 8))
    v = rng.standard_normal((1, 30, 8))
    o = attend(np.zeros((1, 1, 8)), k, v, 1.0)                   # q = 0 -> mean of V
    assert np.max(np.abs(o[0, 0] - v[0].mean(axis=0))) <= 1e-12


def test_gqa_mapping_constant_v_per_kv_head():
    """kv-head h holds constant V = h+1 -> q-head hq must return floor(hq/G)+1 (A6)."""
    rng = np.random.default_rng(3)
    hkv, g, lb, d = 4, 3, 20, 8
    k = rng.standard_normal((hkv, lb, d))
    v = np.stack([np.full((lb, d), h + 1.0) for h in range(hkv)])
    o = attend(rng.standard_normal((2, hkv * g, d)), k, v, 0.5)
    for hq in range(hkv * g):
        assert np.max(np.abs(o[:, hq] - (hq // g + 1.0))) <= 1e-12


def test_mask_perturbation_beyond_causal_bound():
    """Perturbing keys/values beyond each row's causal bound leaves that row unchanged."""
    rng = np.random.default_rng(4)
    k = rng.standard_normal((1, 30, 8))
    v = rng.standard_normal((1, 30, 8))
    q = rng.standard_normal((10, 2, 8))
    base = attend(q, k, v, 0.4)
    k2, v2 = k.copy(), v.copy()
    k2[:, 25:] += 100.0
    v2[:, 25:] -= 50.0
    pert = attend(q, k2, v2, 0.4)
    # rows t with i = 20 + t <= 24 see only keys < 25
    assert np.array_equal(base[:5], pert[:5])
    assert not np.allclose(base[5:], pert[5:])


def test_chunk_equals_sequential_decodes():
    """Causal consistency: prefill of C rows = C decodes on growing prefixes."""
    rng = np.random.default_rng(5)
    k = rng.standard_normal((2, 40, 16))
    v = rng.standard_normal((2, 40, 16))
    q = rng.standard_normal((8, 4, 16))
    full = attend(q, k, v, 0.25)
    for t in range(8):
        lb = 40 - 8 + t + 1
        dec = attend(q[t:t + 1], k[:, :lb], v[:, :lb], 0.25)
        assert np.max(np.abs(full[t] - dec[0])) <= 1e-12


# --------------------------------------------------------------------------- paging
def _place(cache: OracleCache, seq: int, num_pages: int, rng: random.Random, L: int):
    """Independent test-side placement: random physical page per table entry."""
    tab = cache.expected_table(seq)
    pages = rng.sample(range(num_pages), len(tab))
    P, h, d = cache.P, cache.Hkv, cache.d
    kp = np.full((L, num_pages, h, P, d), 7.0)   # finite junk in unused rows
    vp = np.full((L, num_pages, h, P, d), -3.0)
    for layer in range(L):
        k, v = cache.logical_kv(seq, layer)
        for (kind, valid, pos0), pg in zip(tab, pages):
            kp[layer, pg, :, :valid] = k[:, pos0:pos0 + valid]
            vp[layer, pg, :, :valid] = v[:, pos0:pos0 + valid]
    meta = [valid | (META_LATENT_BIT if kind == "latent" else 0) for kind, valid, _ in tab]
    return kp, vp, pages, meta


def test_paged_equals_contiguous_under_random_permutations():
    """Route 2 (physical dump + table) == route 1 (model) bitwise for several
    random physical placements, and attention over it is identical."""
    shape = Shape(2, 4, 2, 16, 16)
    script = [("latent", 128), ("latent", 8), ("tokens", 37), ("latent", 20), ("tokens", 5)]
    c, d = build_cache(shape, script)
    q = f64(d.queries(shape, 1))
    outs = []
    for trial in range(4):
        kp, vp, pages, meta = _place(c, 0, 64, random.Random(trial), 2)
        for layer in range(2):
            k1, v1 = c.logical_kv(0, layer)
            k2, v2 = gather_physical(kp, vp, pages, meta, layer)
            assert np.array_equal(k1, k2) and np.array_equal(v1, v2)
        outs.append(attend(q, *gather_physical(kp, vp, pages, meta, 1), shape.scale))
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


def test_expected_table_structure():
    """Every segment starts on a fresh page; only its last page may be partial;
    pos0 = prefix sum of valid_rows; kinds follow the op log (reading A7)."""
    tab = expected_table([("latent", 128), ("latent", 8), ("token", 37), ("latent", 20)], 16)
    valid = [v for _, v, _ in tab]
    assert valid == [16] * 8 + [8] + [16, 16, 5] + [16, 4]
    assert [p for _, _, p in tab] == list(np.cumsum([0] + valid[:-1]))
    assert [k for k, _, _ in tab] == ["latent"] * 9 + ["token"] * 3 + ["latent"] * 2
    # m=8, B=16 -> 1 compressed block; n=17, B=16 -> 2 blocks
    assert len(expected_table([("latent", 8)], 16)) == 1
    assert len(expected_table([("token", 17)], 16)) == 2


def test_uncompressed_replacement_equals_plain_causal_attention():
    """Replacing a latent set by the document's N uncompressed token rows gives
    plain causal attention over the contiguous [doc, rest] (library SDPA)."""
    shape = Shape(1, 4, 2, 32, 16)
    c, d = build_cache(shape, [("latent", 128), ("tokens", 50)])
    doc = f64(d.latent(shape, 300))          # "uncompressed" doc rows, N=300
    c.install(0, 0, doc)                     # replace set 0 (different row count)
    k, v = c.logical_kv(0, 0)
    assert k.shape[1] == 350
    q = f64(d.queries(shape, 3))
    got = attend(q, k, v, shape.scale)
    kk = torch.from_numpy(np.concatenate([doc[0, 0].transpose(1, 0, 2), k[:, 300:]], axis=1))
    vv = torch.from_numpy(np.concatenate([doc[0, 1].transpose(1, 0, 2), v[:, 300:]], axis=1))
    mask = torch.arange(350)[None, :] <= (torch.arange(3)[:, None] + 347)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q).transpose(0, 1), kk.repeat_interleave(2, 0), vv.repeat_interleave(2, 0),
        attn_mask=mask, scale=shape.scale).transpose(0, 1)
    assert np.max(np.abs(got - ref.numpy())) <= 1e-12


def test_replacement_is_o1_and_leaves_token_rows_untouched():
    """O(1) update: replacing a latent set changes only that set's rows."""
    shape = Shape(1, 2, 1, 16, 16)
    c, d = build_cache(shape, [("latent", 128), ("tokens", 100), ("latent", 128), ("tokens", 9)])
    k0, v0 = c.logical_kv(0, 0)
    c.install(0, 1, f64(d.latent(shape, 128)))
    k1, v1 = c.logical_kv(0, 0)
    assert np.array_equal(k0[:, :228], k1[:, :228]) and np.array_equal(k0[:, 356:], k1[:, 356:])
    assert not np.array_equal(k0[:, 228:356], k1[:, 228:356])
    assert c.latent_rows(0) == 256  # per-doc rows = m regardless of document length


def test_set_ids_and_remove():
    shape = Shape(1, 2, 1, 16, 16)
    c, d = build_cache(shape, [("latent", 16), ("latent", 32)])
    assert [s.set_id for s in c.seqs[0]] == [0, 1]
    c.remove(0, 0)
    assert c.install(0, -1, f64(d.latent(shape, 4))) == 2
    assert [(s.kind, s.rows) for s in c.seqs[0]] == [("latent", 32), ("latent", 4)]
    with pytest.raises(KeyError):
        c.remove(0, 7)
    with pytest.raises(ValueError):
        attend(np.zeros((3, 1, 4)), np.zeros((1, 2, 4)), np.zeros((1, 2, 4)), 1.0)


def test_compress_keeps_latent_rows_and_drops_document():
    """NEXT-1 (in-cache compression): [prefix | doc | latents] -> [prefix | LATENT(latents)];
    logical KV equals the explicit concatenation, attention equals SDPA over it, and the
    stored rows are m regardless of the document length (O(1) memory)."""
    shape = Shape(1, 4, 2, 32, 16)
    for n_doc in (0, 7, 300):
        c, d = build_cache(shape, [("latent", 128), ("tokens", 21 + n_doc + 64)])
        k_before, v_before = c.logical_kv(0, 0)
        sid = c.compress(0, n_doc, 64)
        assert sid == 1 and [(s.kind, s.rows) for s in c.seqs[0]] == [("latent", 128), ("token", 21), ("latent", 64)]
        k, v = c.logical_kv(0, 0)
        keep = 128 + 21
        exp_k = np.concatenate([k_before[:, :keep], k_before[:, keep + n_doc:]], axis=1)
        exp_v = np.concatenate([v_before[:, :keep], v_before[:, keep + n_doc:]], axis=1)
        assert np.array_equal(k, exp_k) and np.array_equal(v, exp_v)
        assert c.latent_rows(0) == 128 + 64
        q = f64(d.queries(shape, 2))
        mask = torch.arange(k.shape[1])[None, :] <= (torch.arange(2)[:, None] + k.shape[1] - 2)
        ref = torch.nn.functional.scaled_dot_product_attention(
            torch.from_numpy(q).transpose(0, 1), torch.from_numpy(exp_k).repeat_interleave(2, 0),
            torch.from_numpy(exp_v).repeat_interleave(2, 0), attn_mask=mask, scale=shape.scale).transpose(0, 1)
        assert np.max(np.abs(attend(q, k, v, shape.scale) - ref.numpy())) <= 1e-12
    c, _ = build_cache(shape, [("tokens", 10)])
    with pytest.raises(ValueError):
        c.compress(0, 5, 6)


def test_share_copies_logical_rows_and_isolates_updates():
    """NEXT-2 (shared document memories): the shared set reads as the source's rows; a later
    replacement in either sequence does not change the other (copy-on-write semantics)."""
    shape = Shape(1, 2, 1, 16, 16)
    c = OracleCache(1, 2, 1, 16, 16)
    d = Draw(3)
    for s in (0, 1):
        c.create_seq(s)
    doc = f64(d.latent(shape, 40))
    c.install(0, -1, doc)
    k, v = d.tokens(shape, 5)
    c.append(1, f64(k), f64(v))
    assert c.share(1, 0, 0) == 0
    k1, _ = c.logical_kv(1, 0)
    assert np.array_equal(k1[:, 5:], doc[0, 0].transpose(1, 0, 2))
    c.install(0, 0, f64(d.latent(shape, 40)))           # replace in the source only
    assert np.array_equal(c.logical_kv(1, 0)[0], k1)    # destination unchanged
    with pytest.raises(KeyError):
        c.share(1, 0, 5)


def test_attend_span_vs_sdpa_and_absent_segment():
    """NEXT-4a: the GRC mask-out span. (i) equals SDPA with the explicit mask;
    (ii) for segment-3 queries it equals plain causal attention over the cache with segment 1
    removed (reading A4: at inference the segment-1 pages are simply absent); (iii) the
    latent-token queries (i < q_from) still see segment 1."""
    from oracle import attend_span
    rng = np.random.default_rng(11)
    n1, m, n3, hq, hkv, d = 40, 8, 12, 4, 2, 16
    lb = n1 + m + n3
    k = rng.standard_normal((hkv, lb, d))
    v = rng.standard_normal((hkv, lb, d))
    q = rng.standard_normal((m + n3, hq, d))
    got = attend_span(q, k, v, 0.25, 0, n1, n1 + m)
    i = torch.arange(m + n3)[:, None] + n1
    j = torch.arange(lb)[None, :]
    mask = (j <= i) & ~((i >= n1 + m) & (j < n1))
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q).transpose(0, 1), torch.from_numpy(k).repeat_interleave(2, 0),
        torch.from_numpy(v).repeat_interleave(2, 0), attn_mask=mask, scale=0.25).transpose(0, 1)
    assert np.max(np.abs(got - ref.numpy())) <= 1e-12
    absent = attend(q[m:], k[:, n1:], v[:, n1:], 0.25)
    assert np.max(np.abs(got[m:] - absent)) <= 1e-12
    assert np.max(np.abs(got[:m] - attend(q, k, v, 0.25)[:m])) <= 1e-12


def test_partial_attend_and_merge_equal_full_attention():
    """NEXT-4b: shard softmaxes recombined by LSE equal attention over all keys (SDPA)."""
    from oracle import merge_partials, partial_attend
    rng = np.random.default_rng(12)
    hq, hkv, d, lb = 8, 2, 16, 97
    k = rng.standard_normal((hkv, lb, d))
    v = rng.standard_normal((hkv, lb, d))
    q = rng.standard_normal((hq, d))
    cuts = [0, 30, 31, 80, lb]
    parts = [partial_attend(q, k[:, a:b], v[:, a:b], 0.3) for a, b in zip(cuts[:-1], cuts[1:])]
    got = merge_partials(np.stack([p[0] for p in parts]), np.stack([p[1] for p in parts]))
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q)[:, None], torch.from_numpy(k).repeat_interleave(4, 0),
        torch.from_numpy(v).repeat_interleave(4, 0), scale=0.3)[:, 0]
    assert np.max(np.abs(got - ref.numpy())) <= 1e-12
    o1, l1 = partial_attend(q, k, v, 0.3)           # one shard: lse is log2 sum exp(s)
    s0 = 0.3 * (k[0] @ q[0])
    assert abs(l1[0] - np.log2(np.exp(s0).sum())) <= 1e-12


# ----------------------------------------------------------------------------- NEXT-4c fp8 token pages
def _nearest_e4m3_bruteforce(y):
    """Independent e4m3 rounding: nearest finite code value, ties to the even mantissa,
    saturating at +-448 -- by search over the 254 finite codes."""
    from oracle import e4m3_values
    vals = e4m3_values()
    codes = [c for c in range(256) if np.isfinite(vals[c])]
    out = []
    for t in np.asarray(y, dtype=np.float64).ravel():
        t = min(max(t, -448.0), 448.0)
        best = None
        for c in codes:
            dist = abs(vals[c] - t)
            key = (dist, c & 1)  # ties: even mantissa (lowest code bit) first
            if best is None or key < best[0]:
                best = (key, c)
        c = best[1]
        if vals[c] == 0.0:  # +0 / -0 both encode the value 0: keep the sign of t
            c = 0x80 if np.signbit(t) else 0x00
        out.append(c)
    return np.array(out, dtype=np.uint8).reshape(np.shape(y))


def test_e4m3_format_values():
    from oracle import e4m3_values
    v = e4m3_values()
    assert v[0x7E] == 448.0 and v[0xFE] == -448.0           # largest finite
    assert v[0x01] == 2.0 ** -9 and v[0x08] == 2.0 ** -6     # smallest subnormal / normal
    assert np.isnan(v[0x7F]) and np.isnan(v[0xFF])
    assert np.all(v[:0x7F] == -v[0x80:0xFF])
    assert np.all(np.diff(v[:0x7F]) > 0)                     # codes 0..126 increase strictly


def test_e4m3_encode_matches_bruteforce_including_ties():
    from oracle import e4m3_encode, e4m3_values
    rng = np.random.default_rng(5)
    v = e4m3_values()
    pos = v[:0x7F]
    mids = (pos[:-1] + pos[1:]) / 2                           # exact ties between neighbours
    y = np.concatenate([rng.uniform(-460, 460, 2000), rng.standard_normal(2000) * 0.01,
                        mids, -mids, [0.0, 448.0, 449.0, 463.9, -500.0]]).astype(np.float32)
    got = e4m3_encode(y)
    ref = _nearest_e4m3_bruteforce(y.astype(np.float64))
    same_value = v[got] == v[ref]
    assert np.all(same_value), y[~same_value][:10]


def test_row_quantization_scheme_a20():
    from oracle import dequantize_rows_e4m3, e4m3_values, quantize_rows_e4m3
    rng = np.random.default_rng(6)
    x = (rng.standard_normal((2, 7, 4, 128)) * rng.uniform(0.01, 5, (2, 7, 4, 1))).astype(np.float32)
    x[0, 3, 2] = 0.0                                          # an all-zero row
    codes, s = quantize_rows_e4m3(x)
    v = e4m3_values()
    assert s[0, 3, 2] == 1.0 and np.all(codes[0, 3, 2] == 0)
    amax = np.abs(x).max(-1)
    nz = amax > 0
    # the row's largest magnitude lands on +-448 and the scale is amax / 448 (fp32)
    assert np.all(np.abs(v[codes]).max(-1)[nz] == 448.0)
    assert np.all(s[nz] == (amax[nz] / np.float32(448)).astype(np.float32))
    # dequantized error: at most half a code spacing, i.e. <= 2^-4 relative in the normal
    # range and <= 2^-10 * s below it
    d = dequantize_rows_e4m3(codes, s)
    y = np.abs(x / s[..., None])
    bound = np.where(y >= 2.0 ** -6, 2.0 ** -4 * np.abs(x), 2.0 ** -10 * s[..., None]) * (1 + 1e-6)
    assert np.all(np.abs(d - x) <= bound)


def _bf16(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).to(torch.float64).numpy()


def test_oracle_cache_fp8_tokens_and_bf16_latents():
    from oracle import OracleCache, bf16_round, dequantize_rows_e4m3, e4m3_values, quantize_rows_e4m3
    rng = np.random.default_rng(8)
    c = OracleCache(1, 2, 1, 64, 16, token_fp8=True)
    c.create_seq(0)
    lat = _bf16(rng.standard_normal((1, 2, 16, 1, 64)))
    c.install(0, -1, lat)
    k, v = _bf16(rng.standard_normal((1, 40, 1, 64))), _bf16(rng.standard_normal((1, 40, 1, 64)))
    c.append(0, k, v)
    kl, vl = c.logical_kv(0, 0)
    assert np.array_equal(kl[0, :16], lat[0, 0, :, 0])         # latent rows untouched (bf16)
    kc, ks = quantize_rows_e4m3(k)
    assert np.array_equal(kl[0, 16:], dequantize_rows_e4m3(kc, ks)[0, :, 0])
    assert not np.array_equal(kl[0, 16:], k[0, :, 0])          # tokens really are quantized
    codes = c.token_codes(0, 0)
    assert len(codes) == 1 and np.array_equal(codes[0][0], kc[0])
    # compress moves the trailing m token rows into a bf16 latent set: bf16(fp32(code) * scale)
    c.compress(0, 24, 16)
    kl2, _ = c.logical_kv(0, 0)
    assert kl2.shape[1] == 32
    exp = bf16_round(e4m3_values()[kc[0, 24:, 0]].astype(np.float32) * ks[0, 24:, 0][:, None])
    assert np.array_equal(kl2[0, 16:], exp)


# --------------------------------------------------------------------------- bf16 rounding
def _bf16_rne_bits(x32: float) -> float:
    """Independent fp32 -> bf16 round-to-nearest-even on the bit pattern (pure Python):
    keep the upper 16 bits after adding 0x7FFF + (bit 16), the textbook RNE carry trick;
    NaN stays NaN (quieted), +-inf stay +-inf, overflow past the largest bf16 gives inf."""
    import struct
    u = struct.unpack("<I", struct.pack("<f", x32))[0]
    if (u & 0x7F800000) == 0x7F800000 and (u & 0x007FFFFF):       # NaN
        return float("nan")
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    return struct.unpack("<f", struct.pack("<I", u & 0xFFFFFFFF))[0]


def test_bf16_round_matches_bit_level_rne():
    """Pins oracle.bf16_round (used by the fp8 -> bf16 latent conversion of compress,
    reading A20) against the bit-level RNE definition: ties to even in both directions,
    subnormals, the overflow edge, +-inf, NaN, signed zero, and random fp32 values.
    A truncating or ties-away rounding fails the tie rows."""
    import struct
    from oracle import bf16_round

    def f32(bits):
        return struct.unpack("<f", struct.pack("<I", bits))[0]

    ulp = 2.0 ** -7
    hand = [  # (input, expected) fixed by the format: 7 stored mantissa bits
        (1.0 + ulp / 2, 1.0),                      # tie, lower neighbour even
        (1.0 + 3 * ulp / 2, 1.0 + 2 * ulp),        # tie, upper neighbour even
        (-(1.0 + 3 * ulp / 2), -(1.0 + 2 * ulp)),
        (1.0 + ulp / 2 + 2.0 ** -20, 1.0 + ulp),   # just above a tie
        (1.0 + ulp / 2 - 2.0 ** -20, 1.0),         # just below a tie
    ]
    for x, want in hand:
        assert bf16_round(np.array([x]))[0] == want, (x, want)
    edge_bits = [0x00000000, 0x80000000, 0x00000001, 0x00008000, 0x00018000, 0x00008001,
                 0x007FFFFF, 0x00800000, 0x3F808000, 0x3F818000, 0x7F7F7FFF, 0x7F7F8000,
                 0x7F7FFFFF, 0xFF7FFFFF, 0x7F800000, 0xFF800000, 0x3F800000, 0xC0490FDB]
    rng = np.random.default_rng(11)
    rand_bits = [int(b) for b in rng.integers(0, 2 ** 32, 4000, dtype=np.uint64)]
    rand_bits = [b for b in rand_bits if not ((b & 0x7F800000) == 0x7F800000 and b & 0x7FFFFF)]
    bits = edge_bits + rand_bits
    xs = np.array([f32(b) for b in bits], dtype=np.float32)
    got = bf16_round(xs)
    want = np.array([_bf16_rne_bits(float(x)) for x in xs])
    assert np.array_equal(got, want)
    assert np.array_equal(np.signbit(got), np.signbit(want))      # -0 stays -0
    assert np.isnan(bf16_round(np.array([np.nan], dtype=np.float32))[0])
    # the checker itself distinguishes RNE from truncation and from ties-away
    assert _bf16_rne_bits(f32(0x3F808000)) == 1.0                 # tie -> even (down)
    assert _bf16_rne_bits(f32(0x3F818000)) == f32(0x3F820000)     # tie -> even (up)
    assert math.isinf(_bf16_rne_bits(f32(0x7F7FFFFF)))


def test_fp8_staged_logical_kv_is_the_compress_conversion():
    """logical_kv(fp8_staged=True) (the rows prefill attends over, reading A20) equals, row by
    row, the bf16 latent rows that compress produces from the same fp8 token rows (the
    conversion pinned bit-exact against the GPU in test_gpu_fp8.py), and leaves latent rows
    and the default (decode) view unchanged."""
    from oracle import OracleCache
    rng = np.random.default_rng(12)
    c = OracleCache(1, 2, 1, 64, 16, token_fp8=True)
    c.create_seq(0)
    lat = _bf16(rng.standard_normal((1, 2, 16, 1, 64)))
    c.install(0, -1, lat)
    k, v = _bf16(rng.standard_normal((1, 40, 1, 64)) * 300), _bf16(rng.standard_normal((1, 40, 1, 64)))
    c.append(0, k, v)
    ks, vs = c.logical_kv(0, 0, fp8_staged=True)
    kd, vd = c.logical_kv(0, 0)
    assert np.array_equal(ks[:, :16], kd[:, :16]) and np.array_equal(vs[:, :16], vd[:, :16])
    assert not np.array_equal(ks, kd)                              # staging really rounds
    assert np.all(np.abs(ks - kd) <= 2.0 ** -8 * np.abs(kd))      # by at most a bf16 half-ulp
    c.compress(0, 0, 40)                                           # the 40 token rows -> a latent set
    kc, vc = c.logical_kv(0, 0)
    assert np.array_equal(kc[:, 16:], ks[:, 16:]) and np.array_equal(vc[:, 16:], vs[:, 16:])
