"""Property-based pins of the oracle (hypothesis; CPU, `-m "not gpu"`).

Each property is an identity that holds for any input, so a plausible slip in the
oracle (a dropped term, an off-by-one in a cut, a wrong reduction axis) fails it on some
generated case:
  * partial attention over any cut of the keys + LSE merge == attention over all keys
    (SURVEY 8(f) NEXT-4b; the LSE algebra of P:L248-251's softmax);
  * attention with no mask is invariant to permuting the keys (with their values);
  * the e4m3 row quantizer (A20) is idempotent: re-quantizing dequantized rows
    reproduces the codes and scales exactly;
  * table pos0 is the prefix sum of valid rows, every segment starts on a fresh page and
    only a segment's last page may be partial (reading A7).
"""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import (attend, dequantize_rows_e4m3, expected_table, merge_partials, partial_attend,
                    quantize_rows_e4m3)

SET = settings(max_examples=25, deadline=None)


@SET
@given(st.integers(1, 4), st.integers(1, 3), st.integers(2, 70), st.integers(0, 2 ** 31 - 1),
       st.lists(st.floats(0.0, 1.0), min_size=0, max_size=3))
def test_partials_merge_to_full_attention(g, hkv, n, seed, cuts):
    rng = np.random.default_rng(seed)
    d = 16
    q = rng.standard_normal((hkv * g, d))
    k = rng.standard_normal((hkv, n, d)) * 2.0
    v = rng.standard_normal((hkv, n, d))
    edges = sorted({0, n, *[int(c * n) for c in cuts]})
    parts = [partial_attend(q, k[:, a:b], v[:, a:b], 0.3) for a, b in zip(edges[:-1], edges[1:]) if b > a]
    merged = merge_partials(np.stack([p[0] for p in parts]), np.stack([p[1] for p in parts]))
    full = attend(q[None], k, v, 0.3)[0]
    np.testing.assert_allclose(merged, full, rtol=1e-11, atol=1e-12)


@SET
@given(st.integers(1, 40), st.integers(0, 2 ** 31 - 1))
def test_unmasked_attention_is_key_permutation_invariant(n, seed):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((1, 4, 8))
    k = rng.standard_normal((2, n, 8))
    v = rng.standard_normal((2, n, 8))
    perm = rng.permutation(n)
    a = attend(q, k, v, 0.5)
    b = attend(q, k[:, perm], v[:, perm], 0.5)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13)


@SET
@given(st.integers(1, 6), st.integers(0, 2 ** 31 - 1), st.floats(1e-3, 50.0))
def test_e4m3_row_quantizer_is_idempotent(rows, seed, spread):
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((rows, 64)) * spread).astype(np.float32)
    codes, s = quantize_rows_e4m3(x)
    x2 = dequantize_rows_e4m3(codes, s).astype(np.float32)
    codes2, s2 = quantize_rows_e4m3(x2)
    assert np.array_equal(s, s2)
    assert np.array_equal(codes, codes2)


@SET
@given(st.lists(st.tuples(st.sampled_from(["latent", "token"]), st.integers(1, 90)), min_size=1, max_size=8),
       st.sampled_from([16, 32, 64]))
def test_table_pos0_is_prefix_sum_and_pages_start_fresh(segments, P):
    # merge adjacent token segments the way append does (one trailing token segment)
    segs = []
    for kind, n in segments:
        if segs and kind == "token" and segs[-1][0] == "token":
            segs[-1] = ("token", segs[-1][1] + n)
        else:
            segs.append((kind, n))
    table = expected_table(segs, P)
    pos = 0
    i = 0
    for kind, n in segs:
        npages = -(-n // P)
        rows = [table[i + j][1] for j in range(npages)]
        assert all(r == P for r in rows[:-1]) and 1 <= rows[-1] <= P and sum(rows) == n
        for j in range(npages):
            assert table[i + j][0] == kind and table[i + j][2] == pos
            pos += table[i + j][1]
        i += npages
    assert i == len(table) and pos == sum(n for _, n in segs)
