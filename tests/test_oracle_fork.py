"""Pins for OracleCache.fork (prefix sharing, "prefix KV cache
for user prompts", reading A21) against things other than itself (CPU only):
  * a forked sequence + later ops == a sequence built from scratch with the same op script
    (independent construction: same logical K/V, same expected block table, same attention);
  * attention after fork + append == torch fp64 SDPA with an explicit bottom-right mask over
    the concatenation [prefix rows, appended rows];
  * isolation: ops on the source after the fork leave the fork unchanged and vice versa;
  * the invalid cuts (inside a latent set, beyond the length) raise."""
import numpy as np
import pytest
import torch

from oracle import OracleCache, attend, expected_table
from workloads import Draw, Shape

SH = Shape(1, 4, 2, 32, 16)


def f64(t):
    return t.to(torch.float64).numpy()


def _script_rows(d, script):
    """Draw the rows of a script once: list of (kind, k, v) with k, v [L][n][H][d] fp64."""
    out = []
    for kind, n in script:
        if kind == "latent":
            kv = f64(d.latent(SH, n))
            out.append((kind, kv[:, 0], kv[:, 1]))
        else:
            k, v = d.tokens(SH, n)
            out.append((kind, f64(k), f64(v)))
    return out


def _replay(c, s, rows):
    for kind, k, v in rows:
        if kind == "latent":
            c.install(s, -1, np.stack([k, v], 1))
        else:
            c.append(s, k, v)


def _cut(rows, n):
    """The first n logical rows of a drawn script as a script of its own (token cut only)."""
    out, left = [], n
    for kind, k, v in rows:
        if left == 0:
            break
        take = min(left, k.shape[1])
        out.append((kind, k[:, :take], v[:, :take]))
        left -= take
    return out


@pytest.mark.parametrize("cut", [0, 16, 23, 40, 41, 64, 65, 100, 104])
def test_fork_plus_ops_equals_scratch_build(cut):
    d = Draw(3)
    rows = _script_rows(d, [("latent", 16), ("tokens", 25), ("latent", 23), ("tokens", 40)])
    c = OracleCache(1, SH.num_q_heads, SH.num_kv_heads, SH.head_dim, SH.page_size)
    c.create_seq(0)
    _replay(c, 0, rows)
    c.fork(0, cut, 1)
    extra_k, extra_v = (f64(x) for x in d.tokens(SH, 19))
    c.append(1, extra_k, extra_v)
    # independent construction: a fresh cache fed the cut script and the same appended rows
    r = OracleCache(1, SH.num_q_heads, SH.num_kv_heads, SH.head_dim, SH.page_size)
    r.create_seq(7)
    _replay(r, 7, _cut(rows, cut))
    r.append(7, extra_k, extra_v)
    ka, va = c.logical_kv(1, 0)
    kb, vb = r.logical_kv(7, 0)
    assert np.array_equal(ka, kb) and np.array_equal(va, vb)
    assert c.expected_table(1) == r.expected_table(7)
    assert c.seq_len(1) == cut + 19 and c.latent_rows(1) == r.latent_rows(7)
    q = f64(d.queries(SH, 5))
    assert np.array_equal(attend(q, ka, va, SH.scale), attend(q, kb, vb, SH.scale))
    # set ids continue from the source's counter: a new set gets id 2 (the source has 0 and 1)
    assert c.install(1, -1, np.zeros((1, 2, 3, SH.num_kv_heads, SH.head_dim))) == 2


def test_fork_attention_matches_sdpa_over_prefix_plus_new_rows():
    d = Draw(4)
    c = OracleCache(1, SH.num_q_heads, SH.num_kv_heads, SH.head_dim, SH.page_size)
    c.create_seq(0)
    rows = _script_rows(d, [("latent", 32), ("tokens", 70)])
    _replay(c, 0, rows)
    c.fork(0, 32 + 50, 5)
    nk, nv = (f64(x) for x in d.tokens(SH, 12))
    c.append(5, nk, nv)
    K = np.concatenate([rows[0][1][0], rows[1][1][0, :50], nk[0]], 0)    # [Lb][H][d]
    V = np.concatenate([rows[0][2][0], rows[1][2][0, :50], nv[0]], 0)
    lb = K.shape[0]
    tq = 7
    q = f64(d.queries(SH, tq))
    G = SH.num_q_heads // SH.num_kv_heads
    Kt = torch.from_numpy(K).permute(1, 0, 2).repeat_interleave(G, 0)      # [Hq][Lb][d]
    Vt = torch.from_numpy(V).permute(1, 0, 2).repeat_interleave(G, 0)
    Qt = torch.from_numpy(q).permute(1, 0, 2)                              # [Hq][Tq][d]
    mask = torch.ones(tq, lb, dtype=torch.bool).tril(diagonal=lb - tq)    # bottom-right causal
    ref = torch.nn.functional.scaled_dot_product_attention(Qt, Kt, Vt, attn_mask=mask, scale=SH.scale)
    got = attend(q, *c.logical_kv(5, 0), SH.scale)
    assert np.max(np.abs(got - ref.permute(1, 0, 2).numpy())) <= 1e-12


def test_fork_isolation_both_ways():
    d = Draw(5)
    c = OracleCache(1, SH.num_q_heads, SH.num_kv_heads, SH.head_dim, SH.page_size)
    c.create_seq(0)
    _replay(c, 0, _script_rows(d, [("tokens", 30), ("latent", 16), ("tokens", 9)]))
    c.fork(0, 55, 1)
    c.fork(0, 20, 2)
    k1 = [x.copy() for x in c.logical_kv(1, 0)]
    k2 = [x.copy() for x in c.logical_kv(2, 0)]
    c.append(0, *(f64(x) for x in d.tokens(SH, 4)))
    c.install(0, 0, f64(d.latent(SH, 16)))                 # replace the shared set in the source
    assert all(np.array_equal(a, b) for a, b in zip(k1, c.logical_kv(1, 0)))
    assert all(np.array_equal(a, b) for a, b in zip(k2, c.logical_kv(2, 0)))
    src = [x.copy() for x in c.logical_kv(0, 0)]
    c.append(2, *(f64(x) for x in d.tokens(SH, 3)))
    c.release(1)
    assert all(np.array_equal(a, b) for a, b in zip(src, c.logical_kv(0, 0)))
    assert expected_table([("token", 23)], SH.page_size) == c.expected_table(2)


def test_fork_invalid_cuts():
    d = Draw(6)
    c = OracleCache(1, SH.num_q_heads, SH.num_kv_heads, SH.head_dim, SH.page_size)
    c.create_seq(0)
    _replay(c, 0, _script_rows(d, [("tokens", 10), ("latent", 16), ("tokens", 5)]))
    with pytest.raises(ValueError):
        c.fork(0, 11, 1)          # inside the latent set
    with pytest.raises(ValueError):
        c.fork(0, 32, 1)          # beyond the length
    c.fork(0, 26, 1)              # right after the set: fine
    assert c.seq_len(1) == 26
    with pytest.raises(KeyError):
        c.fork(0, 1, 1)           # dst exists
