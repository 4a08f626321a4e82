"""NEXT-2 prefix sharing (hpa_seq_fork; "prefix KV cache for user prompts"; DESIGN.md
reading A21) through the C ABI, against the oracle's fork (pinned in test_oracle_fork.py).

Checks: after fork -> appends on either side (copy-on-write of a shared partial page, or
in-place when the appender owns the page's claimed rows) -> latent replacement -> release in
any order: every live sequence's logical K/V is bit-exact three ways (oracle model, export
kernel, physical pool dump walked through the exported table), its table equals the expected
table, decode and prefill match the oracle, pages are shared (the pool's used-page count is
the number of DISTINCT referenced pages), and releasing everything returns every page."""
import random

import numpy as np
import pytest
import torch

from oracle import attend, gather_physical
from oracle.hpa_oracle import META_LATENT_BIT
from tests.hpa_testutil import Pair, check_close, f64
from workloads import Shape


def _valid_cuts(orc, s):
    """Fork cuts the reading allows: 0..len except strictly inside a latent set."""
    cuts, pos = [0], 0
    for sg in orc.seqs[s]:
        if sg.kind == "token":
            cuts += list(range(pos + 1, pos + sg.rows + 1))
        else:
            cuts.append(pos + sg.rows)
        pos += sg.rows
    return sorted(set(cuts))


def _fork(p, src, n):
    d = p.cache.seq_fork(src, n)
    p.orc.fork(src, n, d)
    return d


def _distinct_pages(p, live):
    pages = set()
    for s in live:
        pg, _, _ = p.cache.export_table(s)
        pages |= set(int(x) for x in pg)
    return pages


def _check_views(p, live, layer=0):
    torch.cuda.synchronize()
    kp, vp = p.cache.pools()
    kp, vp = f64(kp), f64(vp)
    for s in live:
        k1, v1 = p.orc.logical_kv(s, layer)
        k2, v2 = p.cache.export_logical_kv(layer, s)
        assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2)), s
        pages, pos0, meta = p.cache.export_table(s)
        k3, v3 = gather_physical(kp, vp, [int(x) for x in pages], [int(m) for m in meta], layer)
        assert np.array_equal(k1, k3) and np.array_equal(v1, v3), s
        assert [(("latent" if m & META_LATENT_BIT else "token"), int(m & 0x7fff), int(x))
                for m, x in zip(meta, pos0)] == p.orc.expected_table(s)


def _check_attention(p, live, tag, qmax=200):
    alive = [s for s in live if p.orc.seq_len(s) > 0]
    if not alive:
        return
    q = p.queries(len(alive))
    got = p.cache.decode(0, alive, q.cuda())
    torch.cuda.synchronize()
    ref = np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, 0), p.shape.scale)[0] for i, s in enumerate(alive)])
    check_close(got, ref, f"{tag} decode")
    q_lens = [min(qmax, p.orc.seq_len(s)) for s in alive]
    qp = p.queries(sum(q_lens))
    got = p.cache.prefill(0, alive, q_lens, qp.cuda())
    torch.cuda.synchronize()
    off, ref = 0, []
    for s, n in zip(alive, q_lens):
        ref.append(attend(f64(qp[off:off + n]), *p.orc.logical_kv(s, 0), p.shape.scale))
        off += n
    check_close(got, np.concatenate(ref), f"{tag} prefill")


@pytest.mark.gpu
@pytest.mark.parametrize("P", [16, 64])
def test_fork_cuts_cow_and_release_any_order(P):
    shape = Shape(1, 8, 2, 128, P)
    p = Pair(shape, num_pages=400, max_seqs=12, max_pages_per_seq=128)
    src = p.build([("latent", 40), ("tokens", 3 * P + 5), ("latent", 128), ("tokens", 2 * P + 7)])
    L = p.orc.seq_len(src)
    cuts = [0, 40, 41, 40 + P, 40 + 2 * P + 3, 40 + 3 * P + 5, 40 + 3 * P + 5 + 128, L - 1, L]
    forks = [_fork(p, src, n) for n in cuts]
    live = [src] + forks
    used_before = p.cache.stats()[1]
    # the forks add no pages: every referenced page is one of src's
    assert _distinct_pages(p, live) == _distinct_pages(p, [src])
    _check_views(p, live)
    # appends in one call: src first (owns its last page's rows: in place), then forks cut at
    # the same length (one claims in place), forks cut mid-page (copy-on-write)
    p.tokens(live, [3] * len(live))
    _check_views(p, live)
    _check_attention(p, live, f"fork P={P} after appends")
    assert p.cache.stats()[1] > used_before                 # copies were made
    # replace the shared latent set in one fork (copy-on-write of latent pages) and append more
    f = forks[-1]
    p.latent(f, 128, set_id=1)
    p.tokens([forks[4], src], [P + 1, 2])
    _check_views(p, live)
    _check_attention(p, live, f"fork P={P} after replace")
    # release in a scrambled order, checking the survivors each time
    order = live[:]
    random.Random(P).shuffle(order)
    for s in order:
        p.cache.seq_release(s)
        p.orc.release(s)
        live.remove(s)
        _check_views(p, live)
        free, used, _ = p.cache.stats()
        assert used == len(_distinct_pages(p, live)) and free + used == 400
    assert p.cache.stats()[:2] == (400, 0)


@pytest.mark.gpu
def test_fork_errors_leave_cache_unchanged():
    from paper_2605_09100_b200 import HPAError
    shape = Shape(1, 4, 1, 64, 16)
    p = Pair(shape, num_pages=64, max_seqs=2, max_pages_per_seq=32)
    s = p.build([("tokens", 20), ("latent", 16), ("tokens", 5)])
    before = (p.cache.stats(), p.cache.export_table(s))
    for bad in (-1, 42, 25):                                  # < 0, > len, inside the latent set
        with pytest.raises(HPAError) as e:
            p.cache.seq_fork(s, bad)
        assert e.value.name == "HPA_ERR_INVALID_ARG"
    with pytest.raises(HPAError) as e:
        p.cache.seq_fork(99, 1)
    assert e.value.name == "HPA_ERR_UNKNOWN_SEQ"
    d = _fork(p, s, 36)                                       # the second and last slot
    with pytest.raises(HPAError) as e:
        p.cache.seq_fork(s, 3)
    assert e.value.name == "HPA_ERR_SEQ_CAPACITY"
    p.cache.seq_release(d)
    p.orc.release(d)
    after = (p.cache.stats(), p.cache.export_table(s))
    assert before[0] == after[0] and all(np.array_equal(a, b) for a, b in zip(before[1], after[1]))
    _check_views(p, [s])


@pytest.mark.gpu
def test_fork_fp8_token_pages_cow_bit_exact():
    """fp8 token pages (NEXT-4c): the copy-on-write copies the 16-row code/scale blocks raw; the
    stored codes of every sequence stay bit-exact and decode matches the oracle."""
    shape = Shape(2, 8, 2, 128, 16)
    p = Pair(shape, num_pages=256, max_seqs=6, max_pages_per_seq=64, token_fp8=True, num_token_pages=256)
    src = p.build([("latent", 32), ("tokens", 45)])
    a = _fork(p, src, 32 + 40)
    b = _fork(p, src, 32 + 45)
    p.tokens([src, a, b], [4, 9, 2])                          # src in place, a and b copy
    torch.cuda.synchronize()
    k8, v8, ks, vs, _ = p.cache.token_pool()
    k8, v8, ks, vs = k8.cpu().numpy(), v8.cpu().numpy(), ks.cpu().numpy(), vs.cpu().numpy()
    for s in (src, a, b):
        for layer in range(2):
            segs = p.orc.token_codes(s, layer)
            exp = [np.concatenate([g[i] for g in segs]) for i in range(4)]
            pages, _, meta = p.cache.export_table(s)
            got = [[], [], [], []]
            for pg, m in zip(pages, meta):
                if int(m) & META_LATENT_BIT:
                    continue
                n = int(m) & 0x7fff
                got[0].append(k8[layer, pg, :, :n].transpose(1, 0, 2))
                got[1].append(ks[layer, pg, :, :n].T)
                got[2].append(v8[layer, pg, :, :n].transpose(1, 0, 2))
                got[3].append(vs[layer, pg, :, :n].T)
            for i in range(4):
                assert np.array_equal(np.concatenate(got[i]), exp[i]), (s, layer, i)
    for layer in (0, 1):
        q = p.queries(3)
        out = p.cache.decode(layer, [src, a, b], q.cuda())
        ref = np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, layer), shape.scale)[0]
                        for i, s in enumerate([src, a, b])])
        check_close(out, ref, f"fp8 fork decode layer {layer}")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(2))
def test_fork_ops_fuzz(seed):
    """300 random ops mixing fork with append / install / replace / remove / compress /
    release; views bit-exact and page accounting exact every 30 ops, attention every 60."""
    from paper_2605_09100_b200 import HPAError
    rng = random.Random(100 + seed)
    shape = Shape(1, 8, 2, 128, rng.choice([16, 32]))
    p = Pair(shape, num_pages=900, max_seqs=8, max_pages_per_seq=200, seed=seed)
    live = []
    for step in range(300):
        op = rng.random()
        try:
            if op < 0.08 and len(live) < 8:
                live.append(p.new_seq())
            elif op < 0.22 and live and len(live) < 8:
                s = rng.choice(live)
                live.append(_fork(p, s, rng.choice(_valid_cuts(p.orc, s))))
            elif op < 0.55 and live:
                ss = rng.sample(live, rng.randint(1, len(live)))
                p.tokens(ss, [rng.randint(1, 40) for _ in ss])
            elif op < 0.70 and live:
                s = rng.choice(live)
                ids = [sg.set_id for sg in p.orc.seqs[s] if sg.kind == "latent"]
                sid = rng.choice(ids) if ids and rng.random() < 0.5 else -1
                p.latent(s, rng.choice([8, 16, 40, 128]), set_id=sid)
            elif op < 0.76 and live:
                s = rng.choice(live)
                ids = [sg.set_id for sg in p.orc.seqs[s] if sg.kind == "latent"]
                if ids:
                    sid = rng.choice(ids)
                    p.cache.latent_remove(s, sid)
                    p.orc.remove(s, sid)
            elif op < 0.84 and live:
                s = rng.choice(live)
                segs = p.orc.seqs[s]
                if segs and segs[-1].kind == "token" and segs[-1].rows >= 12:
                    m = rng.randint(1, 8)
                    n_doc = rng.randint(0, segs[-1].rows - m)
                    assert p.cache.compress(s, n_doc, m) == p.orc.compress(s, n_doc, m)
            elif op < 0.92 and live:
                s = live.pop(rng.randrange(len(live)))
                p.cache.seq_release(s)
                p.orc.release(s)
        except HPAError as e:
            assert e.name in ("HPA_ERR_OUT_OF_PAGES", "HPA_ERR_SEQ_CAPACITY"), e
        if step % 30 == 29:
            _check_views(p, live)
            free, used, nlive = p.cache.stats()
            assert used == len(_distinct_pages(p, live)) and free + used == 900 and nlive == len(live)
        if step % 60 == 59:
            _check_attention(p, live, f"fork fuzz seed {seed} step {step}", qmax=64)
