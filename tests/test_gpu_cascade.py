"""NEXT-2 cascade decode ("prefix KV cache for user prompts"; P:L63
shared document memories) through the C ABI.

Requests whose block tables begin with the same page run -- prompt prefixes shared by
hpa_seq_fork, latent sets shared by hpa_latent_set_share and installed first -- are decoded as
group units (the run read once for up to 32/G requests) plus per-request units over the rest,
merged by the LSE combine. The oracle knows nothing about this: every output is compared with
the plain definition (oracle.attend over the oracle's logical K/V of each request, fp64), and
the plan introspection (hpa_decode_plan_info) proves the group units ran. Cascade off vs on
must agree to fp32 rounding."""
import numpy as np
import pytest
import torch

from oracle import attend
from tests.hpa_testutil import Pair, check_close, f64
from workloads import Shape

pytestmark = pytest.mark.gpu


def _shape(hq, hkv, d, P, L=2):
    return Shape(num_layers=L, num_q_heads=hq, num_kv_heads=hkv, head_dim=d, page_size=P)


def _fork(p, src, n):
    d = p.cache.seq_fork(src, n)
    p.orc.fork(src, n, d)
    return d


def _valid_cuts(orc, s):
    """Fork cuts the reading allows (A21): any row boundary except strictly inside a latent set."""
    cuts, pos = [0], 0
    for sg in orc.seqs[s]:
        if sg.kind == "token":
            cuts += list(range(pos + 1, pos + sg.rows + 1))
        else:
            cuts.append(pos + sg.rows)
        pos += sg.rows
    return sorted(set(cuts))


def _ref(p, seqs, q, layer):
    return np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, layer), p.shape.scale)[0]
                     for i, s in enumerate(seqs)])


def _decode_both(p, seqs, q, layer, what):
    """Cascade on (must plan group units) and off; both against the oracle, and each other."""
    p.cache.set_decode_cascade(True)
    on = p.cache.decode(layer, seqs, q.cuda())
    torch.cuda.synchronize()
    info = p.cache.decode_plan_info()
    p.cache.set_decode_cascade(False)
    off = p.cache.decode(layer, seqs, q.cuda())
    torch.cuda.synchronize()
    assert p.cache.decode_plan_info()["group_units"] == 0
    p.cache.set_decode_cascade(True)
    ref = _ref(p, seqs, q, layer)
    check_close(on, ref, f"{what} cascade")
    check_close(off, ref, f"{what} plain")
    # both bf16 outputs of fp32 results that differ only in summation order
    d = np.abs(f64(on) - f64(off)).max()
    assert d <= 2.0 ** -7 * (1.0 + np.abs(f64(off)).max()), (what, d)
    return info


@pytest.mark.parametrize("hq,hkv,d,P", [(32, 8, 128, 16), (16, 2, 128, 32), (8, 8, 64, 16),
                                        (16, 2, 64, 64), (8, 1, 128, 16)])
def test_cascade_forked_prompt(hq, hkv, d, P):
    """n requests forked from one prompt (latent set + tokens, cut inside a page), each with
    its own continuation; group sizes 32/G -> several groups and a remainder."""
    shape = _shape(hq, hkv, d, P)
    G = hq // hkv
    p = Pair(shape, 4096, 40, 400, seed=11)
    src = p.build([("latent", 128), ("tokens", 40 * P + 5)])
    n = 32 // G + 3  # one full group + a partial one
    seqs = []
    for i in range(n):
        s = _fork(p, src, 128 + 40 * P + 5)
        p.tokens([s], [1 + (7 * i) % (3 * P)])  # own rows: copy-on-write of the shared partial page
        seqs.append(s)
    q = p.queries(n)
    for layer in (0, 1):
        info = _decode_both(p, seqs, q, layer, f"fork hq={hq} hkv={hkv} d={d} P={P} L={layer}")
        assert info["group_units"] > 0, info


def test_cascade_mixed_batch_and_growth():
    """Forks of two prompts, unrelated requests, a request that IS the shared prefix (no own
    rows), a short shared run below the cascade threshold; then steps of appends (the plan is
    rebuilt as own runs grow, and when the prefix owner's partial last page grows)."""
    shape = _shape(32, 8, 128, 16)
    p = Pair(shape, 8192, 48, 600, seed=5)
    a = p.build([("tokens", 700)])
    b = p.build([("latent", 256), ("tokens", 333)])
    lone = p.build([("tokens", 900)])
    short = p.build([("tokens", 40)])
    seqs = [a, b, lone, short]
    for i in range(9):
        seqs.append(_fork(p, a, 700 - 16 * (i % 3)))    # different cut points: LCP differs
    for i in range(5):
        seqs.append(_fork(p, b, 256 + 333))
    seqs.append(_fork(p, short, 40))                     # a 3-chunk run: below the threshold
    for i, s in enumerate(seqs[4:]):
        p.tokens([s], [3 + i])
    for step in range(4):
        q = p.queries(len(seqs))
        info = _decode_both(p, seqs, q, step % 2, f"mixed step {step}")
        assert info["group_units"] > 0, info
        p.tokens(seqs, [1 + (step * 5 + i) % 17 for i in range(len(seqs))])


def test_cascade_shared_latent_sets():
    """Document memories shared by many requests (hpa_latent_set_share), installed first, then
    each request's own tokens; one request also has a private set in between."""
    shape = _shape(32, 8, 128, 16)
    p = Pair(shape, 8192, 40, 300, seed=9)
    owner = p.new_seq()
    set0 = p.latent(owner, 128)
    set1 = p.latent(owner, 96)
    seqs = []
    for i in range(12):
        s = p.new_seq()
        for sid in (set0, set1):
            got = p.cache.latent_share(s, owner, sid)
            assert got == p.orc.share(s, owner, sid)
        if i == 3:
            p.latent(s, 64)
        p.tokens([s], [50 + 13 * i])
        seqs.append(s)
    q = p.queries(len(seqs))
    info = _decode_both(p, seqs, q, 0, "shared sets")
    assert info["group_units"] > 0, info


def test_cascade_forced_splits_and_partial_api():
    """Group units next to forced own splits, and through hpa_decode_partial (fp32 O + LSE of the
    whole request) and hpa_append_decode (which then takes the two-launch path)."""
    shape = _shape(16, 4, 128, 16)
    p = Pair(shape, 4096, 24, 400, seed=21)
    src = p.build([("tokens", 1500)])
    seqs = [src] + [_fork(p, src, 1500) for _ in range(9)]
    for i, s in enumerate(seqs):
        p.tokens([s], [20 + 37 * i])
    p.cache.set_decode_splits(3)
    q = p.queries(len(seqs))
    info = _decode_both(p, seqs, q, 0, "forced splits")
    assert info["group_units"] > 0 and info["splits"] >= 4, info
    p.cache.set_decode_splits(0)
    o, lse = p.cache.decode_partial(0, seqs, q.cuda())
    torch.cuda.synchronize()
    assert p.cache.decode_plan_info()["group_units"] > 0
    check_close(o, _ref(p, seqs, q, 0), "partial O")
    # append + decode in one call == append, then decode
    k, v = p.draw.tokens(shape, len(seqs))
    out = torch.empty((len(seqs), 16, 128), dtype=torch.bfloat16, device="cuda")
    p.cache.append_decode(1, seqs, k.cuda(), v.cuda(), q.cuda(), out)
    for i, s in enumerate(seqs):
        p.orc.append(s, f64(k[:, i:i + 1]), f64(v[:, i:i + 1]))
    torch.cuda.synchronize()
    assert p.cache.decode_plan_info()["group_units"] > 0
    check_close(out, _ref(p, seqs, q, 1), "append_decode cascade")


@pytest.mark.parametrize("hq,hkv,d,P", [(32, 8, 128, 16), (16, 2, 64, 32), (8, 1, 128, 64)])
def test_cascade_fp8_token_pages(hq, hkv, d, P):
    """fp8 token pages (NEXT-4c) with a forked prompt: group units on the 32-row fp8 kernel,
    latent (bf16) and token (fp8) chunks in the shared run, own fp8 rows after it."""
    shape = _shape(hq, hkv, d, P)
    G = hq // hkv
    p = Pair(shape, 2048, 24, 300, seed=3, token_fp8=True, num_token_pages=2048)
    src = p.build([("latent", 64), ("tokens", 20 * P + 7)])
    seqs = [src] + [_fork(p, src, 64 + 20 * P + 7) for _ in range(32 // G + 2)]
    for i, s in enumerate(seqs):
        p.tokens([s], [1 + (5 * i) % (2 * P)])
    q = p.queries(len(seqs))
    for layer in (0, 1):
        info = _decode_both(p, seqs, q, layer, f"fp8 forks hq={hq} hkv={hkv} d={d} P={P} L={layer}")
        assert info["group_units"] > 0, info


def test_cascade_none_without_sharing():
    """A batch without two requests sharing a first page plans no group units."""
    p2 = Pair(_shape(32, 8, 128, 16), 2048, 12, 300, seed=4)
    seqs2 = [p2.build([("tokens", 300 + 50 * i)]) for i in range(5)]
    q2 = p2.queries(5)
    out2 = p2.cache.decode(0, seqs2, q2.cuda())
    torch.cuda.synchronize()
    assert p2.cache.decode_plan_info()["group_units"] == 0
    check_close(out2, _ref(p2, seqs2, q2, 0), "no sharing")


def test_cascade_fuzz():
    """Random fork trees (forks of forks at random cuts), random own growth and batch subsets,
    cascade on vs off vs oracle."""
    rng = np.random.default_rng(1234)
    shape = _shape(32, 8, 128, 16)
    p = Pair(shape, 16384, 64, 800, seed=77)
    roots = [p.build([("latent", 128), ("tokens", int(rng.integers(200, 1200)))]) for _ in range(3)]
    live = list(roots)
    for _ in range(30):
        src = int(rng.choice(live))
        L = p.orc.seq_len(src)
        cut = int(rng.integers(129, L + 1))
        s = _fork(p, src, cut)
        p.tokens([s], [int(rng.integers(1, 40))])
        live.append(s)
    for it in range(6):
        batch = sorted(rng.choice(live, size=int(rng.integers(8, len(live))), replace=False).tolist())
        q = p.queries(len(batch))
        _decode_both(p, batch, q, it % 2, f"fuzz {it}")
        grow = [s for s in live if rng.random() < 0.5]
        p.tokens(grow, [int(rng.integers(1, 30)) for _ in grow])


@pytest.mark.parametrize("seed,hq,hkv,d,P,fp8,need", [(0, 16, 4, 128, 16, False, True), (1, 16, 4, 128, 16, False, True),
                                                       (2, 8, 8, 64, 32, False, True), (3, 32, 4, 128, 64, False, False),
                                                       (4, 16, 4, 128, 16, True, False), (5, 8, 1, 128, 16, True, True)])
def test_cascade_step_fuzz(seed, hq, hkv, d, P, fp8, need):
    """200 random ops on a fork tree -- forks at random cuts, fused decode steps
    (hpa_append_decode) on random subsets, bulk appends, latent replacement in forked requests
    (copy-on-write of shared latent pages) or new latent sets, releases -- with cascade decode vs
    plain vs the oracle every 20 ops; in most cases the cascade must have run in some checks."""
    import random

    from paper_2605_09100_b200 import HPAError
    import os
    rng = random.Random(700 + seed)
    shape = _shape(hq, hkv, d, P, L=1)
    p = Pair(shape, 6000, 24, 4800 // P, seed=seed, token_fp8=fp8, num_token_pages=6000 if fp8 else 0)
    if os.environ.get("HPA_TEST_CASCADE_OFF"):
        p.cache.set_decode_cascade(False)
    roots = [p.build([("latent", 128), ("tokens", rng.randint(300, 900))]) for _ in range(2)]
    live = list(roots)
    grouped = 0
    for step in range(200):
        op = rng.random()
        try:
            if op < 0.25 and len(live) < 24:
                src = rng.choice(live)
                cuts = [c for c in _valid_cuts(p.orc, src) if c > 128]
                if cuts:
                    live.append(_fork(p, src, rng.choice(cuts)))
            elif op < 0.55 and live:
                ss = sorted(rng.sample(live, rng.randint(1, len(live))))
                k, v = p.draw.tokens(shape, len(ss))
                q = p.queries(len(ss))
                out = p.cache.append_decode(0, ss, k.cuda(), v.cuda(), q.cuda())
                for i, s in enumerate(ss):
                    p.orc.append(s, f64(k[:, i:i + 1]), f64(v[:, i:i + 1]))
                torch.cuda.synchronize()
                check_close(out, _ref(p, ss, q, 0), f"fused step seed {seed} op {step}")
            elif op < 0.75 and live:
                ss = rng.sample(live, rng.randint(1, len(live)))
                p.tokens(ss, [rng.randint(1, 40) for _ in ss])
            elif op < 0.85 and live:
                s = rng.choice(live)
                ids = [sg.set_id for sg in p.orc.seqs[s] if sg.kind == "latent"]
                if ids and rng.random() < 0.3:  # same size: in place, or copy-on-write if shared
                    p.latent(s, 128, set_id=rng.choice(ids))
                else:  # a new set at the end of the request
                    p.latent(s, rng.choice([16, 40, 128]))
            elif op < 0.92 and len(live) > 2:
                s = live.pop(rng.randrange(len(live)))
                p.cache.seq_release(s)
                p.orc.release(s)
        except HPAError as e:
            assert e.name in ("HPA_ERR_OUT_OF_PAGES", "HPA_ERR_SEQ_CAPACITY"), e
        if step % 20 == 19 and live:
            batch = sorted(live)
            q = p.queries(len(batch))
            info = _decode_both(p, batch, q, 0, f"step fuzz seed {seed} op {step}")
            grouped += info["group_units"] > 0
    # (the random trees of some cases never pass the 1/3-of-reads rule; the others must cascade)
    assert grouped > 0 or not need


def test_cascade_forced_mode_below_threshold():
    """hpa_set_decode_cascade(c, 2) keeps groups the planner would drop for saving < 1/3 of the
    reads: two requests forked from a 2K prompt, each with 6K rows of its own (saving 1/7) --
    planner mode plans none, forced mode plans group units, both match the oracle; modes
    outside [0, 2] are INVALID_ARG."""
    from paper_2605_09100_b200 import HPAError
    p = Pair(_shape(32, 8, 128, 16, L=1), 4096, 8, 600, seed=21)
    src = p.build([("tokens", 2048)])
    seqs = [src, _fork(p, src, 2048)]
    p.tokens(seqs, [6144, 6144])
    q = p.queries(2)
    ref = _ref(p, seqs, q, 0)
    got = {}
    for mode in (1, 2):
        p.cache.set_decode_cascade(mode)
        got[mode] = p.cache.decode(0, seqs, q.cuda())
        torch.cuda.synchronize()
        n = p.cache.decode_plan_info()["group_units"]
        assert (n > 0) == (mode == 2), (mode, n)
        check_close(got[mode], ref, f"cascade mode {mode}")
    for bad in (-1, 3):
        with pytest.raises(HPAError):
            p.cache.set_decode_cascade(bad)


def test_cascade_full_size_forked_prompt_sampled():
    """bench.py's next.prefix_cascade at full size: B = 64 forks of one 16384-row prompt with
    1024 rows of their own, decoded with the planner's cascade (group units present). Two forks
    are mirrored in the oracle (the prompt and their own rows drawn on the CPU); the others get
    GPU-drawn own rows and are checked for finiteness; cascade off must agree."""
    from workloads import Draw, qwen3_8b_shape
    from oracle import OracleCache
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    B, prompt, own, sampled = 64, 16384, 1024, [0, 63]
    cache = Cache(1, 32, 8, 128, 16, prompt // 16 + B * (own // 16 + 1) + 64, B + 1, prompt // 16 + own // 16 + 4,
                  0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    d = Draw(41)
    src = cache.seq_create()
    orc.create_seq(src)
    k, v = d.tokens(shape, prompt)
    cache.append_kv([src], [prompt], k.cuda(), v.cuda())
    orc.append(src, f64(k), f64(v))
    g = torch.Generator(device="cuda").manual_seed(42)
    forks, ks, vs = [], [], []
    for i in range(B):
        f = cache.seq_fork(src, prompt)
        forks.append(f)
        if i in sampled:
            orc.fork(src, prompt, f)
            k, v = d.tokens(shape, own)
            orc.append(f, f64(k), f64(v))
            ks.append(k.cuda())
            vs.append(v.cuda())
        else:
            ks.append(torch.randn((1, own, 8, 128), generator=g, device="cuda").to(torch.bfloat16))
            vs.append(torch.randn((1, own, 8, 128), generator=g, device="cuda").to(torch.bfloat16))
    cache.append_kv(forks, [own] * B, torch.cat(ks, 1), torch.cat(vs, 1))
    q = torch.randn((B, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    qs = d.queries(shape, len(sampled))
    for i, s in enumerate(sampled):
        q[s] = qs[i].cuda()
    on = cache.decode(0, forks, q)
    torch.cuda.synchronize()
    assert cache.decode_plan_info()["group_units"] > 0
    cache.set_decode_cascade(False)
    off = cache.decode(0, forks, q)
    torch.cuda.synchronize()
    assert torch.isfinite(on.float()).all()
    ref = np.stack([attend(f64(qs[i:i + 1]), *orc.logical_kv(forks[s], 0), shape.scale)[0]
                    for i, s in enumerate(sampled)])
    check_close(on[sampled], ref, "full-size forked prompt, cascade")
    check_close(off[sampled], ref, "full-size forked prompt, plain")
    dmax = (on.float() - off.float()).abs().max().item()
    assert dmax <= 2.0 ** -7 * (1.0 + off.float().abs().max().item()), dmax
    cache.close()


def test_shared_latent_sets_full_size_sampled():
    """bench.py's next.shared_sets at full size: B = 64 requests sharing the same 8 latent sets
    of 128 rows (stored once, refcounted) followed by 4096 token rows each; the planner decides
    (the shared run is 1/5 of the reads: no group units at the default threshold), forced cascade
    (mode 2) and cascade off must all match the oracle on two CPU-drawn requests."""
    from workloads import Draw, LATENT_ROWS, qwen3_8b_shape
    from oracle import OracleCache
    from paper_2605_09100_b200 import Cache
    shape = qwen3_8b_shape(16)
    B, tokens, sampled = 64, 4096, [5, 40]
    cache = Cache(1, 32, 8, 128, 16, 64 + B * (tokens // 16 + 1) + 64, B + 1, 64 + tokens // 16 + 4, 0, 99)
    orc = OracleCache(1, 32, 8, 128, 16)
    d = Draw(51)
    owner = cache.seq_create()
    orc.create_seq(owner)
    for _ in range(8):
        kv = d.latent(shape, LATENT_ROWS)
        assert cache.latent_install(owner, -1, kv.cuda()) == orc.install(owner, -1, f64(kv))
    seqs = [cache.seq_create() for _ in range(B)]
    g = torch.Generator(device="cuda").manual_seed(52)
    ks = []
    for i, s in enumerate(seqs):
        if i in sampled:
            orc.create_seq(s)
        for sid in range(8):
            got = cache.latent_share(s, owner, sid)
            if i in sampled:
                assert got == orc.share(s, owner, sid)
    for i, s in enumerate(seqs):
        if i in sampled:
            k, v = d.tokens(shape, tokens)
            orc.append(s, f64(k), f64(v))
            ks.append((k.cuda(), v.cuda()))
        else:
            ks.append((torch.randn((1, tokens, 8, 128), generator=g, device="cuda").to(torch.bfloat16),) * 2)
    cache.append_kv(seqs, [tokens] * B, torch.cat([a for a, _ in ks], 1), torch.cat([b for _, b in ks], 1))
    q = torch.randn((B, 32, 128), generator=g, device="cuda").to(torch.bfloat16)
    qs = d.queries(shape, len(sampled))
    for i, s in enumerate(sampled):
        q[s] = qs[i].cuda()
    ref = np.stack([attend(f64(qs[i:i + 1]), *orc.logical_kv(seqs[s], 0), shape.scale)[0]
                    for i, s in enumerate(sampled)])
    for mode in (1, 2, 0):
        cache.set_decode_cascade(mode)
        out = cache.decode(0, seqs, q)
        torch.cuda.synchronize()
        assert torch.isfinite(out.float()).all()
        if mode == 2:
            assert cache.decode_plan_info()["group_units"] > 0
        check_close(out[sampled], ref, f"full-size shared latent sets, cascade mode {mode}")
    cache.close()
