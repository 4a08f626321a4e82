"""Random-operation fuzz over the whole C ABI surface against the oracle
(tests/test_gpu_fuzz_all.py runs short sequences; scripts/fuzz_all.py long ones). Ops: create / release, bulk append, fused decode step
(hpa_append_decode), latent install / replace / remove / share, fork, compress (single and
batched), host-staged install; checks every CHECK ops: bit-exact logical views, decode
(cascade on and off), decode_partial, prefill and prefill_span parity, page accounting.
"""
import random

import numpy as np
import torch

from oracle import attend, attend_span
from paper_2605_09100_b200 import HPAError
from workloads import Shape

from tests.hpa_testutil import Pair, check_close, f64


def check_tol(got, ref, what, stats):
    """stats["strict"]: the north_star bound only (the committed tests). Otherwise: north_star tolerance (max abs 1e-2, rel L2 5e-3); where it fails only on elements with
    |o| >= 2 -- bf16 output spacing 2^-6 there, so half an ulp plus the bf16 rounding of P
    (reading A9) can pass 1e-2 -- accept an error of at most one output ulp and count it."""
    try:
        check_close(got, ref, what)
    except AssertionError:
        if stats["strict"]:
            raise
        g = f64(got)
        err = np.abs(g - ref)
        ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
        rel = np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30)
        if not (np.all(np.isfinite(g)) and rel <= 5e-3 and np.all(err <= np.maximum(1e-2, ulp))):
            raise
        stats["ulp_edge"] += 1


def valid_cuts(orc, s):
    cuts, pos = [0], 0
    for sg in orc.seqs[s]:
        if sg.kind == "token":
            cuts += list(range(pos + 1, pos + sg.rows + 1))
        else:
            cuts.append(pos + sg.rows)
        pos += sg.rows
    return sorted(set(cuts))


def run(seed, n_ops, fp8, check_every, strict=False):
    rng = random.Random(seed)
    hq, hkv, d, P = rng.choice([(32, 8, 128, 16), (16, 2, 128, 32), (8, 8, 64, 16), (16, 4, 64, 64), (8, 1, 128, 16)])
    L = rng.choice([1, 2])
    shape = Shape(L, hq, hkv, d, P)
    npages = 3000
    p = Pair(shape, npages, 16, 4000 // P, seed=seed, token_fp8=fp8, num_token_pages=npages if fp8 else 0)
    live = []
    stats = {"ops": 0, "checks": 0, "cascade": 0, "errors": 0, "ulp_edge": 0, "strict": strict}

    def latents(s):
        return [sg.set_id for sg in p.orc.seqs[s] if sg.kind == "latent"]

    def check(tag):
        alive = sorted(s for s in live if p.orc.seq_len(s) > 0)
        if not alive:
            return
        stats["checks"] += 1
        torch.cuda.synchronize()
        for layer in range(L):
            for s in alive:
                k1, v1 = p.orc.logical_kv(s, layer, fp8_staged=fp8)
                k2, v2 = p.cache.export_logical_kv(layer, s)
                assert np.array_equal(k1, f64(k2)) and np.array_equal(v1, f64(v2)), (tag, "view", s, layer)
        layer = rng.randrange(L)
        q = p.queries(len(alive))
        ref = np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, layer), shape.scale)[0]
                        for i, s in enumerate(alive)])
        for mode in (1, 2, 0):  # planner, every shared run, off
            p.cache.set_decode_cascade(mode)
            got = p.cache.decode(layer, alive, q.cuda())
            torch.cuda.synchronize()
            if mode and p.cache.decode_plan_info()["group_units"] > 0:
                stats["cascade"] += 1
            check_tol(got, ref, f"{tag} decode cascade={mode}", stats)
        p.cache.set_decode_cascade(rng.choice((1, 2)))  # for decode_partial and the fused steps
        o, lse = p.cache.decode_partial(layer, alive, q.cuda())
        torch.cuda.synchronize()
        check_tol(o, ref, f"{tag} decode_partial", stats)
        sub = alive[:4]
        q_lens = [rng.randint(1, min(p.orc.seq_len(s), 64)) for s in sub]
        qp = p.queries(sum(q_lens))
        got = p.cache.prefill(layer, sub, q_lens, qp.cuda())
        torch.cuda.synchronize()
        refs, off = [], 0
        for s, n in zip(sub, q_lens):
            k, v = p.orc.logical_kv(s, layer, fp8_staged=fp8)  # prefill reads staged rows (A20)
            refs.append(attend(f64(qp[off:off + n]), k, v, shape.scale))
            off += n
        try:
            check_tol(got, np.concatenate(refs), f"{tag} prefill", stats)
        except AssertionError:
            off = 0
            for s, n, r in zip(sub, q_lens, refs):
                g = f64(got[off:off + n])
                e = np.abs(g - r)
                i = np.unravel_index(np.argmax(e), e.shape)
                segs = [(sg.kind, sg.rows) for sg in p.orc.seqs[s]]
                print(f"seq {s} n={n} len={p.orc.seq_len(s)} maxerr={e.max():.3e} at {i} ref={r[i]:.4f} "
                      f"got={g[i]:.4f} max|ref|={np.abs(r).max():.3f} rel={np.linalg.norm(g - r) / np.linalg.norm(r):.2e} segs={segs}")
                off += n
            raise
        if not fp8:  # GRC span: queries from q_from on do not see rows [lo, hi)
            spans, refs, off = [], [], 0
            for s, n in zip(sub, q_lens):
                Ls = p.orc.seq_len(s)
                lo = rng.randint(0, min(Ls // 2, Ls - n))
                hi = rng.randint(lo, Ls - n)
                spans.append((lo, hi, Ls - n + rng.randint(0, n - 1)))
            got = p.cache.prefill_span(layer, sub, q_lens, spans, qp.cuda())
            torch.cuda.synchronize()
            for (s, n), sp in zip(zip(sub, q_lens), spans):
                k, v = p.orc.logical_kv(s, layer)
                refs.append(attend_span(f64(qp[off:off + n]), k, v, shape.scale, *sp))
                off += n
            check_tol(got, np.concatenate(refs), f"{tag} prefill_span", stats)

    for step in range(n_ops):
        op = rng.random()
        stats["ops"] += 1
        try:
            if op < 0.07 and len(live) < 16:
                live.append(p.new_seq())
            elif op < 0.15 and live and len(live) < 16:
                src = rng.choice(live)
                live.append(p.cache.seq_fork(src, c := rng.choice(valid_cuts(p.orc, src))))
                p.orc.fork(src, c, live[-1])
            elif op < 0.35 and live:
                ss = rng.sample(live, rng.randint(1, len(live)))
                p.tokens(ss, [rng.randint(1, 60) for _ in ss])
            elif op < 0.50 and live:
                ss = sorted(rng.sample(live, rng.randint(1, len(live))))
                ss = [s for s in ss if p.orc.seq_len(s) > 0] or ss[:0]
                if ss:
                    k, v = p.draw.tokens(shape, len(ss))
                    q = p.queries(len(ss))
                    layer = rng.randrange(L)
                    out = p.cache.append_decode(layer, ss, k.cuda(), v.cuda(), q.cuda())
                    for i, s in enumerate(ss):
                        p.orc.append(s, f64(k[:, i:i + 1]), f64(v[:, i:i + 1]))
                    torch.cuda.synchronize()
                    ref = np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, layer), shape.scale)[0]
                                    for i, s in enumerate(ss)])
                    check_tol(out, ref, f"seed {seed} op {step} fused step", stats)
            elif op < 0.62 and live:
                s = rng.choice(live)
                ids = latents(s)
                sid = rng.choice(ids) if ids and rng.random() < 0.4 else -1
                p.latent(s, rng.choice([8, 16, 40, 128]), set_id=sid)
            elif op < 0.66 and live:
                s = rng.choice(live)
                ids = latents(s)
                if ids:
                    sid = rng.choice(ids)
                    p.cache.latent_remove(s, sid)
                    p.orc.remove(s, sid)
            elif op < 0.72 and len(live) >= 2:
                src, dst = rng.sample(live, 2)
                ids = latents(src)
                if ids:
                    sid = rng.choice(ids)
                    assert p.cache.latent_share(dst, src, sid) == p.orc.share(dst, src, sid)
            elif op < 0.80 and live:
                cand = [s for s in live if p.orc.seqs[s] and p.orc.seqs[s][-1].kind == "token"
                        and p.orc.seqs[s][-1].rows >= 12]
                if cand:
                    ss = rng.sample(cand, rng.randint(1, len(cand)))
                    ms = [rng.randint(1, 8) for _ in ss]
                    nds = [rng.randint(0, p.orc.seqs[s][-1].rows - m) for s, m in zip(ss, ms)]
                    if len(ss) == 1 and rng.random() < 0.5:
                        got = [p.cache.compress(ss[0], nds[0], ms[0])]
                    else:
                        got = list(p.cache.compress_batch(ss, nds, ms))
                    for g, s, nd, m in zip(got, ss, nds, ms):
                        assert g == p.orc.compress(s, nd, m)
            elif op < 0.84 and live:
                ss = rng.sample(live, min(len(live), rng.randint(1, 3)))
                kv = torch.stack([p.draw.latent(shape, 64) for _ in ss]).pin_memory()
                got = p.cache.latent_install_host(ss, [-1] * len(ss), kv)
                for i, s in enumerate(ss):
                    assert got[i] == p.orc.install(s, -1, f64(kv[i]))
            elif op < 0.90 and len(live) > 1:
                s = live.pop(rng.randrange(len(live)))
                p.cache.seq_release(s)
                p.orc.release(s)
        except HPAError as e:
            stats["errors"] += 1
            assert e.name in ("HPA_ERR_OUT_OF_PAGES", "HPA_ERR_SEQ_CAPACITY"), (seed, step, e)
        if step % check_every == check_every - 1:
            check(f"seed {seed} op {step}")
    p.cache.close()
    return (hq, hkv, d, P, L), stats
