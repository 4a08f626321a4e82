"""Randomised parity sweeps (seeded): random head layouts, head dims, page sizes, segment
scripts (latent sets of various sizes, partial pages, token runs), query lengths, split and
CTA settings and GRC spans, each checked element by element against the fp64 oracle."""
import numpy as np
import pytest
import torch

from oracle import attend, attend_span
from tests.hpa_testutil import Pair, check_close, f64
from workloads import Shape

pytestmark = pytest.mark.gpu

LAYOUTS = [(32, 8), (8, 2), (6, 2), (16, 1), (4, 4), (12, 4), (2, 1)]


def _script(rng, max_rows):
    segs, rows = [], 0
    for _ in range(int(rng.integers(1, 6))):
        if rng.random() < 0.4:
            m = int(rng.choice([8, 16, 40, 128, 130]))
            segs.append(("latent", m))
            rows += m
        else:
            n = int(rng.integers(1, 600))
            segs.append(("tokens", n))
            rows += n
        if rows > max_rows:
            break
    if all(k == "latent" for k, _ in segs):
        segs.append(("tokens", int(rng.integers(1, 300))))
    return segs


@pytest.mark.parametrize("case", range(40))
def test_prefill_fuzz(case):
    rng = np.random.default_rng(1000 + case)
    hq, hkv = LAYOUTS[int(rng.integers(len(LAYOUTS)))]
    d = int(rng.choice([64, 128]))
    P = int(rng.choice([16, 32, 64, 128, 256]))
    shape = Shape(2, hq, hkv, d, P)
    p = Pair(shape, num_pages=40000 // P + 256, max_seqs=8, max_pages_per_seq=2048, seed=case)
    n_seqs = int(rng.integers(1, 4))
    seqs = [p.build(_script(rng, 2500)) for _ in range(n_seqs)]
    lens = [p.cache.seq_info(s)[0] for s in seqs]
    q_lens = [min(int(rng.integers(1, L + 1)) if rng.random() < 0.7 else L, 900) for L in lens]
    layer = int(rng.integers(2))
    p.cache.set_prefill_splits(int(rng.choice([0, 0, 1, 2, 3, 5, 16])))
    p.cache.set_prefill_ctas(int(rng.choice([-1, -1, -2, -3, 0, 1, 3])))
    q = p.queries(sum(q_lens))
    use_span = rng.random() < 0.3
    if use_span:
        spans = []
        for L, ql in zip(lens, q_lens):
            q_from = L - ql
            lo = int(rng.integers(0, max(1, q_from)))
            hi = int(rng.integers(lo, q_from + 1))
            spans.append((lo, hi, q_from))
        got = p.cache.prefill_span(layer, seqs, q_lens, spans, q.cuda())
    else:
        got = p.cache.prefill(layer, seqs, q_lens, q.cuda())
    torch.cuda.synchronize()
    ref, off = [], 0
    for i, (s, n) in enumerate(zip(seqs, q_lens)):
        k, v = p.orc.logical_kv(s, layer)
        if use_span:
            lo, hi, qf = spans[i]
            ref.append(attend_span(f64(q[off:off + n]), k, v, shape.scale, lo, hi, qf))
        else:
            ref.append(attend(f64(q[off:off + n]), k, v, shape.scale))
        off += n
    check_close(got, np.concatenate(ref), f"prefill fuzz case {case}: {hq}/{hkv}/{d}/P{P} q_lens={q_lens}")


@pytest.mark.parametrize("case", range(40))
def test_decode_fuzz(case):
    rng = np.random.default_rng(2000 + case)
    hq, hkv = LAYOUTS[int(rng.integers(len(LAYOUTS)))]
    d = int(rng.choice([64, 128]))
    P = int(rng.choice([16, 32, 64, 128, 256]))
    shape = Shape(2, hq, hkv, d, P)
    p = Pair(shape, num_pages=40000 // P + 256, max_seqs=16, max_pages_per_seq=2048, seed=case)
    n_seqs = int(rng.integers(1, 9))
    seqs = [p.build(_script(rng, 3000)) for _ in range(n_seqs)]
    layer = int(rng.integers(2))
    p.cache.set_decode_splits(int(rng.choice([0, 0, 1, 2, 7])))
    q = p.queries(n_seqs)
    got = p.cache.decode(layer, seqs, q.cuda())
    torch.cuda.synchronize()
    ref = np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, layer), shape.scale)[0]
                    for i, s in enumerate(seqs)])
    check_close(got, ref, f"decode fuzz case {case}: {hq}/{hkv}/{d}/P{P} n={n_seqs}")


@pytest.mark.parametrize("case", range(16))
def test_fp8_token_pages_fuzz(case):
    """fp8 (e4m3) token pages with bf16 latent pages (reading A20): random shapes and scripts,
    decode and prefill on a random layer against the oracle's quantized cache."""
    rng = np.random.default_rng(3000 + case)
    hq, hkv = LAYOUTS[int(rng.integers(len(LAYOUTS)))]
    d = int(rng.choice([64, 128]))
    P = int(rng.choice([16, 32, 64, 128, 256]))
    shape = Shape(2, hq, hkv, d, P)
    npg = 40000 // P + 256
    p = Pair(shape, num_pages=npg, max_seqs=8, max_pages_per_seq=2048, seed=case, token_fp8=True,
             num_token_pages=npg)
    n_seqs = int(rng.integers(1, 5))
    seqs = [p.build(_script(rng, 2500)) for _ in range(n_seqs)]
    layer = int(rng.integers(2))
    q = p.queries(n_seqs)
    got = p.cache.decode(layer, seqs, q.cuda())
    torch.cuda.synchronize()
    ref = np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, layer), shape.scale)[0]
                    for i, s in enumerate(seqs)])
    check_close(got, ref, f"fp8 decode fuzz case {case}")
    lens = [p.cache.seq_info(s)[0] for s in seqs]
    q_lens = [min(int(rng.integers(1, L + 1)), 600) for L in lens]
    p.cache.set_prefill_splits(int(rng.choice([0, 1, 3])))
    qp = p.queries(sum(q_lens))
    got = p.cache.prefill(layer, seqs, q_lens, qp.cuda())
    torch.cuda.synchronize()
    ref, off = [], 0
    for s, n in zip(seqs, q_lens):
        k, v = p.orc.logical_kv(s, layer, fp8_staged=True)
        ref.append(attend(f64(qp[off:off + n]), k, v, shape.scale))
        off += n
    check_close(got, np.concatenate(ref), f"fp8 prefill fuzz case {case}")


@pytest.mark.parametrize("seed", range(3))
def test_cache_ops_fuzz_with_attention(seed):
    """400 random cache operations -- appends, latent installs and replacements of other
    sizes, removals, in-cache compression, sharing a set from another request, releases --
    with decode and prefill parity for every live request every 40 operations."""
    import random
    from paper_2605_09100_b200 import HPAError
    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    shape = Shape(1, 8, 2, 128, int(rng.choice([16, 32])))
    p = Pair(shape, num_pages=1200, max_seqs=6, max_pages_per_seq=256, seed=seed)
    live = []

    def latents(s):
        return [sg.set_id for sg in p.orc.seqs[s] if sg.kind == "latent"]

    def check(tag):
        alive = [s for s in live if p.cache.seq_info(s)[0] > 0]
        if not alive:
            return
        q = p.queries(len(alive))
        got = p.cache.decode(0, alive, q.cuda())
        torch.cuda.synchronize()
        ref = np.stack([attend(f64(q[i:i + 1]), *p.orc.logical_kv(s, 0), shape.scale)[0]
                        for i, s in enumerate(alive)])
        check_close(got, ref, f"ops fuzz decode {tag}")
        lens = [p.cache.seq_info(s)[0] for s in alive]
        q_lens = [int(nrng.integers(1, min(L, 300) + 1)) for L in lens]
        qp = p.queries(sum(q_lens))
        got = p.cache.prefill(0, alive, q_lens, qp.cuda())
        torch.cuda.synchronize()
        ref, off = [], 0
        for s, n in zip(alive, q_lens):
            k, v = p.orc.logical_kv(s, 0)
            ref.append(attend(f64(qp[off:off + n]), k, v, shape.scale))
            off += n
        check_close(got, np.concatenate(ref), f"ops fuzz prefill {tag}")

    for step in range(400):
        op = rng.random()
        try:
            if op < 0.12 and len(live) < 6:
                live.append(p.new_seq())
            elif op < 0.40 and live:
                p.tokens([rng.choice(live)], [rng.randint(1, 90)])
            elif op < 0.58 and live:
                s = rng.choice(live)
                ids = latents(s)
                sid = rng.choice(ids) if ids and rng.random() < 0.5 else -1
                p.latent(s, rng.choice([8, 16, 40, 64, 128]), set_id=sid)
            elif op < 0.66 and live:
                s = rng.choice(live)
                ids = latents(s)
                if ids:
                    sid = rng.choice(ids)
                    p.cache.latent_remove(s, sid)
                    p.orc.remove(s, sid)
            elif op < 0.76 and live:
                s = rng.choice(live)
                segs = p.orc.seqs[s]
                if segs and segs[-1].kind == "token" and segs[-1].rows >= 24:
                    m = rng.randint(1, 8)
                    n_doc = rng.randint(0, segs[-1].rows - m)
                    assert p.cache.compress(s, n_doc, m) == p.orc.compress(s, n_doc, m)
            elif op < 0.84 and len(live) >= 2:
                src, dst = rng.sample(live, 2)
                ids = latents(src)
                if ids:
                    sid = rng.choice(ids)
                    assert p.cache.latent_share(dst, src, sid) == p.orc.share(dst, src, sid)
            elif op < 0.90 and live:
                s = live.pop(rng.randrange(len(live)))
                p.cache.seq_release(s)
                p.orc.release(s)
        except HPAError as e:
            assert e.name in ("HPA_ERR_OUT_OF_PAGES", "HPA_ERR_SEQ_CAPACITY"), e
        if step % 40 == 39:
            check(f"seed {seed} step {step}")
