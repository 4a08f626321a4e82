"""Replays test_cascade_step_fuzz[seed] and reports the first wrong fused step in detail."""
import os, random, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import attend
from tests.hpa_testutil import Pair, f64
from tests.test_gpu_cascade import _shape, _fork, _valid_cuts, _ref, _decode_both
from paper_2605_09100_b200 import HPAError

seed = int(os.environ.get("SEED", "1"))
print("env MIN_SAVED", os.environ.get("HPA_CASC_MIN_SAVED"), "NO_FUSE", os.environ.get("HPA_NO_FUSE"), flush=True)
rng = random.Random(700 + seed)
shape = _shape(16, 4, 128, 16, L=1)
p = Pair(shape, 6000, 24, 300, seed=seed)
if os.environ.get("CASC_OFF"):
    p.cache.set_decode_cascade(False)
roots = [p.build([("latent", 128), ("tokens", rng.randint(300, 900))]) for _ in range(2)]
live = list(roots)
for step in range(200):
    op = rng.random()
    try:
        if op < 0.25 and len(live) < 24:
            src = rng.choice(live)
            cuts = [c for c in _valid_cuts(p.orc, src) if c > 128]
            if cuts:
                live.append(_fork(p, src, rng.choice(cuts)))
                print(step, "fork", src, "->", live[-1])
        elif op < 0.55 and live:
            ss = sorted(rng.sample(live, rng.randint(1, len(live))))
            k, v = p.draw.tokens(shape, len(ss))
            q = p.queries(len(ss))
            before = {s: p.cache.export_table(s) for s in ss}
            out = p.cache.append_decode(0, ss, k.cuda(), v.cuda(), q.cuda())
            for i, s in enumerate(ss):
                p.orc.append(s, f64(k[:, i:i + 1]), f64(v[:, i:i + 1]))
            torch.cuda.synchronize()
            ref = _ref(p, ss, q, 0)
            err = np.abs(f64(out) - ref).reshape(len(ss), -1).max(axis=1)
            print(step, "fused step", ss, "max err", float(err.max()))
            if err.max() > 1e-2:
                for i, s in enumerate(ss):
                    if err[i] > 1e-2:
                        pg, p0, mt = p.cache.export_table(s)
                        bpg, bp0, bmt = before[s]
                        print("  seq", s, "err", err[i], "segments", [(sg.kind, sg.rows) for sg in p.orc.seqs[s]])
                        print("   before: pages", list(bpg[-4:]), "meta", [int(x) for x in bmt[-4:]], "n", len(bpg))
                        print("   after : pages", list(pg[-4:]), "meta", [int(x) for x in mt[-4:]], "n", len(pg))
                        k2, v2 = p.cache.export_logical_kv(0, s)
                        k1, v1 = p.orc.logical_kv(s, 0)
                        dk = np.abs(f64(k2) - k1).max(axis=(0, 2))
                        print("   export vs oracle: rows differing", np.nonzero(dk)[0][:10], "of", len(dk))
                print("  plan", p.cache.decode_plan_info())
                out2 = p.cache.decode(0, ss, q.cuda())
                torch.cuda.synchronize()
                print("  decode (cascade) after it: max err", float(np.abs(f64(out2) - ref).max()), p.cache.decode_plan_info())
                p.cache.set_decode_cascade(False)
                out3 = p.cache.decode(0, ss, q.cuda())
                torch.cuda.synchronize()
                print("  decode (plain) after it: max err", float(np.abs(f64(out3) - ref).max()))
                break
        elif op < 0.75 and live:
            ss = rng.sample(live, rng.randint(1, len(live)))
            p.tokens(ss, [rng.randint(1, 40) for _ in ss])
        elif op < 0.85 and live:
            s = rng.choice(live)
            ids = [sg.set_id for sg in p.orc.seqs[s] if sg.kind == "latent"]
            if ids and rng.random() < 0.3:
                p.latent(s, 128, set_id=rng.choice(ids)); print(step, "replace set in", s)
            else:
                m = rng.choice([16, 40, 128]); p.latent(s, m); print(step, "new set", m, "in", s)
        elif op < 0.92 and len(live) > 2:
            s = live.pop(rng.randrange(len(live)))
            p.cache.seq_release(s); p.orc.release(s); print(step, "release", s)
    except HPAError as e:
        print(step, "error", e)
    if step % 20 == 19 and live:
        batch = sorted(live)
        qq = p.queries(len(batch))
        info = _decode_both(p, batch, qq, 0, f"check {step}")
        print(step, "check ok", info)
        if os.environ.get("CASC_OFF"):
            p.cache.set_decode_cascade(False)
