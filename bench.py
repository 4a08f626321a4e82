#!/usr/bin/env python
"""bench.py -- hybrid paged attention (HPA) on B200: the BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Step (N=1 workload = BASELINE.json configs[1], "Qwen3-8B-shaped decode"):
  B=64 requests per GPU, Hq=32 / H_kv=8 / d=128, page 16; each request holds
  8 retrieved documents compressed to m=128-row latent sets + 4K reasoning
  tokens. One step = append the current token's KV for every request (a2,
  with the a1 table update) + split-KV decode + combine (a4, a5) for one layer.
  value = decode tokens/s over all ranks (weak scaling: 64 requests per GPU).
The same run also measures chunked prefill (configs[2], a6, TFLOP/s) and the
LMAG step with per-request latent replacement (configs[3], a3), reported as
sub-objects. Inputs are resident in HBM before timing; the KV working set
(1.4 GB) is >10x L2, so no L2 flush is needed between steps.

--impl reference times the fp64 CPU oracle (oracle/, test infrastructure) on
a bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attn tokens/s + achieved HBM GB/s vs 8 TB/s; prefill TFLOP/s, 1/2/4/8 B200"
NOMINAL_HBM_GBS = 8000.0
NOMINAL_BF16_TFLOPS = 2250.0
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--page-size", type=int, default=16)
    ap.add_argument("--batch", type=int, default=64, help="requests per GPU (configs[1]: 64)")
    ap.add_argument("--no-extra", action="store_true", help="skip the prefill / LMAG sub-benchmarks")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--splits", type=int, default=0, help="force decode split count (0 = planner)")
    ap.add_argument("--sweep", action="store_true", help="configs[4] sweep (per-GPU shard), JSON per point")
    ap.add_argument("--sweep-n", type=int, default=8, help="GPUs the sweep's global batch is sharded over")
    ap.add_argument("--sweep-max-gb", type=float, default=120.0)
    ap.add_argument("--sweep-min-gb", type=float, default=0.0, help="only points with at least this pool size")
    ap.add_argument("--mode", default="request", choices=["request", "head_shard", "context_parallel"],
                    help="multi-GPU partition of the configs[1] step (SURVEY 8(e)): request shard (default, weak "
                         "scaling, no collective), KV-head shard + NCCL all-gather of the outputs, or "
                         "context-parallel row shards + NCCL all-gather of fp32 partials + LSE merge (both strong "
                         "scaling: the global batch of --batch requests is fixed)")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if a.gpus != world:
        # never run fewer GPUs than asked for and report it as N: multi-GPU runs are launched by
        # torchrun, which sets WORLD_SIZE (python -m torch.distributed.run --nproc-per-node N ...)
        sys.exit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}; launch N > 1 GPUs with "
                 f"python -m torch.distributed.run --nnodes=1 --nproc-per-node {a.gpus} bench.py --gpus {a.gpus}")
    return a


def init_dist():
    """(world, rank, local) from the torchrun environment; NCCL process group when world > 1."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return world, rank, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return dict(FALLBACK), "fallback"


# ----------------------------------------------------------------------------- clocks
_SAMPLER = r"""
import sys, time, pynvml as nv
nv.nvmlInit()
bus = sys.argv[1]
try:
    h = nv.nvmlDeviceGetHandleByPciBusId(bus)
except Exception:
    h = nv.nvmlDeviceGetHandleByIndex(0)
out = open(sys.argv[2], "w")
out.write(f"max {nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)}\n"); out.flush()
while True:
    t = time.time()
    try:
        c = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        try:
            pw = nv.nvmlDeviceGetPowerUsage(h)
        except Exception:
            pw = -1
        out.write(f"{t:.6f} {c} {r} {pw}\n"); out.flush()
    except Exception:
        pass
    time.sleep(0.0005)
"""

_REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}


class ClockSampler:
    """NVML SM clock + throttle reasons polled every ~0.5 ms by a separate process;
    summary() keeps the samples that fall inside [start(), stop()]."""

    def __init__(self, device: int):
        import subprocess
        import tempfile
        import torch
        self.path = tempfile.mktemp(prefix="hpa_clk_")
        p = torch.cuda.get_device_properties(device)
        bus = f"{getattr(p, 'pci_domain_id', 0):08x}:{getattr(p, 'pci_bus_id', 0):02x}:{getattr(p, 'pci_device_id', 0):02x}.0"
        self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, bus, self.path],
                                     stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        self.t0 = self.t1 = None
        deadline = time.time() + 20
        while time.time() < deadline:  # wait until the sampler produces data
            try:
                with open(self.path) as f:
                    if len(f.read().splitlines()) >= 3:
                        break
            except FileNotFoundError:
                pass
            time.sleep(0.05)

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()
        time.sleep(0.01)
        self.proc.terminate()
        self.proc.wait()

    def summary(self):
        try:
            lines = open(self.path).read().splitlines()
            os.unlink(self.path)
        except Exception as e:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": str(e)}
        mx, clk, reasons, pw = None, [], set(), []
        for ln in lines:
            parts = ln.split()
            if parts[0] == "max":
                mx = int(parts[1])
                continue
            t, c, r = float(parts[0]), int(parts[1]), int(parts[2])
            if self.t0 is not None and self.t0 <= t <= self.t1:
                clk.append(c)
                reasons |= {k for k, b in _REASONS.items() if r & b}
                if len(parts) > 3 and int(parts[3]) >= 0:
                    pw.append(int(parts[3]) / 1000.0)
        out = {"sm_mhz": statistics.median(clk) if clk else None, "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(clk)}
        if pw:
            out["power_w"] = round(statistics.median(pw), 1)
        return out


# ----------------------------------------------------------------------------- workload build
def build_decode_cache(torch, Cache, shape, n_req, docs, tokens, extra_rows, device, seed, placement_seed=99,
                       token_kv_dtype="bf16", bf16_headroom_pages=0):
    """Creates a cache holding n_req requests of `docs` latent sets (m=128) followed by
    `tokens` token rows (an int, or one count per request for the ragged variant);
    returns (cache, seq ids). Inputs drawn on the GPU (seeded)."""
    from workloads import LATENT_ROWS
    P = shape.page_size
    if not isinstance(tokens, int):
        return _build_ragged(torch, Cache, shape, n_req, docs, list(tokens), extra_rows, device, seed,
                             placement_seed)
    rows_max = docs * LATENT_ROWS + tokens + extra_rows
    pages_per_seq = docs * math.ceil(LATENT_ROWS / P) + math.ceil((tokens + extra_rows) / P) + 1
    if token_kv_dtype == "fp8":  # NEXT-4c: token pages in their own fp8 pool
        lat_pages = docs * math.ceil(LATENT_ROWS / P)
        cache = Cache(shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, P,
                      n_req * lat_pages + 64 + bf16_headroom_pages, n_req, pages_per_seq, device, placement_seed,
                      "fp8", n_req * (pages_per_seq - lat_pages) + 64)
    else:
        cache = Cache(shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, P,
                      n_req * pages_per_seq + 64, n_req, pages_per_seq, device, placement_seed)
    g = torch.Generator(device=f"cuda:{device}").manual_seed(seed)
    seqs = [cache.seq_create() for _ in range(n_req)]
    for _ in range(docs):
        kv = torch.randn((n_req, shape.num_layers, 2, LATENT_ROWS, shape.num_kv_heads, shape.head_dim),
                         generator=g, device=f"cuda:{device}").to(torch.bfloat16)
        cache.latent_install_batch(seqs, [-1] * n_req, [kv[i] for i in range(n_req)])
        del kv
    if tokens:
        chunk = max(1, (1 << 28) // (tokens * shape.num_kv_heads * shape.head_dim * 2))  # <= 256 MB per draw
        for lo in range(0, n_req, chunk):
            ids = seqs[lo:lo + chunk]
            s = (shape.num_layers, len(ids) * tokens, shape.num_kv_heads, shape.head_dim)
            k = torch.randn(s, generator=g, device=f"cuda:{device}").to(torch.bfloat16)
            v = torch.randn(s, generator=g, device=f"cuda:{device}").to(torch.bfloat16)
            cache.append_kv(ids, [tokens] * len(ids), k, v)
            del k, v
    torch.cuda.synchronize(device)
    return cache, seqs, rows_max


def _build_ragged(torch, Cache, shape, n_req, docs, tokens, extra_rows, device, seed, placement_seed):
    from workloads import LATENT_ROWS
    P = shape.page_size
    pages = [docs * math.ceil(LATENT_ROWS / P) + math.ceil((t + extra_rows) / P) + 1 for t in tokens]
    cache = Cache(shape.num_layers, shape.num_q_heads, shape.num_kv_heads, shape.head_dim, P,
                  sum(pages) + 64, n_req, max(pages), device, placement_seed)
    g = torch.Generator(device=f"cuda:{device}").manual_seed(seed)
    seqs = [cache.seq_create() for _ in range(n_req)]
    for _ in range(docs):
        kv = torch.randn((n_req, shape.num_layers, 2, LATENT_ROWS, shape.num_kv_heads, shape.head_dim),
                         generator=g, device=f"cuda:{device}").to(torch.bfloat16)
        cache.latent_install_batch(seqs, [-1] * n_req, [kv[i] for i in range(n_req)])
        del kv
    for sq, t in zip(seqs, tokens):
        s = (shape.num_layers, t, shape.num_kv_heads, shape.head_dim)
        k = torch.randn(s, generator=g, device=f"cuda:{device}").to(torch.bfloat16)
        v = torch.randn(s, generator=g, device=f"cuda:{device}").to(torch.bfloat16)
        cache.append_kv([sq], [t], k, v)
    torch.cuda.synchronize(device)
    return cache, seqs, docs * LATENT_ROWS + max(tokens) + extra_rows


def time_decode_calls(torch, cache, seqs, shape, dev, stream, K, W, seed=77):
    """Decode-only timing (CUDA events on the launch stream), mean ms per call."""
    import numpy as np
    ids = np.asarray(seqs, dtype=np.int32)
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(seed)
    q = torch.randn((len(seqs), shape.num_q_heads, shape.head_dim), generator=g,
                    device=f"cuda:{dev}").to(torch.bfloat16)
    out = torch.empty_like(q)
    for _ in range(W):
        cache.decode(0, ids, q, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(K):
        cache.decode(0, ids, q, out)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / K


def bench_decode_variants(torch, Cache, dev, stream, pk, page_size):
    """configs[1] variants: ragged reasoning lengths ~ U[1K, 8K], and the other
    page size (P=64 when the headline runs P=16). Decode call only, CUDA events."""
    from workloads import qwen3_8b_shape
    out = {}
    g = torch.Generator().manual_seed(1234 + 7)
    ragged = [int(torch.randint(1024, 8193, (1,), generator=g).item()) for _ in range(64)]
    for name, P, toks in (("ragged_U1K_8K", page_size, ragged), (f"page_size_{64 if page_size != 64 else 16}",
                                                                   64 if page_size != 64 else 16, 4096)):
        shape = qwen3_8b_shape(P)
        cache, seqs, _ = build_decode_cache(torch, Cache, shape, 64, 8, toks, 0, dev, seed=1234)
        ms = time_decode_calls(torch, cache, seqs, shape, dev, stream, 50, 5)
        lens = [cache.seq_info(sq)[0] for sq in seqs]
        byts = decode_bytes(lens, shape)
        out[name] = {"page_size": P, "requests": 64, "mean_len": round(sum(lens) / len(lens), 1),
                     "decode_ms": round(ms, 4), "tokens_per_s": round(64 / (ms / 1e3), 1),
                     "achieved_gbs": round(byts / (ms / 1e3) / 1e9, 1),
                     "frac": round(byts / (ms / 1e3) / 1e9 / pk["hbm_gbs"], 4)}
        cache.close()
        torch.cuda.empty_cache()
    # NEXT-4c: the same configs[1] batch with fp8 token pages (latent pages stay bf16)
    shape = qwen3_8b_shape(page_size)
    cache, seqs, _ = build_decode_cache(torch, Cache, shape, 64, 8, 4096, 0, dev, seed=1234, token_kv_dtype="fp8")
    ms = time_decode_calls(torch, cache, seqs, shape, dev, stream, 50, 5)
    hkv, d = shape.num_kv_heads, shape.head_dim
    lat_rows, tok_rows = 8 * 128, 4096
    per_req = (lat_rows * hkv * d * 2 * 2 + tok_rows * hkv * (d + 4) * 2 + 2 * shape.num_q_heads * d * 2
               + 4 * math.ceil((lat_rows + tok_rows) / shape.page_size))
    byts = 64 * per_req
    bf16_ms = out.get(f"page_size_{64 if page_size != 64 else 16}", {}).get("decode_ms")
    out["fp8_token_pages"] = {"page_size": page_size, "requests": 64, "latent_rows": lat_rows, "token_rows": tok_rows,
                              "decode_ms": round(ms, 4), "tokens_per_s": round(64 / (ms / 1e3), 1),
                              "bytes_per_call": byts, "achieved_gbs": round(byts / (ms / 1e3) / 1e9, 1),
                              "frac": round(byts / (ms / 1e3) / 1e9 / pk["hbm_gbs"], 4),
                              "note": "token rows: e4m3 codes + fp32 K/V row scales (reading A20); bytes are those read"}
    cache.close()
    torch.cuda.empty_cache()
    return out


def bench_sweep(args):
    """configs[4]: the 8xB200 request-sharded sweep. Each rank holds B/n requests (no data-path
    collective), so one GPU measures exactly the per-GPU work of the n-GPU run; whole-job
    requests/s = n x per-GPU (weak in requests per GPU), max over ranks when run under torchrun.
    Latent rows = floor(r*ctx/128)*128 as whole sets placed first;
    achieved GB/s must be flat (+-3 %) across r at fixed (B, ctx). One JSON line per point,
    then a summary line. Points whose pool exceeds --sweep-max-gb are reported as skipped."""
    import torch
    import torch.distributed as dist
    from paper_2605_09100_b200 import Cache
    from paper_2605_09100_b200.dist import max_over_ranks
    from workloads import LATENT_ROWS, qwen3_8b_shape
    world, rank, dev = init_dist()
    stream = torch.cuda.current_stream(dev)
    pk, pk_kind = peaks()
    shape = qwen3_8b_shape(args.page_size)
    # under torchrun every rank holds its own B/n shard and the job rate uses the slowest rank;
    # run alone (one process), the GPU measures one shard of an --sweep-n-GPU job
    n = world if world > 1 else args.sweep_n
    rows_bytes = shape.num_kv_heads * shape.head_dim * 2 * 2
    points = []
    for B in (512, 1024, 2048, 4096):
        b = B // n
        for ctx in (8192, 16384, 32768, 65536):
            for r in (0.1, 0.5, 0.9):
                sets = int(r * ctx) // LATENT_ROWS
                tok = ctx - sets * LATENT_ROWS
                gb = b * ctx * rows_bytes / 1e9
                pt = {"global_batch": B, "n_gpus": n, "requests_per_gpu": b, "context": ctx,
                      "latent_ratio": r, "latent_sets": sets, "token_rows": tok, "kv_gb_per_gpu": round(gb, 2)}
                if gb < args.sweep_min_gb:
                    continue
                if gb > args.sweep_max_gb:
                    pt["skipped"] = f"pool {gb:.0f} GB > --sweep-max-gb {args.sweep_max_gb}"
                    if rank == 0:
                        print(json.dumps(pt), flush=True)
                    points.append(pt)
                    continue
                cache, seqs, _ = build_decode_cache(torch, Cache, shape, b, sets, tok, 0, dev, seed=1234 + rank)
                if world > 1:
                    dist.barrier(device_ids=[dev])
                ms_local = time_decode_calls(torch, cache, seqs, shape, dev, stream, args.steps, args.warmup)
                ms = max_over_ranks(ms_local, device=f"cuda:{dev}")
                byts = decode_bytes([ctx] * b, shape)
                pt.update({"decode_ms": round(ms, 4), "requests_per_s_per_gpu": round(b / (ms_local / 1e3), 1),
                           "requests_per_s_job": round(n * b / (ms / 1e3), 1),
                           "job_rate": "max over ranks (torchrun)" if world > 1 else
                                       f"one GPU's shard x {n} (no data-path collective)",
                           "achieved_gbs": round(byts / (ms_local / 1e3) / 1e9, 1),
                           "frac": round(byts / (ms_local / 1e3) / 1e9 / pk["hbm_gbs"], 4)})
                cache.close()
                torch.cuda.empty_cache()
                if rank == 0:
                    print(json.dumps(pt), flush=True)
                points.append(pt)
    flat = []
    for B in (512, 1024, 2048, 4096):
        for ctx in (8192, 16384, 32768, 65536):
            g = [p["achieved_gbs"] for p in points if p["global_batch"] == B and p["context"] == ctx
                 and "achieved_gbs" in p]
            if len(g) == 3:
                flat.append({"global_batch": B, "context": ctx,
                             "spread": round((max(g) - min(g)) / (sum(g) / 3), 4)})
    if rank == 0:
        print(json.dumps({"sweep": "configs[4]", "peak": pk["hbm_gbs"], "peak_kind": pk_kind,
                          "page_size": args.page_size, "n_gpus": n, "ranks_run": world,
                          "max_latent_ratio_spread": max((f["spread"] for f in flat), default=None),
                          "flatness": flat}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def decode_bytes(lens, shape):
    """Algorithmic bytes of one decode call: K+V rows + q + out + table."""
    hkv, d, hq, P = shape.num_kv_heads, shape.head_dim, shape.num_q_heads, shape.page_size
    return sum(L * hkv * d * 2 * 2 + 2 * hq * d * 2 + 4 * math.ceil(L / P) for L in lens)


def append_bytes(n, shape):
    """Algorithmic bytes of appending one K and V row per request (every layer): read + write."""
    return 2 * 2 * n * shape.num_layers * shape.num_kv_heads * shape.head_dim * 2


def prefill_flops(prior, c, shape):
    """4 Hq d (C L_prior + C(C+1)/2) per request."""
    return 4 * shape.num_q_heads * shape.head_dim * (c * prior + c * (c + 1) // 2)


# ----------------------------------------------------------------------------- our arm
def headline_config(B, world, page_size, docs=8, tokens=4095):
    """The bench line's config (both arms: ours and --impl reference)."""
    return {"workload": "configs[1] Qwen3-8B-shaped HPA decode step (append 1 token + decode, hpa_append_decode), one layer",
            "requests_per_gpu": B, "global_batch": B * world, "num_q_heads": 32, "num_kv_heads": 8,
            "head_dim": 128, "page_size": page_size, "latent_sets": docs, "latent_rows": 128,
            "reasoning_tokens": tokens + 1, "seq_len": docs * 128 + tokens + 1,
            "parallelism": f"request-shard x{world}" if world > 1 else "single GPU",
            "l2": "working set 1.4 GB/GPU >> 126 MB L2 (no flush needed)",
            "placement": "seeded random physical page permutation"}


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2605_09100_b200 import Cache
    from paper_2605_09100_b200.dist import max_over_ranks
    from workloads import qwen3_8b_shape

    world, rank, dev = init_dist()
    stream = torch.cuda.current_stream(dev)
    pk, pk_kind = peaks()
    shape = qwen3_8b_shape(args.page_size)
    B, docs, tokens = args.batch, 8, 4095  # + the current token appended each step -> Lb = 5120
    K, W = args.steps, args.warmup

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[dev])

    # ------------------------------------------------------------------ configs[1] decode step
    # One step = hpa_append_decode: the current token's K/V row of every request written into
    # its page slot (a1 + a2) and the split decode + combine (a4 + a5), one kernel launch
    # (+ the combine). Region A (the `value`) has nothing but the steps between its two
    # events; then the e2e region (host copies, same lengths as region A); region B repeats the
    # steps with an event pair around every call for the per-launch duration of the roofline
    # (events between launches break the programmatic dependent launch overlap, so they stay
    # out of region A).
    cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, docs, tokens, 3 * K + W + 16, dev,
                                        seed=1234 + rank)
    if args.splits:
        cache.set_decode_splits(args.splits)
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(4321 + rank)
    nsteps = 2 * K + W
    knew = torch.randn((nsteps, 1, B, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    vnew = torch.randn((nsteps, 1, B, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    qs = torch.randn((nsteps, B, 32, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    out = torch.empty((B, 32, 128), dtype=torch.bfloat16, device=f"cuda:{dev}")
    import numpy as np
    ids = np.asarray(seqs, dtype=np.int32)
    for i in range(W):
        cache.append_decode(0, ids, knew[i], vnew[i], qs[i], out)
    torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = cache.launch_count()
    clk = ClockSampler(dev)
    barrier()
    torch.cuda.synchronize(dev)
    clk.start()
    t0.record(stream)
    for i in range(K):
        cache.append_decode(0, ids, knew[W + i], vnew[W + i], qs[W + i], out)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    clk.stop()
    barrier()
    launches = cache.launch_count() - launches0
    step_ms = t0.elapsed_time(t1) / K
    step_ms_max = max_over_ranks(step_ms, device=f"cuda:{dev}")
    total_tokens = B * world
    value = total_tokens / (step_ms_max / 1e3)
    # ------------------------------------------------------------------ e2e through the public API
    # pinned host inputs -> device (copy stream, double-buffered) -> append + decode
    # (compute stream) -> output -> pinned host; all copies inside the timed region.
    # the step's inputs (new K row, new V row, q) travel as ONE packed pinned buffer per step
    # (one H2D copy; the device views are k / v / q), the output comes back in one D2H copy
    n_k, n_q = knew[0].numel(), qs[0].numel()
    pin_in = torch.cat([knew.reshape(nsteps, -1), vnew.reshape(nsteps, -1), qs.reshape(nsteps, -1)],
                       dim=1).cpu().pin_memory()
    pin_o = torch.empty((K, B, 32, 128), dtype=torch.bfloat16).pin_memory()
    dbuf = [torch.empty(2 * n_k + n_q, dtype=torch.bfloat16, device=f"cuda:{dev}") for _ in range(2)]
    dk = [d[:n_k].view(knew[0].shape) for d in dbuf]
    dv = [d[n_k:2 * n_k].view(vnew[0].shape) for d in dbuf]
    dq = [d[2 * n_k:].view(qs[0].shape) for d in dbuf]
    do = [torch.empty_like(out) for _ in range(2)]
    cstream = torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def h2d(i):
        sl = i % 2
        with torch.cuda.stream(cstream):
            if i >= 2:
                cstream.wait_event(ev_done[sl])  # buffers of step i-2 are free
            dbuf[sl].copy_(pin_in[i], non_blocking=True)
            ev_in[sl].record(cstream)

    barrier()
    torch.cuda.synchronize(dev)
    e0.record(cstream)
    h2d(0)
    for i in range(K):
        sl = i % 2
        if i + 1 < K:
            h2d(i + 1)
        stream.wait_event(ev_in[sl])
        cache.append_decode(0, ids, dk[sl], dv[sl], dq[sl], do[sl])
        ev_done[sl].record(stream)
        with torch.cuda.stream(cstream):
            cstream.wait_event(ev_done[sl])
            pin_o[i].copy_(do[sl], non_blocking=True)
    stream.wait_stream(cstream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / K, device=f"cuda:{dev}")
    h2d_bytes = dbuf[0].numel() * 2
    d2h = out.numel() * 2
    # region B (after the e2e region, so that e2e runs at region A's lengths): per-call events
    # (the launch duration for the roofline)
    lensB = [cache.seq_info(s)[0] for s in seqs]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize(dev)
    for i in range(K):
        evs[i][0].record(stream)
        cache.append_decode(0, ids, knew[W + K + i], vnew[W + K + i], qs[W + K + i], out)
        evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    dec_ms = [a.elapsed_time(b) for a, b in evs]
    dec_mean = sum(dec_ms) / K
    dec_mean_max = max_over_ranks(dec_mean, device=f"cuda:{dev}")
    # algorithmic bytes per call, averaged over region B's calls (lengths grow by one per step):
    # the decode's K/V + q + out + table, plus the appended rows (read once, written once)
    app_bytes = append_bytes(B, shape)
    bytes_per_call = sum(decode_bytes([L + 1 + i for L in lensB], shape) for i in range(K)) / K + app_bytes
    achieved = bytes_per_call / (dec_mean / 1e3) / 1e9
    clocks = clk.summary()

    cache.close()
    del knew, vnew, qs, pin_in, pin_o
    torch.cuda.empty_cache()

    res = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(step_ms_max, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": headline_config(B, world, args.page_size, docs, tokens),
        "clocks": clocks,
        "e2e": {"value": round(total_tokens / (e2e_ms / 1e3), 1), "unit": "tokens/s",
                "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h,
                "ms_per_step": round(e2e_ms, 5)},
        "gpu_launches": launches,
        # the value is one layer's decode; a Qwen3-8B token step runs 36 of them
        "model_equivalent": {"layers": 36, "tokens_per_s": round(value / 36, 1),
                             "note": "decode attention only (one call per layer), no other layer work"},
        "roofline": {"bound": "hbm", "kernel": "hpa_append_decode per call: fused append + split decode (+ combine)",
                     "timing": "region B: an event pair around each call (region A, the value, has none)",
                     "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / pk["hbm_gbs"], 4), "peak_kind": pk_kind,
                     "frac_vs_nominal_8tbs": round(achieved / NOMINAL_HBM_GBS, 4),
                     "algorithmic_bytes_per_launch": int(bytes_per_call),
                     "launch_ms": round(dec_mean, 5), "traffic": traffic_from_profiles("decode")},
        "decode_kernel_ms": {"mean": round(dec_mean, 5), "min": round(min(dec_ms), 5),
                             "median": round(sorted(dec_ms)[len(dec_ms) // 2], 5),
                             "p90": round(sorted(dec_ms)[min(len(dec_ms) - 1, int(0.9 * len(dec_ms)))], 5),
                             "max_over_ranks_mean": round(dec_mean_max, 5)},
    }

    # ------------------------------------------------------------------ sub-benchmarks
    if not args.no_extra:
        res["prefill"] = bench_prefill(torch, Cache, shape, dev, stream, pk, pk_kind, max_over_ranks, sustained_s=3.0)
        res["lmag"] = bench_lmag(torch, Cache, shape, dev, stream, max(3, min(W, 5)), min(K, 20),
                                 world, max_over_ranks, barrier)
        res["next"] = bench_next(torch, Cache, shape, dev, stream, pk, max_over_ranks)
        res["decode_variants"] = bench_decode_variants(torch, Cache, dev, stream, pk, args.page_size)
        res["next"]["fp8_prefill"] = bench_prefill(torch, Cache, shape, dev, stream, pk, pk_kind, max_over_ranks,
                                                   token_kv_dtype="fp8", batches=(4,))
    if rank == 0 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(budget_s=15.0)
        res["cpu_baseline"]["other_configs"] = cpu_baseline_extra()
    if "prefill" in res:
        # compact prefill figures near the front of the line (the driver keeps the line's head)
        summ = {}
        for key in ("B1", "B4"):
            if key in res["prefill"]:
                pf = res["prefill"][key]
                summ[key] = {"ms": pf["ms"], "tflops": pf["tflops"], "frac": pf["frac"],
                             "sm_mhz": pf["clocks"].get("sm_mhz")}
                if "sustained" in pf:
                    summ[key]["sustained_tflops"] = pf["sustained"]["tflops"]
                    summ[key]["sustained_frac"] = round(pf["sustained"]["tflops"] / pk.get(
                        "bf16_tflops_sustained", pk["bf16_tflops"]), 4)
                    summ[key]["sustained_sm_mhz"] = pf["sustained"]["clocks"].get("sm_mhz")
        summ["peak_burst"] = pk["bf16_tflops"]
        summ["peak_sustained"] = pk.get("bf16_tflops_sustained")
        head = {}
        for k_, v_ in res.items():
            head[k_] = v_
            if k_ == "ms_per_step":
                head["prefill_summary"] = summ
        res = head
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args):
    """--mode head_shard | context_parallel (SURVEY 8(e), NEXT-4b): the configs[1] step with the
    global batch of --batch requests fixed (strong scaling) and each request spread over the N
    ranks. head_shard: rank r holds kv-heads [r H_kv/N, (r+1) H_kv/N) of every request (and their
    G q-heads); step = append + decode of its heads + one NCCL all-gather of the bf16 outputs.
    context_parallel: rank r holds a contiguous block of every request's logical rows (cut at
    128-row boundaries; the last rank holds the tail and receives the appended token); step =
    append (last rank) + hpa_decode_partial + NCCL all-gather of the fp32 partials and LSEs +
    hpa_merge_partials. Time = device time of the whole step, max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2605_09100_b200 import Cache, merge_partials
    from paper_2605_09100_b200.dist import gather_head_shards, gather_partials, head_shard, max_over_ranks
    from workloads import LATENT_ROWS, Shape

    world, rank, dev = init_dist()
    stream = torch.cuda.current_stream(dev)
    pk, pk_kind = peaks()
    B, docs, tokens = args.batch, 8, 4095
    Hq, Hkv, D, P = 32, 8, 128, args.page_size
    K, W = args.steps, args.warmup
    cd = f"cuda:{dev}"

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[dev])

    last = rank == world - 1
    if args.mode == "head_shard":
        kv_lo, kv_hi, q_lo, q_hi = head_shard(Hq, Hkv, rank, world)
        shape = Shape(1, q_hi - q_lo, kv_hi - kv_lo, D, P)
        cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, docs, tokens, K + W + 16, dev, seed=1234 + rank)
        appends = True
        part = f"kv-heads [{kv_lo}, {kv_hi}) and q-heads [{q_lo}, {q_hi}) of every request"
    else:
        blocks = (docs * LATENT_ROWS + tokens + 1) // LATENT_ROWS  # 40 blocks of 128 rows
        if blocks % world:
            sys.exit(f"context_parallel needs {blocks} % world == 0")
        lo, hi = rank * blocks // world, (rank + 1) * blocks // world
        lat = max(0, min(hi, docs) - lo)
        tok = (hi - lo - lat) * LATENT_ROWS - (1 if last else 0)
        shape = Shape(1, Hq, Hkv, D, P)
        cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, lat, tok, K + W + 16 if last else 0, dev,
                                            seed=1234 + rank)
        appends = last
        part = f"logical rows [{lo * LATENT_ROWS}, {hi * LATENT_ROWS}) of every request ({lat} latent sets)"
    ids = np.asarray(seqs, dtype=np.int32)
    ones = np.ones(B, dtype=np.int32)
    g = torch.Generator(device=cd).manual_seed(4321 + rank)
    hq_l, hkv_l = shape.num_q_heads, shape.num_kv_heads
    knew = torch.randn((K + W, 1, B, hkv_l, D), generator=g, device=cd).to(torch.bfloat16)
    vnew = torch.randn((K + W, 1, B, hkv_l, D), generator=g, device=cd).to(torch.bfloat16)
    qs = torch.randn((K + W, B, hq_l, D), generator=g, device=cd).to(torch.bfloat16)
    dec_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]

    def step(i, kk, vv, qq, e=None):
        if appends:
            cache.append_kv(ids, ones, kk, vv)
        if e:
            e[0].record(stream)
        if args.mode == "head_shard":
            o = cache.decode(0, ids, qq)
            if e:
                e[1].record(stream)
            return gather_head_shards(o)
        o, lse = cache.decode_partial(0, ids, qq)
        if e:
            e[1].record(stream)
        if world == 1:
            return merge_partials(o[None], lse[None])
        return merge_partials(*gather_partials(o, lse))

    for i in range(W):
        step(i, knew[i], vnew[i], qs[i])
    torch.cuda.synchronize(dev)
    lens0 = [cache.seq_info(s)[0] for s in seqs]
    launches0 = cache.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(dev)
    barrier()
    torch.cuda.synchronize(dev)
    clk.start()
    t0.record(stream)
    for i in range(K):
        full = step(W + i, knew[W + i], vnew[W + i], qs[W + i], dec_ev[i])
    t1.record(stream)
    torch.cuda.synchronize(dev)
    clk.stop()
    barrier()
    assert full.shape == (B, Hq, D)
    launches = cache.launch_count() - launches0
    step_ms = max_over_ranks(t0.elapsed_time(t1) / K, device=cd)
    dec_ms = sum(a.elapsed_time(b) for a, b in dec_ev) / K
    dec_ms_max = max_over_ranks(dec_ms, device=cd)
    bytes_local = sum(decode_bytes([L + (1 + i if appends else 0) for L in lens0], shape) for i in range(K)) / K
    achieved = bytes_local / (dec_ms / 1e3) / 1e9
    clocks = clk.summary()
    # e2e: pinned host inputs of this rank's shard in, the gathered output out, every step
    pin_k, pin_v, pin_q = knew.cpu().pin_memory(), vnew.cpu().pin_memory(), qs.cpu().pin_memory()
    pin_o = torch.empty((B, Hq, D), dtype=torch.bfloat16).pin_memory()
    dk, dv, dq = torch.empty_like(knew[0]), torch.empty_like(vnew[0]), torch.empty_like(qs[0])
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(K):
        dk.copy_(pin_k[W + i], non_blocking=True)
        dv.copy_(pin_v[W + i], non_blocking=True)
        dq.copy_(pin_q[W + i], non_blocking=True)
        full = step(W + i, dk, dv, dq)
        pin_o.copy_(full, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / K, device=cd)
    h2d = (dk.numel() * 2 + dv.numel() * 2 if appends else 0) + dq.numel() * 2
    cache.close()
    res = {
        "metric": METRIC, "value": round(B / (step_ms / 1e3), 1), "unit": "tokens/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(step_ms, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"configs[1] Qwen3-8B-shaped HPA decode step, {args.mode} over {world} GPU(s)",
                   "mode": args.mode, "global_batch": B, "num_q_heads": Hq, "num_kv_heads": Hkv, "head_dim": D,
                   "page_size": P, "seq_len": docs * LATENT_ROWS + tokens + 1,
                   "parallelism": f"{args.mode} x{world}", "rank0_holds": part,
                   "l2": "working set >> 126 MB L2 per GPU at N <= 8 (no flush needed)"},
        "clocks": clocks,
        "e2e": {"value": round(B / (e2e_ms / 1e3), 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": B * Hq * D * 2, "ms_per_step": round(e2e_ms, 5)},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "hpa decode of this rank's shard", "achieved": round(achieved, 1),
                     "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
                     "peak_kind": pk_kind, "algorithmic_bytes_per_launch": int(bytes_local),
                     "launch_ms": round(dec_ms, 5), "max_over_ranks_ms": round(dec_ms_max, 5), "traffic": None},
        "collective": {"head_shard": "all_gather_into_tensor of bf16 [B][Hq/N][d] (NCCL)",
                       "context_parallel": "2 x all_gather_into_tensor of fp32 [B][Hq][d] + [B][Hq] (NCCL), "
                                           "then hpa_merge_partials"}[args.mode] if world > 1 else "none (N = 1)",
    }
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


def traffic_from_profiles(kernel: str):
    """dram bytes (read + write) per launch from the committed ncu summary, if present."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(kernel)
    except Exception:
        return None


def bench_prefill(torch, Cache, shape, dev, stream, pk, pk_kind, max_over_ranks, reps=5, token_kv_dtype="bf16",
                  batches=(1, 4), windows=5, sustained_s=0.0):
    """configs[2]: C = 2048 new rows over 8 latent sets (1024 rows) + 16384 cached token rows.
    token_kv_dtype "fp8" (NEXT-4c): the token pages are fp8; each call first dequantizes
    them into temporary bf16 pages (included in the time)."""
    out = {}
    for bp in batches:
        c_rows, prior_tok = 2048, 16384
        tok_pages = bp * (math.ceil((prior_tok + c_rows) / shape.page_size) + 1)  # fp8: temporaries of a call
        cache, seqs, _ = build_decode_cache(torch, Cache, shape, bp, 8, prior_tok + c_rows, 0, dev, seed=777,
                                            token_kv_dtype=token_kv_dtype,
                                            bf16_headroom_pages=tok_pages if token_kv_dtype == "fp8" else 0)
        g = torch.Generator(device=f"cuda:{dev}").manual_seed(99)
        q = torch.randn((bp * c_rows, 32, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
        o = torch.empty_like(q)
        for _ in range(3):
            cache.prefill(0, seqs, [c_rows] * bp, q, o)
        torch.cuda.synchronize(dev)
        # `windows` timed windows of `reps` calls each (the tensor-bound kernel runs into the
        # board power cap within a few ms, so single windows scatter by ~10 %): median window
        clk = ClockSampler(dev)
        clk.start()
        win = []
        for _ in range(windows):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                cache.prefill(0, seqs, [c_rows] * bp, q, o)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            win.append(e0.elapsed_time(e1) / reps)
        clk.stop()
        ms = max_over_ranks(statistics.median(win), device=f"cuda:{dev}")
        flops = bp * prefill_flops(8 * 128 + prior_tok, c_rows, shape)
        tf = flops / (ms / 1e3) / 1e12
        out[f"B{bp}"] = {"ms": round(ms, 4), "tflops": round(tf, 1),
                         "frac": round(tf / pk["bf16_tflops"], 4), "peak": pk["bf16_tflops"],
                         "peak_kind": f"{pk_kind} bf16 dense (burst)",
                         "frac_vs_nominal_2250": round(tf / NOMINAL_BF16_TFLOPS, 4),
                         "flops": flops, "ms_windows": [round(w, 4) for w in win],
                         "tflops_best_window": round(flops / (min(win) / 1e3) / 1e12, 1),
                         "plan": cache.prefill_plan_info(), "clocks": clk.summary()}
        if sustained_s > 0 and bp == max(batches):
            # the same call back to back for sustained_s seconds: the tensor-bound kernel runs into
            # the board power limit (1000 W) and the SM clock drops from 1965 to ~1630 MHz
            clk2 = ClockSampler(dev)
            clk2.start()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n, t_end = 0, time.time() + sustained_s
            e0.record(stream)
            while time.time() < t_end:
                for _ in range(10):
                    cache.prefill(0, seqs, [c_rows] * bp, q, o)
                n += 10
                torch.cuda.synchronize(dev)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            clk2.stop()
            ms_s = max_over_ranks(e0.elapsed_time(e1) / n, device=f"cuda:{dev}")
            out[f"B{bp}"]["sustained"] = {"seconds": sustained_s, "calls": n, "ms": round(ms_s, 4),
                                          "tflops": round(flops / (ms_s / 1e3) / 1e12, 1),
                                          "clocks": clk2.summary()}
        cache.close()
        del q, o
    out["workload"] = "configs[2] chunked prefill C=2048 over 1024 latent + 16384 cached token rows"
    if token_kv_dtype == "bf16":
        out["roofline"] = {"bound": "tensor", "unit": "TFLOP/s", "traffic": traffic_from_profiles("prefill")}
    return out


def bench_lmag(torch, Cache, shape, dev, stream, W, K, world, max_over_ranks, barrier):
    """configs[3]: B=256 decode; each step replaces latent set (step mod 8) of every
    request from a device staging buffer (one batched install), appends 1 token, decodes."""
    import numpy as np
    B = 256
    cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, 8, 4095, 2 * K + W + 8, dev, seed=555)
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(1)
    stage = torch.randn((2, B, 1, 2, 128, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    kn = torch.randn((1, B, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    vn = torch.randn((1, B, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    q = torch.randn((B, 32, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    o = torch.empty_like(q)
    ids = np.asarray(seqs, dtype=np.int32)
    sets = [np.full(B, k, dtype=np.int32) for k in range(8)]
    # region A (the step rate): install + fused append/decode back to back, no events between;
    # region B: the same steps with events around each call (install / decode breakdown)
    for i in range(W):
        cache.latent_install_packed(ids, sets[i % 8], stage[i % 2])
        cache.append_decode(0, ids, kn, vn, q, o)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize(dev)
    a0.record(stream)
    for i in range(W, W + K):
        cache.latent_install_packed(ids, sets[i % 8], stage[i % 2])
        cache.append_decode(0, ids, kn, vn, q, o)
    a1.record(stream)
    torch.cuda.synchronize(dev)
    step = max_over_ranks(a0.elapsed_time(a1) / K, device=f"cuda:{dev}")
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    for i in range(K):
        e = ev[i]
        e[0].record(stream)
        cache.latent_install_packed(ids, sets[i % 8], stage[i % 2])
        e[1].record(stream)
        cache.append_decode(0, ids, kn, vn, q, o)
        e[2].record(stream)
    torch.cuda.synchronize(dev)
    inst = max_over_ranks(sum(a[0].elapsed_time(a[1]) for a in ev) / K, device=f"cuda:{dev}")
    dec = max_over_ranks(sum(a[1].elapsed_time(a[2]) for a in ev) / K, device=f"cuda:{dev}")
    lens = [cache.seq_info(s)[0] for s in seqs]
    inst_bytes = 2 * B * 128 * 8 * 128 * 2 * 2  # K+V, read + write
    dbytes = decode_bytes([L - K // 2 for L in lens], shape) + append_bytes(B, shape)
    cache.close()
    # O(1) check (SURVEY 8(d) configs[3]): the install must not depend on the token context.
    # Device time only: a 20 ms spin kernel holds the stream while the host enqueues the 10
    # install calls, so the events bracket back-to-back device work and the host planning
    # (timed separately, per call) is hidden behind the spin.
    o1, o1_host = {}, {}
    for tokens in (1024, 8192, 32768):
        cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, 8, tokens, 0, dev, seed=556)
        ids = np.asarray(seqs, dtype=np.int32)
        for _ in range(3):
            cache.latent_install_packed(ids, sets[0], stage[0])
        dev_us, host_us = [], []
        for _rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            torch.cuda._sleep(40_000_000)  # ~20 ms of device spin at 1.9 GHz
            e0.record(stream)
            h0 = time.perf_counter()
            for k in range(10):
                cache.latent_install_packed(ids, sets[k % 8], stage[k % 2])
            host_us.append((time.perf_counter() - h0) / 10 * 1e6)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            dev_us.append(e0.elapsed_time(e1) / 10 * 1e3)
        o1[str(tokens)] = round(statistics.median(dev_us), 1)
        o1_host[str(tokens)] = round(statistics.median(host_us), 1)
        cache.close()
        torch.cuda.empty_cache()
    return {"workload": "configs[3] LMAG: B=256 decode + per-request latent set replacement each step",
            "tokens_per_s": round(B * world / (step / 1e3), 1),
            "tokens_per_s_without_install": round(B * world / ((step - inst) / 1e3), 1),
            "step_ms": round(step, 4), "install_ms": round(inst, 4), "decode_ms": round(dec, 4),
            "timing": "step: install + hpa_append_decode back to back; install / decode: separate pass "
                      "with events around each call",
            "install_gbs": round(inst_bytes / (inst / 1e3) / 1e9, 1),
            "decode_gbs": round(dbytes / (dec / 1e3) / 1e9, 1),
            "install_us_vs_reasoning_tokens": o1,
            "install_host_us_vs_reasoning_tokens": o1_host,
            "install_timing": "device time per batched call (256 requests x 128 rows), host enqueue hidden "
                              "behind a spin kernel; host planning per call reported separately"}


def bench_next(torch, Cache, shape, dev, stream, pk, max_over_ranks):
    """Measurements for the SURVEY §8(f) NEXT rows (one layer each)."""
    import numpy as np
    from workloads import LATENT_ROWS
    out = {}
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(31)
    # NEXT-1: in-cache compression of a 4096-token document into m = 128 latent rows, B = 64
    B, n_doc, m = 64, 4096, LATENT_ROWS
    moved = B * m * shape.num_kv_heads * shape.head_dim * 2 * 2 * 2  # K+V rows read + written
    res = {}
    for mode in ("batch", "per_call"):  # hpa_seq_compress_batch (one launch) / hpa_seq_compress per request
        cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, 8, n_doc + m, 0, dev, seed=41)
        free0 = cache.stats()[0]
        torch.cuda.synchronize(dev)
        e0, e1 = ev(), ev()
        t0 = time.perf_counter()
        e0.record(stream)
        if mode == "batch":
            cache.compress_batch(seqs, [n_doc] * B, [m] * B)
        else:
            for s in seqs:
                cache.compress(s, n_doc, m)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        res[mode] = (e0.elapsed_time(e1), time.perf_counter() - t0, cache.stats()[0] - free0)
        cache.close()
    ms, host_s, freed = res["batch"]
    out["compress"] = {"workload": f"B={B}: 4096-token document + 128 meta-latent rows -> 128-row latent set, "
                                   "one hpa_seq_compress_batch call",
                       "ms_total": round(ms, 4), "us_per_document": round(ms * 1e3 / B, 2),
                       "host_us_per_document": round(host_s * 1e6 / B, 1),
                       "pages_freed": freed, "moved_gbs": round(moved / (ms / 1e3) / 1e9, 1),
                       "per_call_ms_total": round(res["per_call"][0], 4),
                       "per_call_host_us_per_document": round(res["per_call"][1] * 1e6 / B, 1)}
    # NEXT-2: decode with 8 document sets shared by all 64 requests vs private copies
    B, tokens = 64, 4095
    P = shape.page_size
    pages = 8 * (LATENT_ROWS // P) + B * (-(-(tokens + 64) // P) + 1) + 64
    cache = Cache(1, 32, 8, 128, P, pages, B + 1, 8 * (LATENT_ROWS // P) + (tokens + 64) // P + 2, dev, 99)
    owner = cache.seq_create()
    kv = torch.randn((8, 1, 2, LATENT_ROWS, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    for i in range(8):
        cache.latent_install(owner, -1, kv[i])
    seqs = [cache.seq_create() for _ in range(B)]
    for s in seqs:
        for i in range(8):
            cache.latent_share(s, owner, i)
    k = torch.randn((1, B * tokens, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    cache.append_kv(seqs, [tokens] * B, k, k)
    q = torch.randn((B, 32, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    o = torch.empty_like(q)
    ids = np.asarray(seqs, dtype=np.int32)

    def time_decode(cascade, n=20):
        cache.set_decode_cascade(cascade)
        for _ in range(3):
            cache.decode(0, ids, q, o)
        torch.cuda.synchronize(dev)
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(n):
            cache.decode(0, ids, q, o)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / n, cache.decode_plan_info()

    ms_off, _ = time_decode(False)
    ms, plan = time_decode(True)
    lens = [cache.seq_info(s)[0] for s in seqs]
    out["shared_sets"] = {"workload": "B=64 decode, the same 8 latent sets shared by every request (stored once)",
                          "decode_ms": round(ms, 4), "tokens_per_s": round(B / (ms / 1e3), 1),
                          "logical_gbs": round(decode_bytes(lens, shape) / (ms / 1e3) / 1e9, 1),
                          "cascade_group_units": plan["group_units"],
                          "decode_ms_cascade_off": round(ms_off, 4),
                          "latent_pages_stored": 8 * (LATENT_ROWS // P),
                          "latent_pages_if_private": B * 8 * (LATENT_ROWS // P)}
    cache.close()
    # NEXT-2 cascade: B = 64 requests forked from one 16384-token prompt (hpa_seq_fork: the
    # prompt's pages stored once), each with 1024 own tokens; the prompt is read once per group
    # of 32 / G = 8 requests (cascade) or once per request (off)
    B, n_prompt, n_own = 64, 16384, 1024
    pages = n_prompt // P + B * (n_own // P + 2) + 64
    cache = Cache(1, 32, 8, 128, P, pages, B + 1, (n_prompt + n_own) // P + 4, dev, 99)
    src = cache.seq_create()
    kp = torch.randn((1, n_prompt, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    cache.append_kv([src], [n_prompt], kp, kp.flip(1))
    seqs = [cache.seq_fork(src, n_prompt) for _ in range(B)]
    ko = torch.randn((1, B * n_own, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    cache.append_kv(seqs, [n_own] * B, ko, ko.flip(1))
    ids = np.asarray(seqs, dtype=np.int32)
    ms_off, plan_off = time_decode(False)
    ms, plan = time_decode(True)
    lens = [cache.seq_info(s)[0] for s in seqs]

    def time_steps(cascade, n=20):  # the serving step: hpa_append_decode (append + decode, fused)
        cache.set_decode_cascade(cascade)
        kn = torch.randn((n + 3, 1, B, 8, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
        for i in range(3):
            cache.append_decode(0, ids, kn[i], kn[i], q, o)
        torch.cuda.synchronize(dev)
        e0, e1 = ev(), ev()
        e0.record(stream)
        for i in range(n):
            cache.append_decode(0, ids, kn[3 + i], kn[3 + i], q, o)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / n

    step_off = time_steps(False)
    step_on = time_steps(True)
    row_bytes = shape.num_kv_heads * shape.head_dim * 2 * 2  # K + V of one row, all KV heads
    groups = -(-B // (32 // (shape.num_q_heads // shape.num_kv_heads)))
    phys = (groups * n_prompt + B * n_own) * row_bytes + 2 * B * shape.num_q_heads * shape.head_dim * 2
    out["prefix_cascade"] = {
        "workload": f"B={B} forks of one {n_prompt}-token prompt + {n_own} own tokens each (P:L251 prefix KV)",
        "decode_ms": round(ms, 4), "tokens_per_s": round(B / (ms / 1e3), 1),
        "decode_ms_cascade_off": round(ms_off, 4), "speedup_vs_off": round(ms_off / ms, 2),
        "cascade_group_units": plan["group_units"], "units": plan["units"],
        "logical_gbs": round(decode_bytes(lens, shape) / (ms / 1e3) / 1e9, 1),
        "physical_bytes": phys, "physical_gbs": round(phys / (ms / 1e3) / 1e9, 1),
        "physical_frac_of_copy_peak": round(phys / (ms / 1e3) / 1e9 / pk["hbm_gbs"], 4),
        "logical_gbs_cascade_off": round(decode_bytes(lens, shape) / (ms_off / 1e3) / 1e9, 1),
        "append_decode_step_ms": round(step_on, 4), "append_decode_step_ms_cascade_off": round(step_off, 4)}
    cache.close()
    # NEXT-3: LMAG-style replacement from pinned host payloads (copy stream) overlapped with decode
    B = 256
    cache, seqs, _ = build_decode_cache(torch, Cache, shape, B, 8, 4095, 16, dev, seed=43)
    ids = np.asarray(seqs, dtype=np.int32)
    host = torch.randn((2, B, 1, 2, LATENT_ROWS, 8, 128), generator=g, device=f"cuda:{dev}").to(
        torch.bfloat16).cpu().pin_memory()
    q = torch.randn((B, 32, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    o = torch.empty_like(q)
    sets = [np.full(B, k, dtype=np.int32) for k in range(8)]
    for i in range(2):
        cache.latent_install_host(ids, sets[i], host[i % 2])
        cache.decode(0, ids, q, o)
    torch.cuda.synchronize(dev)
    e0, e1 = ev(), ev()
    e0.record(stream)
    steps = 6
    for i in range(steps):
        cache.latent_install_host(ids, sets[i % 8], host[i % 2])
        cache.decode(0, ids, q, o)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    payload = B * LATENT_ROWS * 8 * 128 * 2 * 2
    out["host_staged_install"] = {"workload": "B=256: replace one 128-row set per request from pinned host + decode",
                                  "step_ms": round(ms, 4), "h2d_bytes_per_step": payload,
                                  "h2d_gbs": round(payload / (ms / 1e3) / 1e9, 1)}
    cache.close()
    # NEXT-4a: GRC mask-out-span prefill: C = 2048 queries, segment 1 = the first 8192 token rows
    n1, c_rows = 8192, 2048
    cache, seqs, _ = build_decode_cache(torch, Cache, shape, 1, 8, 16384 + c_rows, 0, dev, seed=45)
    q = torch.randn((c_rows, 32, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
    span = [(1024, 1024 + n1, 1024 + 16384)]  # all C queries are in segment 3; segment 1 follows the latents
    for _ in range(2):
        cache.prefill_span(0, seqs, [c_rows], span, q)
    torch.cuda.synchronize(dev)
    e0, e1 = ev(), ev()
    e0.record(stream)
    for _ in range(5):
        cache.prefill_span(0, seqs, [c_rows], span, q)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / 5
    flops = prefill_flops(8 * 128 + 16384 - n1, c_rows, shape)  # visible pairs only
    out["span_prefill"] = {"workload": "configs[2] with a masked 8192-row segment 1 (GRC Eq. 1 mask)",
                           "ms": round(ms, 4), "tflops_visible": round(flops / (ms / 1e3) / 1e12, 1)}
    cache.close()
    return out


# ----------------------------------------------------------------------------- CPU baseline
def _oracle_requests(n, seed=11):
    """n requests of configs[1] shape built in the oracle's own cache model (CPU)."""
    import torch
    from oracle import OracleCache
    from workloads import Draw, rag_decode
    w = rag_decode(1)
    sh = w.shape
    c = OracleCache(1, 32, 8, 128, 16)
    d = Draw(seed)
    for s in range(n):
        c.create_seq(s)
        for kind, m in w.seqs[0].segments:
            if kind == "latent":
                c.install(s, -1, d.latent(sh, m).to(torch.float64).numpy())
            else:
                k, v = d.tokens(sh, m)
                c.append(s, k.to(torch.float64).numpy(), v.to(torch.float64).numpy())
    qs = d.queries(sh, n).to(torch.float64).numpy()
    return c, qs, sh


def _oracle_worker(args):
    """One host process: builds its own request(s) and times oracle decodes for budget_s (1 BLAS thread)."""
    seed, budget_s = args
    from threadpoolctl import threadpool_limits
    from oracle.hpa_oracle import decode_reference
    c, qs, sh = _oracle_requests(1, seed=seed)
    done, t_work = 0, 0.0
    with threadpool_limits(1):
        while t_work < budget_s:
            t = time.perf_counter()
            decode_reference(c, 0, 0, qs[0], sh.scale)
            t_work += time.perf_counter() - t
            done += 1
    return done, t_work


def cpu_baseline(budget_s: float = 15.0):
    """The fp64 oracle as it stands on a bounded sample of configs[1] requests (SURVEY 8(d)
    "Oracle timing beside it"): first on 1 host core (BLAS pinned to one thread), then on all
    host cores (one process per core, each with its own request, BLAS pinned to one thread).
    `value` / `cores` describe the all-cores run; the 1-core figure is reported beside it."""
    import multiprocessing as mp
    from threadpoolctl import threadpool_limits
    from oracle.hpa_oracle import decode_reference
    n_req = 4
    c, qs, sh = _oracle_requests(n_req)
    done, t_work = 0, 0.0
    half = budget_s / 2
    with threadpool_limits(1):
        while t_work < half:
            s = done % n_req
            t = time.perf_counter()
            decode_reference(c, s, 0, qs[s], sh.scale)
            t_work += time.perf_counter() - t
            done += 1
    one = done / t_work
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_oracle_worker, [(100 + i, half) for i in range(cores)])
    wall = time.perf_counter() - t0
    all_cores = sum(d / t for d, t in res)  # each process's own rate (spawn/setup excluded)
    kv_gb = 5120 * 8 * 128 * 2 * 2 / 1e9     # bf16-equivalent KV bytes per configs[1] request
    return {"value": round(all_cores, 3), "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "single_core_value": round(one, 3), "kv_gbs_processed": round(all_cores * kv_gb, 3),
            "sample": f"{done} decode queries over {n_req} configs[1] requests (Lb=5120, 32 q-heads) on 1 core "
                      f"({t_work:.1f} s of fp64 numpy work), then {sum(d for d, _ in res)} queries on {cores} "
                      f"processes x {half:.1f} s (1 BLAS thread each; {wall:.1f} s wall incl. spawn)"}


def _oracle_prefill_group_worker(args):
    """configs[2] B_p = 1, one GQA group: this process draws the request's rows of kv-head h
    (workloads.Draw, the bench recipe) and times oracle.attend for the sampled query rows of
    the group's G q-heads (1 BLAS thread). Returns (flops, seconds)."""
    seed, h, rows, budget_s = args
    import numpy as np
    import torch
    from threadpoolctl import threadpool_limits
    from oracle import attend
    from workloads import Shape
    C, prior, G, d = 2048, 1024 + 16384, 4, 128
    lb = prior + C
    g = torch.Generator().manual_seed(seed + h)
    k = torch.randn((1, lb, d), generator=g).to(torch.bfloat16).double().numpy()
    v = torch.randn((1, lb, d), generator=g).to(torch.bfloat16).double().numpy()
    q = torch.randn((C, G, d), generator=g).to(torch.bfloat16).double().numpy()
    scale = Shape(1, 32, 8, d, 16).scale
    flops, t_work, n = 0, 0.0, 0
    with threadpool_limits(1):
        while t_work < budget_s:
            t = rows[n % len(rows)]
            i = prior + t
            t0 = time.perf_counter()
            attend(q[t:t + 1], k[:, :i + 1], v[:, :i + 1], scale)
            t_work += time.perf_counter() - t0
            flops += 4 * G * d * (i + 1)
            n += 1
    return flops, t_work


def cpu_baseline_extra(budget_s: float = 8.0):
    """SURVEY 8(d) "Oracle timing beside it" for the other configs (the fp64 oracle as it
    stands, host cores of this box): configs[0] latency, configs[2] B_p = 1 prefill on sampled
    query rows (extrapolated to the full chunk), configs[3] LMAG step on 8 requests
    (extrapolated to B = 256). Each sub-object states its sample and core count."""
    import multiprocessing as mp
    import numpy as np
    import torch
    from threadpoolctl import threadpool_limits
    from oracle import OracleCache, attend
    from oracle.hpa_oracle import decode_reference
    from workloads import Draw, tiny_decode
    out = {}
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    # configs[0]: tiny decode latency
    w = tiny_decode("a")
    sh = w.shape
    c = OracleCache(1, 2, 1, 64, 16)
    dr = Draw(5)
    c.create_seq(0)
    for kind, m in w.seqs[0].segments:
        if kind == "latent":
            c.install(0, -1, dr.latent(sh, m).double().numpy())
        else:
            k, v = dr.tokens(sh, m)
            c.append(0, k.double().numpy(), v.double().numpy())
    qt = dr.queries(sh, 1).double().numpy()[0]
    lat = []
    with threadpool_limits(1):
        t_end = time.perf_counter() + 1.0
        while time.perf_counter() < t_end:
            t0 = time.perf_counter()
            decode_reference(c, 0, 0, qt, sh.scale)
            lat.append(time.perf_counter() - t0)
    out["configs0_tiny_decode"] = {"value": round(statistics.median(lat) * 1e6, 2), "unit": "us per decode",
                                   "cores": 1, "kind": "oracle",
                                   "sample": f"{len(lat)} decodes of the tiny config (Lb = 64) in 1 s, median"}
    # configs[2]: B_p = 1 prefill, sampled rows
    C, prior = 2048, 1024 + 16384
    full_flops = 4 * 32 * 128 * (C * prior + C * (C + 1) // 2)
    rows = [int(x) for x in np.linspace(0, C - 1, 16)]
    f1, t1 = _oracle_prefill_group_worker((2025, 0, rows, budget_s / 2))
    n_proc = min(cores, 8)
    with mp.get_context("spawn").Pool(n_proc) as pool:
        res = pool.map(_oracle_prefill_group_worker, [(2025, h, rows, budget_s / 2) for h in range(n_proc)])
    rate_all = sum(f / t for f, t in res)
    out["configs2_prefill_B1"] = {
        "value": round(rate_all / 1e9, 3), "unit": "GFLOP/s", "cores": n_proc, "kind": "oracle",
        "single_core_gflops": round(f1 / t1 / 1e9, 3),
        "extrapolated_s_per_request": round(full_flops / rate_all, 1),
        "extrapolated_s_per_request_1core": round(full_flops / (f1 / t1), 1),
        "sample": f"oracle.attend on 16 query rows spread over the C = 2048 chunk (each over its causal prefix "
                  f"of {prior}+t+1 keys), one GQA group (4 q-heads, 1 kv-head) per process, {budget_s / 2:.1f} s "
                  f"per process; FLOPs counted as 4 G d (i+1) per row, extrapolated to the full request "
                  f"({full_flops / 1e12:.3f} TFLOP)"}
    # configs[3]: LMAG step (replace set step mod 8, append 1 token, decode) on 8 requests
    n_req = 8
    oc, qs, shp = _oracle_requests(n_req, seed=31)
    dr = Draw(32)
    steps, t_work = 0, 0.0
    with threadpool_limits(1):
        while t_work < budget_s / 2:
            inp = [(dr.latent(shp, 128).double().numpy(), *(x.double().numpy() for x in dr.tokens(shp, 1)))
                   for _ in range(n_req)]
            t0 = time.perf_counter()
            for s in range(n_req):
                oc.install(s, steps % 8, inp[s][0])
                oc.append(s, inp[s][1], inp[s][2])
                decode_reference(oc, s, 0, qs[s], shp.scale)
            t_work += time.perf_counter() - t0
            steps += 1
    req_s = steps * n_req / t_work
    out["configs3_lmag"] = {"value": round(req_s, 3), "unit": "tokens/s", "cores": 1, "kind": "oracle",
                            "extrapolated_ms_per_B256_step": round(256 / req_s * 1e3, 1),
                            "sample": f"{steps} LMAG steps over {n_req} requests (Lb ~ 5120; per request: replace a "
                                      f"128-row latent set, append 1 token, decode; input draws excluded), "
                                      f"extrapolated linearly to B = 256"}
    return out


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    from threadpoolctl import threadpool_limits
    from oracle.hpa_oracle import decode_reference
    from workloads import Draw
    n_req = 2
    c, qs, sh = _oracle_requests(n_req, seed=21)
    K, W = args.steps, args.warmup
    # each step = one request's step of the workload: append its new K/V row, then decode
    d = Draw(5)
    rows = [tuple(t.to(torch.float64).numpy() for t in d.tokens(sh, 1)) for _ in range(W + K)]
    with threadpool_limits(1):
        for i in range(W):
            c.append(i % n_req, *rows[i])
            decode_reference(c, i % n_req, 0, qs[i % n_req], sh.scale)
        t = time.perf_counter()
        for i in range(K):
            c.append(i % n_req, *rows[W + i])
            decode_reference(c, i % n_req, 0, qs[i % n_req], sh.scale)
        el = time.perf_counter() - t
    value = K / el
    res = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "tokens/s",
           "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": round(el / K * 1e3, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": headline_config(64, world, args.page_size),
           "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": 1, "kind": "oracle",
                            "sample": f"{K} timed request steps (append the request's new K/V row, then decode its "
                                      f"query) over {n_req} requests of the workload's shape (Lb ~ 5120), fp64 numpy, "
                                      f"1 core; the GPU arm runs 64 requests per step"},
           "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    elif a.sweep:
        bench_sweep(a)
    elif a.mode != "request":
        run_sharded(a)
    else:
        run_ours(a)
