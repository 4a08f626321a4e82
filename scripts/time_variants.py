"""The bench's decode_variants (ragged, P=64, fp8) alone, one line (planner knobs via env)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
pk, _ = bench.peaks()
out = bench.bench_decode_variants(torch, Cache, 0, torch.cuda.current_stream(0), pk, 16)
print(f"C0={os.environ.get('HPA_PLAN_C0', '-')}: " + " | ".join(f"{k} {v['decode_ms'] * 1e3:.1f} us" for k, v in out.items()),
      flush=True)
