"""The bench's NEXT-row measurements alone (bench.bench_next), one JSON object."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_09100_b200 import Cache  # noqa: E402
from paper_2605_09100_b200.dist import max_over_ranks  # noqa: E402
from workloads import qwen3_8b_shape  # noqa: E402

pk, _ = bench.peaks()
out = bench.bench_next(torch, Cache, qwen3_8b_shape(16), 0, torch.cuda.current_stream(0), pk, max_over_ranks)
print(json.dumps({k: v for k, v in out.items() if k in ("shared_sets", "prefix_cascade")}, indent=1))
