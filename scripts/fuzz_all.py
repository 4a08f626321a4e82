"""Long all-API random fuzz against the oracle (bug hunting; driver in tests/hpa_fuzz_all.py).
Usage: SEEDS=0,1 OPS=600 [FP8=1] [CHECK=50] python scripts/fuzz_all.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.hpa_fuzz_all import run  # noqa: E402

if __name__ == "__main__":
    fp8 = os.environ.get("FP8") == "1"
    for sd in [int(x) for x in os.environ.get("SEEDS", "0").split(",")]:
        shp, st = run(sd, int(os.environ.get("OPS", "600")), fp8, int(os.environ.get("CHECK", "50")))
        print(f"seed {sd} shape {shp} fp8={fp8}: {st}", flush=True)
