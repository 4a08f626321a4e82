"""Side-by-side numeric leaves of two bench JSON lines. Usage: python scripts/bench_diff.py a.json b.json [filter]"""
import json
import sys


def leaves(d, pre=""):
    if isinstance(d, dict):
        for k, v in d.items():
            yield from leaves(v, f"{pre}.{k}" if pre else k)
    elif isinstance(d, (int, float)) and not isinstance(d, bool):
        yield pre, d


def load(p):
    return json.loads([ln for ln in open(p) if ln.startswith("{")][-1])


a, b = dict(leaves(load(sys.argv[1]))), dict(leaves(load(sys.argv[2])))
flt = sys.argv[3] if len(sys.argv) > 3 else ""
for k in a:
    if k in b and flt in k and a[k] != b[k]:
        r = b[k] / a[k] if a[k] else float("nan")
        print(f"{k:70s} {a[k]:>14.4f} {b[k]:>14.4f}  x{r:.3f}")
