"""Top source lines by warp-stall samples from an ncu report's cuda,sass source view.
Usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > x.csv; python scripts/ncu_lines.py x.csv [N]"""
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out, fname, h = [], "", None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        h = r
    elif h and r and r[0] not in ("", "Function Name"):
        out.append((num(r[h.index("Warp Stall Sampling (All Samples)")]), fname, r[0], r[1]))
tot = sum(o[0] for o in out)
print(f"total samples {tot:.0f}")
for s, f, ln, src in sorted(out, key=lambda o: -o[0])[:n]:
    print(f"{f}:{ln:>5} {s:6.0f} {100 * s / tot:5.1f}%  {src[:100]}")
