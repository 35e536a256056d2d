#!/usr/bin/env python3
"""Top source lines by warp-stall samples from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
si = hdr.index("Warp Stall Sampling (All Samples)")
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: hdr.index(c) for c in cols}
lines = [r for r in rows if len(r) > si and r[0].isdigit()]
g = lambda r, i: int(r[i]) if r[i].isdigit() else 0
tot = sum(g(r, si) for r in lines) or 1
print("total samples", tot)
for r in sorted(lines, key=lambda r: -g(r, si))[:n]:
    top = sorted(((g(r, idx[c]), c[6:]) for c in cols), reverse=True)[:3]
    print(f"{g(r, si):7d} {100 * g(r, si) / tot:5.1f}% L{r[0]:>4} {r[1].strip()[:60]:60s} {top}")
