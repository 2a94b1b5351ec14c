#!/usr/bin/env python
"""Per-CUDA-source-line warp-stall samples from `ncu -i rep --page source
--csv --print-source cuda,sass` (needs -lineinfo): top lines and their two
leading stall reasons."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
col = {h: i for i, h in enumerate(hdr) if h}
samp = col["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
line_s = defaultdict(int)
line_st = defaultdict(lambda: defaultdict(int))
line_src = {}
cur = None
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        continue
    if r[0].strip():
        if not r[0].strip().isdigit():
            continue
        cur = int(r[0])
        line_src[cur] = r[1]
    try:
        v = int(r[samp] or 0)
    except ValueError:
        continue
    line_s[cur] += v
    for h in stalls:
        try:
            line_st[cur][h] += int(r[col[h]] or 0)
        except (ValueError, KeyError):
            pass
tot = sum(line_s.values()) or 1
print(f"total samples {tot}")
for ln, v in sorted(line_s.items(), key=lambda x: -x[1])[:top_n]:
    st = sorted(line_st[ln].items(), key=lambda x: -x[1])[:2]
    print(f"{ln:5d} {100 * v / tot:5.1f}% {line_src.get(ln, '')[:70]:70s} {st}")
