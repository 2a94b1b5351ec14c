#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launches, total/avg device time and share of all launches."""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    m = re.search(r"(\w+)(<[^()]*>)?\(", name)
    base = m.group(1) if m else name[:40]
    targ = (m.group(2) or "") if m else ""
    if "double" in targ:
        base += "<f64>"
    elif "float" in targ:
        base += "<f32>"
    return base


def main(path, out=None, window=None):
    """window = (first_kernel_substring, last_kernel_substring): restrict to the
    launches from the first match of the former to the last match of the latter
    that precedes the next match of the former (one complete step)."""
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
    note = ""
    if window:
        first, last = window
        i0 = next(i for i, r in enumerate(rows) if first in r["Kernel Name"])
        ilast = max(i for i, r in enumerate(rows) if last in r["Kernel Name"])
        rows = rows[i0: ilast + 1]
        note = f" (window: first '{first}' .. last '{last}')"
    for row in rows:
        k = short(row["Kernel Name"])
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "ns")
        v *= {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1e-9)
        tot[k] += v
        cnt[k] += 1
    all_t = sum(tot.values())
    rows = sorted(tot, key=lambda k: -tot[k])
    lines = [f"# {path}{note}: {sum(cnt.values())} launches, {all_t*1e3:.2f} ms total device time (cold-cache, serialised)",
             f"{'kernel':40s} {'launches':>9s} {'total_ms':>11s} {'avg_us':>9s} {'share':>7s}"]
    for k in rows:
        lines.append(f"{k:40s} {cnt[k]:9d} {tot[k]*1e3:11.3f} {tot[k]/cnt[k]*1e6:9.2f} {tot[k]/all_t*100:6.2f}%")
    txt = "\n".join(lines)
    print(txt)
    if out:
        open(out, "w").write(txt + "\n")


if __name__ == "__main__":
    win = tuple(sys.argv[3].split("..")) if len(sys.argv) > 3 else None
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, win)
