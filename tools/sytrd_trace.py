#!/usr/bin/env python
"""Phase timing of the sytrd panel kernel (k_tridiag.cu) from a diagnostics
build (MPJ_NVCC_EXTRA=-DMPJ_SYTRD_TRACE): runs the tridiagonalisation of an
n x n matrix and prints, for the last panel, per column: phase A (first CTA
start -> last CTA reaching barrier 1), barrier 1 wait, symv (per-CTA span,
max), dots, barrier 2, phase C -- medians over the panel's columns."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2211_03339_b200 as mpj  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
k0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
mpj.lib().mpjacobi_debug_sytrd_trace_panel(k0)
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(n, n, device="cuda", generator=g)
A = (A + A.T) / 2
for first in (True, False):
    d, e, tau, _ = mpj.sytrd(A)
buf = np.zeros(64 * 12 * 320, dtype=np.uint64)
mpj.lib().mpjacobi_debug_sytrd_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)))
t = buf.reshape(64, 12, 320).astype(np.float64)
G = int((t[0, 0] > 0).sum())
t = t[:, :, :G]
rows = []
for jj in range(64):
    ev = t[jj]
    if not ev[0].any():
        continue
    rows.append([
        ev[1].max() - ev[0].min(),        # phase A until the last CTA arrives at barrier 1
        (ev[10][ev[10] > 0] - ev[0][ev[10] > 0]).max() if (ev[10] > 0).any() else 0.0,   # A: own-row work
        ev[2].max() - ev[1].max(),        # barrier 1 release latency
        (ev[3] - ev[2]).max(),            # symv: the slowest CTA
        (ev[4] - ev[3]).max(),            # q + dots
        ev[5].max() - ev[4].max(),        # barrier 2 release latency
        (ev[11] - ev[5]).max(),           # phase C1a: the dots' partials consumed (thread 0)
        (ev[8] - ev[11]).max(),           # phase C1b: y partials, v^T A22 v, two barriers
        (ev[9] - ev[8]).max(),            # phase C2: sum_t dots
        (ev[7] - ev[9]).max(),            # phase C: own rows' w
        (ev[6] - ev[7]).max(),            # phase C: row j+1 of w
        ev[6].max() - ev[0].min(),        # column total
    ])
r = np.array(rows) / 1e3
names = ["A", "A:work", "bar1", "symv", "dots", "bar2", "C1a", "C1b", "C2", "C:w", "C:wnext", "total"]
print(f"n={n} G={G}: panel k0={k0}, {len(rows)} columns; median / max us")
for k, nm in enumerate(names):
    print(f"  {nm:6s} {np.median(r[:, k]):8.2f} {r[:, k].max():8.2f}")
