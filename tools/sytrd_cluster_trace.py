#!/usr/bin/env python
"""Phase timing of the one-cluster tridiagonalisation (k_sytrd_cluster,
k_tridiag.cu) from a diagnostics build (MPJ_NVCC_EXTRA=-DMPJ_SYTRD_TRACE):
thread 0 of every CTA stamps %globaltimer at the phase boundaries of 64
consecutive columns from k0; prints the median / max over those columns of
each phase (the slowest CTA) in microseconds."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2211_03339_b200 as mpj  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
k0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
mpj.lib().mpjacobi_debug_sytrd_trace_panel(k0)
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(n, n, device="cuda", generator=g)
A = (A + A.T) / 2
for _ in range(2):
    mpj.sytrd(A)
buf = np.zeros(64 * 12 * 320, dtype=np.uint64)
mpj.lib().mpjacobi_debug_sytrd_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)))
t = buf.reshape(64, 12, 320)[:, :, :16].astype(np.float64)
names = ["cluster #1", "beta, v", "A22 v", "push y", "cluster #2", "p, cluster #3", "p^T v, w", "rank-2", "push x"]
rows = []
for kk in range(64):
    ev = t[kk]
    if not ev[0].any() or not ev[9].any():
        continue
    rows.append([ev[e + 1].max() - ev[e].max() for e in range(9)] + [ev[9].max() - ev[0].min()])
r = np.array(rows) / 1e3
print(f"n={n}: columns {k0}..{k0 + len(rows) - 1}; median / max us (slowest CTA per phase)")
for k, nm in enumerate(names + ["total"]):
    print(f"  {nm:12s} {np.median(r[:, k]):8.2f} {r[:, k].max():8.2f}")
