"""Alg. 3 (mixed precision) vs Alg. 2 (plain fp64 Jacobi, same kernels and
ordering) on the same matrix: seconds and fp64 sweeps.
usage: python tools/probe_plain.py [n] [mode] [kappa]   (defaults: 8192 3 1e6,
the bench workload)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2211_03339_b200 as mpj
import workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kappa = float(sys.argv[3]) if len(sys.argv) > 3 else 1e6
seed = 2211033390 + 4000 + 100 * mode + 10 * int(round(np.log10(kappa)))
A, lam_true = W.example1_torch(n, kappa, mode, seed, device="cuda")
Acm = A.T
for plain in (False, True):
    r = mpj.eig(Acm, plain=plain, allow_noconv=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = mpj.eig(Acm, plain=plain, allow_noconv=True)
    e1.record()
    torch.cuda.synchronize()
    dlam = float((r.lam - lam_true).abs().max() / lam_true.abs().max())
    print(f"n={n} mode={mode} kappa={kappa:g} {'plain (Alg. 2)' if plain else 'mixed (Alg. 3)'}: "
          f"{e0.elapsed_time(e1) / 1e3:.3f} s, fp64 sweeps {r.sweeps}, fp32 sweeps {r.report.sweeps_low}, "
          f"max|dlam|/|lam|max {dlam:.2e}", flush=True)
