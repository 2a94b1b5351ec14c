#!/usr/bin/env python
"""One mixed-precision SVD of a seeded m x n matrix through the binding (for
ncu captures of the SVD kernels).  Usage: probe_svd.py m n"""
import sys

import torch

import paper_2211_03339_b200 as mpj

m, n = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator().manual_seed(7)
A = torch.randn(m, n, generator=g, dtype=torch.float64).cuda()
res = mpj.mpjacobi_svd(mpj.colmajor(A))
torch.cuda.synchronize()
print("done")
