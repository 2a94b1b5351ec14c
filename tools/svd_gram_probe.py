"""A/B probe for the fp64-stage SVD Gram policy (reading R21): sweeps and
accuracy of the GPU one-sided Jacobi with plain DMMA Gram blocks vs exact
(sliced) Gram blocks, against the oracle's sweep count (test infrastructure:
calls oracle/)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2211_03339_b200 as mpj  # noqa: E402
import workloads as W  # noqa: E402

cases = [(96, 48, 3), (200, 64, 4), (300, 130, 5), (512, 256, 3), (301, 100, 4), (1024, 512, 3)]
out = []
for m, n, mode in cases:
    A, sig_true = W.example3(m, n, 1e3, mode, W.seed_for(5, mode, 1e3))
    ref = oracle.mp_svd(A, oracle.default_cfg("svd", b=32))
    row = {"m": m, "n": n, "mode": mode, "oracle_sweeps": ref.report.sweeps}
    for g in ("dmma", "exact", "default"):
        os.environ["MPJ_SVD_GRAM"] = "" if g == "default" else g
        res = mpj.svd(torch.from_numpy(A).cuda())
        sig = res.sigma.cpu().numpy()
        U, V = res.U.cpu().numpy(), res.V.cpu().numpy()
        row[g] = {"sweeps": res.sweeps, "sweeps_low": res.report.sweeps_low, "rot_low": res.report.rotations_low, "rot": res.report.rotations,
                  "dsig_ref": float(np.max(np.abs(sig - ref.sigma)) / ref.sigma[0]),
                  "resid": float(np.linalg.norm(A @ V - U * sig) / np.linalg.norm(A)),
                  "orth_u": float(np.linalg.norm(U.T @ U - np.eye(n)))}
    row["oracle_rot"] = ref.report.rotations
    row["oracle_sweeps_low"] = ref.report.sweeps_low
    row["oracle_rot_low"] = ref.report.rotations_low
    print(json.dumps(row), flush=True)
    out.append(row)
