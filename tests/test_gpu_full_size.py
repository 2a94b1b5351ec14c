"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times: the oracle cannot run these sizes end to end, so the
checks are (1) properties that hold at any size -- residual, orthogonality,
eigen/singular values against the generator's exact spectrum (the north_star
tolerances) -- and (2) sampled outputs recomputed one by one on the host in
numpy fp64 (independent of the GPU) or, for the batched path, a sample of the
batch run through the oracle itself."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mpj():
    import paper_2211_03339_b200 as m
    return m


def test_full_size_evd_n8192(mpj):
    """BASELINE config 4 at one GPU: Example 1 mode 3, kappa = 1e6, n = 8192
    (the bench workload, the bench's seed and workspace path)."""
    n, mode, kappa = 8192, 3, 1e6
    seed = 2211033390 + 4000 + 100 * mode + 10 * int(round(np.log10(kappa)))
    A, lam_true = W.example1_torch(n, kappa, mode, seed, device="cuda")
    Acm = A.T
    cfg = mpj.default_config("eig")
    ws = mpj.eig_workspace(n, cfg, device=A.device)
    res = mpj.eig(Acm, cfg, workspace=ws)
    lam, V = res.lam, res.V
    nA = torch.linalg.norm(A)
    assert float(torch.linalg.norm(A @ V - V * lam) / nA) <= n * 1e-15
    assert float(torch.linalg.norm(V.T @ V - torch.eye(n, device=A.device, dtype=A.dtype))) <= n * 1e-15
    assert float((lam - lam_true).abs().max() / lam_true.abs().max()) <= 1e-13
    assert res.report.variant == mpj.VARIANT_BLOCK and res.sweeps <= 60
    # sampled eigenpairs, recomputed on the host in numpy fp64
    Ah = A.cpu().numpy()
    rng = np.random.default_rng(8192)
    for i in sorted(rng.choice(n, 4, replace=False)):
        v = V[:, i].cpu().numpy()
        li = float(lam[i])
        r = Ah @ v - li * v
        assert np.linalg.norm(r) <= n * 1e-15 * np.linalg.norm(Ah)
        assert abs(np.dot(v, v) - 1.0) <= 1e-13


@pytest.mark.parametrize("low", ["symqr", "jacobi"])
def test_full_size_batched_4096x64(mpj, low):
    """BASELINE config 3: 4096 x n = 64 (bench workload), step 1 by symmetric
    QR (the default, reading R12') or the fp32 Jacobi (R12).  All matrices:
    residual / orthogonality; 16 sampled matrices against the oracle with the
    same step 1 (eigenvalues; fp64 sweeps identical for the Jacobi step 1,
    within one for symmetric QR; fp32 sweeps identical)."""
    import oracle as orc
    n, batch = 64, 4096
    As = np.stack([W.example1(n, 1e3, 3 + k % 3, W.seed_for(3, 3 + k % 3, 1e3, k))[0] for k in range(batch)])
    A = torch.from_numpy(As).cuda()
    jac = low == "jacobi"
    res = mpj.eig_batched(A, mpj.default_config("eig", low_solver=mpj.LOW_JACOBI if jac else mpj.LOW_SYMQR))
    lam, V = res.lam, res.V
    R = torch.linalg.norm(A @ V - V * lam[:, None, :], dim=(1, 2)) / torch.linalg.norm(A, dim=(1, 2))
    O = torch.linalg.norm(V.transpose(1, 2) @ V - torch.eye(n, device=A.device, dtype=A.dtype), dim=(1, 2))
    assert float(R.max()) <= n * 1e-15 and float(O.max()) <= n * 1e-15
    lam_h, sw, swl = lam.cpu().numpy(), res.sweeps.cpu().numpy(), res.sweeps_low.cpu().numpy()
    rng = np.random.default_rng(4096)
    for k in sorted(rng.choice(batch, 16, replace=False)):
        ref = orc.mp_evd(As[k], orc.default_cfg("eig", b=32, low_solver=orc.LOW_JACOBI if jac else orc.LOW_SYMQR))
        assert np.max(np.abs(lam_h[k] - ref.lam)) <= 1e-13 * np.max(np.abs(ref.lam))
        if jac:
            assert int(sw[k]) == ref.report.sweeps
        else:
            assert abs(int(sw[k]) - ref.report.sweeps) <= 1
        assert int(swl[k]) == ref.report.sweeps_low


def test_full_size_svd_16384x4096(mpj):
    """BASELINE config 5a: Example 3 mode 3, kappa = 1e3, 16384 x 4096 (the
    bench workload): residual, orthogonality of U and V, singular values
    against the generator's, sampled singular triplets on the host."""
    m, n = 16384, 4096
    At, sig_true = W.example3_torch(m, n, 1e3, 3, 2211033390 + 5000 + 300 + 30, device="cuda")
    A = At.T
    cfg = mpj.default_config("svd")
    res = mpj.svd(A, cfg)
    sig, U, V = res.sigma, res.U, res.V
    nA = torch.linalg.norm(A)
    assert float(torch.linalg.norm(A @ V - U * sig) / nA) <= n * 1e-15
    I = torch.eye(n, device=A.device, dtype=A.dtype)
    assert float(torch.linalg.norm(U.T @ U - I)) <= n * 1e-15
    assert float(torch.linalg.norm(V.T @ V - I)) <= n * 1e-15
    assert float((sig - sig_true).abs().max() / sig_true.abs().max()) <= 1e-13
    Ah = A.cpu().numpy()
    rng = np.random.default_rng(16384)
    for i in sorted(rng.choice(n, 4, replace=False)):
        u, v, s = U[:, i].cpu().numpy(), V[:, i].cpu().numpy(), float(sig[i])
        assert np.linalg.norm(Ah @ v - s * u) <= n * 1e-15 * np.linalg.norm(Ah)
