"""GPU parity of Alg. 3 step 1 by "symmetric QR factorization in low
precision" (reading R12'; k_tridiag.cu: blocked binary32 Householder
tridiagonalisation, binary64 bisection + twisted-factorisation eigenvectors,
back-transformation) against the oracle's binary32 Householder + implicit
symmetric QR (oracle.low_evd_symqr).

The two compute the same object -- the eigenvectors of fl32(A) at binary32
accuracy -- by different algorithms and rounding orders, so Z is compared up
to column signs with the eigenvector perturbation bound: for eigenvalue gap
g_k, angle(z_k, z~_k) <= c n upsilon ||A|| / g_k (both are backward stable at
the binary32 level).  Eigenvalue estimates (Rayleigh quotients of the GPU's Z)
must match the oracle's to c n upsilon ||A||_2.  End to end, Alg. 3 with
either Z meets the north_star tolerances; the fp64 stage itself is compared
strictly from a shared Z (tests/test_gpu_scale.py)."""
import numpy as np
import pytest

import workloads as W
from conftest import OMEGA, UPSILON
from parity_rules import sweeps_match

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mpj():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2211_03339_b200 as m
    m.lib()
    return m


def dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).to("cuda", dtype).T


def host(t):
    return t.detach().cpu().numpy()


def gpu_z(mpj, A):
    r = mpj.eig(dev(A), mpj.default_config("eig", low_solver=mpj.LOW_SYMQR), Z_out=True)
    assert r.report.sweeps_low == 0
    return host(r.Z).astype(np.float64), r


@pytest.mark.parametrize("n,mode,kappa", [(3, 4, 1e3), (33, 4, 1e3), (64, 4, 1e3), (130, 5, 1e3),
                                          (200, 4, 1e3), (257, 3, 1e6), (400, 1, 1e3)])
def test_low_stage_vs_oracle(mpj, orc, n, mode, kappa):
    A, lam_true = W.example1(n, kappa, mode, W.seed_for(1, mode, kappa, 3))
    Zg, _ = gpu_z(mpj, A)
    Zo, lam_o, rep = orc.low_evd_symqr(A)
    Zo = Zo.astype(np.float64)
    lam_o = lam_o.astype(np.float64)
    nA2 = np.abs(lam_true).max()
    tol = 10 * n * UPSILON * nA2
    # binary32 backward-stable quality of the GPU's Z
    assert np.linalg.norm(Zg.T @ Zg - np.eye(n)) <= 10 * n * UPSILON
    rq = np.einsum("ij,ij->j", Zg, A @ Zg)
    assert np.all(np.diff(rq) <= tol)                                  # descending order
    assert np.max(np.abs(rq - lam_o)) <= tol                           # Rayleigh quotients vs the oracle's eigenvalues
    assert np.linalg.norm(A @ Zg - Zg * rq) / np.linalg.norm(A) <= 10 * n * UPSILON
    # columns against the oracle's, up to sign, where the eigenvalue is separated
    gaps = np.full(n, np.inf)
    if n > 1:
        dl = np.abs(np.diff(lam_true[::-1]))[::-1]
        gaps[:-1] = np.minimum(gaps[:-1], dl)
        gaps[1:] = np.minimum(gaps[1:], dl)
    for k in range(n):
        bound = 8 * n * UPSILON * nA2 / gaps[k]
        if bound < 0.1:
            c = abs(Zg[:, k] @ Zo[:, k])
            assert 1 - c <= bound ** 2 + 10 * n * UPSILON, (k, 1 - c, bound)


def test_low_stage_edge_cases(mpj, orc):
    # n = 1, 2
    for A in (np.array([[2.5]]), np.array([[1.0, 2.0], [2.0, -3.0]])):
        Zg, r = gpu_z(mpj, A)
        n = A.shape[0]
        assert np.linalg.norm(Zg.T @ Zg - np.eye(n)) <= 10 * UPSILON
        lam = host(r.lam)
        assert np.max(np.abs(lam - np.linalg.eigvalsh(A)[::-1])) <= 1e-14 * np.abs(A).max()
    # diagonal input with repeated entries: the tridiagonal splits everywhere,
    # every block is 1 x 1, Z is a permutation (duplicates kept distinct)
    d = np.array([3.0, -1.0, 7.5, 0.25, 2.0, 2.0, -9.0, 1e-3, 2.0])
    Zg, r = gpu_z(mpj, np.diag(d))
    assert np.array_equal(np.abs(Zg).sum(axis=0), np.ones(len(d)))
    assert np.array_equal(host(r.lam), np.sort(d)[::-1]) and r.sweeps == 0
    # block diagonal with identical blocks: repeated eigenvalues in different blocks
    B = np.array([[2.0, 1.0], [1.0, 2.0]])
    A = np.kron(np.eye(3), B)
    Zg, r = gpu_z(mpj, A)
    assert np.linalg.norm(Zg.T @ Zg - np.eye(6)) <= 60 * UPSILON
    assert np.max(np.abs(host(r.lam) - np.array([3, 3, 3, 1, 1, 1.0]))) <= 1e-14


@pytest.mark.parametrize("n,mode,kappa,gen", [(96, 4, 1e3, "ex1"), (256, 3, 1e6, "ex1"), (300, 5, 1e3, "ex1"),
                                              (512, 4, 1e3, "ex2"), (640, 3, 1e6, "ex1"), (1024, 4, 1e3, "ex1")])
def test_symqr_end_to_end(mpj, orc, n, mode, kappa, gen):
    """Alg. 3 with the symmetric-QR step 1 on both sides: north_star
    tolerances against the oracle, and a fp64 stage within the R20 sweep rule
    of the oracle's (their Z differ at the binary32 rounding level)."""
    g = W.example2 if gen == "ex2" else W.example1
    A, lam_true = g(n, kappa, mode, W.seed_for(1, mode, kappa, 9))
    res = mpj.eig(dev(A), mpj.default_config("eig", low_solver=mpj.LOW_SYMQR))
    ref = orc.mp_evd(A, orc.default_cfg("eig", b=res.report.block_b, low_solver=orc.LOW_SYMQR))
    lam, V = host(res.lam), host(res.V)
    nrm2 = np.abs(lam_true).max()
    assert np.max(np.abs(lam - ref.lam)) <= 1e-13 * nrm2
    assert np.max(np.abs(lam - lam_true)) <= 1e-13 * nrm2
    assert np.linalg.norm(V.T @ V - np.eye(n)) <= n * 1e-15
    assert np.linalg.norm(A @ V - V * lam) / np.linalg.norm(A) <= n * 1e-15
    # T0 quality of both step-1 implementations: the Figure 1 proxy,
    # off(Q^T A Q) <= 2 n ||A||_2 upsilon (the constant as in test_oracle_symqr)
    bd = 2 * n * nrm2 * UPSILON
    assert res.report.off0 <= bd and ref.report.off0 <= bd, (res.report.off0, ref.report.off0, bd)
    assert abs(res.sweeps - ref.report.sweeps) <= 1, (res.sweeps, ref.report.sweeps)


def test_symqr_is_the_default(mpj):
    n = 128
    A, _ = W.example1(n, 1e3, 4, 1)
    r0 = mpj.eig(dev(A))
    r2 = mpj.eig(dev(A), mpj.default_config("eig", low_solver=mpj.LOW_SYMQR))
    assert r0.report.sweeps_low == 0
    assert np.array_equal(host(r0.lam), host(r2.lam)) and np.array_equal(host(r0.V), host(r2.V))
