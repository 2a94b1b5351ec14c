"""Pins for the oracle's MGS (Alg. 3 step 2; Lemma 2.1), the
preconditioning product Q^T A Q (step 3) and the Figure 1 bound
off(Q^T A Q) <= bd = n ||A||_2 upsilon."""
import numpy as np
import pytest
import scipy.linalg

import workloads as W
from conftest import OMEGA, UPSILON, rand_sym


def test_identity_and_scaling(orc):
    n = 12
    Q, R, st = orc.mgs(np.eye(n))
    assert st == 0 and np.array_equal(Q, np.eye(n)) and np.array_equal(R, np.eye(n))
    # orthogonal up to column scaling by 2 -> Q = Z/2, R = 2I
    H = W.haar(n, np.random.default_rng(3))
    Q, R, st = orc.mgs(2.0 * H)
    assert np.max(np.abs(Q - H)) <= 8 * n * OMEGA
    assert np.max(np.abs(R - 2 * np.eye(n))) <= 16 * n * OMEGA


def test_rounded_haar_contract(orc):
    """SPEC acceptance 6 / Lemma 2.1 with kappa(Z) ~ 1: a binary32-rounded Haar
    256 x 256 re-orthogonalised in binary64 has ||Q^T Q - I||_F <= 10 n omega;
    Z = QR to 10 n omega ||Z||; diag(R) = 1 + O(upsilon), off-diag R = O(upsilon)
    (P:289-290)."""
    n = 256
    Z = W.rounded_haar(n, 11)
    Q, R, st = orc.mgs(Z)
    assert st == 0
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 10 * n * OMEGA
    assert np.linalg.norm(Z - Q @ R) <= 10 * n * OMEGA * np.linalg.norm(Z)
    assert np.all(np.abs(np.diag(R) - 1) <= 4 * np.sqrt(n) * UPSILON)
    assert np.max(np.abs(np.triu(R, 1))) <= 4 * np.sqrt(n) * UPSILON
    assert np.allclose(np.tril(R, -1), 0)


def test_rank_deficient(orc):
    Z = np.eye(4)
    Z[:, 3] = Z[:, 1]
    _, _, st = orc.mgs(Z)
    assert st == 3


def test_gemm_against_numpy(orc):
    rng = np.random.default_rng(4)
    A, B = rng.standard_normal((37, 21)), rng.standard_normal((21, 13))
    assert np.allclose(orc.gemm(A, B), A @ B, rtol=0, atol=32 * OMEGA * 21)
    assert np.allclose(orc.gemm(A.T.copy(), B, transA=True), A @ B, rtol=0, atol=32 * OMEGA * 21)


def test_qtaq_special_cases(orc):
    A = rand_sym(20, 9)
    T = orc.qtaq(A, np.eye(20))
    assert np.array_equal(T, A)
    perm = np.random.default_rng(1).permutation(20)
    P = np.eye(20)[:, perm]
    assert np.array_equal(orc.qtaq(A, P), A[perm][:, perm])
    H = W.haar(20, np.random.default_rng(2))
    T = orc.qtaq(A, H)
    assert np.array_equal(T, T.T)
    assert np.max(np.abs(T - H.T @ A @ H)) <= 64 * 20 * OMEGA * np.linalg.norm(A)


@pytest.mark.parametrize("mode", [1, 2, 3, 4, 5])
def test_figure1_bound_with_lapack_low_stage(orc, mode):
    """Figure 1: with the paper's low-precision solver
    (LAPACK SSYEV-class, here scipy's ssyevd on fl32(A)), ||off(Q^T A Q)||_F
    <= bd = n ||A||_2 upsilon for kappa = 1e8 (SPEC acceptance 4)."""
    for n in (64, 128):
        A, lam = W.example1(n, 1e8, mode, W.seed_for(4, mode, 1e8))
        _, Z = scipy.linalg.eigh(A.astype(np.float32), driver="evd")
        res = orc.mp_evd(A, Z=np.asfortranarray(Z.astype(np.float32)))
        bd = n * lam[0] * UPSILON
        assert res.report.off0 <= bd, (n, res.report.off0, bd)
        assert res.status == 0
