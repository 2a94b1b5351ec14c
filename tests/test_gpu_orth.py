"""Alg. 3 step 2 by the two GPU orthogonalisers against the oracle's
literal MGS: blocked CGS + CholeskyQR2 (default) and blocked Householder QR
(the paper's GPU choice).  Both compute the unique
QR factor with a positive diagonal of R, so Q matches MGS's to O(n omega)
when kappa(Z) = 1 + O(upsilon) (reading R10)."""
import numpy as np
import pytest

import workloads as W
from conftest import OMEGA

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mpj():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2211_03339_b200 as m
    m.lib()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).T)).cuda().T


@pytest.mark.parametrize("method", ["cgs", "householder", "series"])
@pytest.mark.parametrize("n", [1, 16, 65, 100, 300, 1000])
def test_orth_matches_mgs(mpj, orc, method, n):
    Z = W.rounded_haar(n, 4000 + n)
    Qo, _, st = orc.mgs(Z)
    assert st == 0
    Qg = mpj.orth(dev(Z), method=method).cpu().numpy()
    assert np.linalg.norm(Qg.T @ Qg - np.eye(n)) <= 10 * n * OMEGA
    assert np.linalg.norm(Qg - Qo) <= 10 * n * OMEGA


def test_orth_householder_n2048(mpj, orc):
    n = 2048
    Z = W.rounded_haar(n, 2049)
    Qo, _, _ = orc.mgs(Z)
    Qg = mpj.orth(dev(Z), method="householder").cpu().numpy()
    assert np.linalg.norm(Qg - Qo) <= 10 * n * OMEGA


def test_orth_householder_rank_deficient(mpj):
    Z = np.eye(8)
    Z[:, 5] = 0.0
    with pytest.raises(mpj.MpjError) as e:
        mpj.orth(dev(Z), method="householder")
    assert e.value.status == mpj.MPJ_ERR_RANKDEF


@pytest.mark.parametrize("n", [256, 700])
def test_eig_with_householder_orth(mpj, orc, n):
    """Alg. 3 with the Householder orthogonaliser: the same T0 as with CGS to
    rounding, hence the same fp64 sweeps, and the north_star tolerances."""
    A, lam = W.example1(n, 1e6, 3, W.seed_for(1, 3, 1e6, 8))
    rh = mpj.eig(dev(A), mpj.default_config("eig", orth=mpj.ORTH_HOUSEHOLDER))
    rc = mpj.eig(dev(A))
    assert rh.sweeps == rc.sweeps
    assert abs(rh.report.off0 - rc.report.off0) <= 1e-6 * rc.report.off0 + 100 * n * OMEGA * rc.report.norm_a
    l = rh.lam.cpu().numpy()
    V = rh.V.cpu().numpy()
    assert np.max(np.abs(l - lam)) <= 1e-13 * np.abs(lam).max()
    assert np.linalg.norm(V.T @ V - np.eye(n)) <= n * 1e-15
    assert np.linalg.norm(A @ V - V * l) / np.linalg.norm(A) <= n * 1e-15
