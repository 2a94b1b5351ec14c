"""Pins for the oracle's Lemma 3.1 rotation and the per-round form
of Eq. (3.2).  None of these retypes the oracle's formula: they
check closed forms, the annihilation property, and high-precision references."""
from decimal import Decimal, getcontext

import numpy as np
import pytest

from conftest import OMEGA, UPSILON, rand_sym


def _J2(s, t):
    """2x2 rotation block [[c, s], [-s, c]] of Eq. (3.1)."""
    c = 1.0 / np.sqrt(1.0 + t * t)
    return np.array([[c, s], [-s, c]])


def test_mu_zero_gives_quarter_turn(orc):
    # (a_ii, a_jj, a_ij) = (0, 0, 1): mu = 0 -> t = 1, c = s = 1/sqrt(2)
    rot, t, s, tau = orc.rotation(0.0, 0.0, 1.0)
    assert rot and t == 1.0
    assert abs(s - 2 ** -0.5) <= OMEGA
    assert abs(tau - (np.sqrt(2) - 1)) <= 2 * OMEGA  # tau = s/(1+c)


def test_two_by_two_closed_form(orc):
    # [[2,1],[1,3]] -> diag((5-sqrt5)/2, (5+sqrt5)/2) after one rotation
    r = orc.jacobi_evd(np.array([[2.0, 1.0], [1.0, 3.0]]), b=1, tol=0.0, max_sweeps=1)
    lo, hi = (5 - np.sqrt(5)) / 2, (5 + np.sqrt(5)) / 2
    assert r.T[0, 1] == 0.0 and r.T[1, 0] == 0.0  # exact zero pivot
    assert abs(r.T[0, 0] - lo) <= 4 * OMEGA * hi and abs(r.T[1, 1] - hi) <= 4 * OMEGA * hi
    # V holds the eigenvectors
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    assert np.linalg.norm(A @ r.V - r.V @ np.diag(np.diag(r.T))) <= 8 * OMEGA * hi


def test_zero_pivot_is_identity(orc):
    # a_ij = 0 -> (c, s) = (1, 0): the threshold test catches it (skip)
    for x in (1.0, -3.5, 0.0):
        rot, t, s, tau = orc.rotation(x, x, 0.0, nu=20 * OMEGA)
        assert not rot and s == 0.0 and tau == 0.0


def test_threshold_rule(orc):
    nu = 20 * OMEGA
    # |a_pq| <= nu min(|a_pp|,|a_qq|) -> skip
    assert not orc.rotation(1.0, 2.0, nu * 1.0, nu=nu)[0]
    assert orc.rotation(1.0, 2.0, nu * 1.0 * (1 + 4 * OMEGA), nu=nu)[0]
    # sqrt rule of Remark 3.1: |a_pq| <= nu sqrt(a_pp a_qq)
    assert not orc.rotation(1.0, 4.0, nu * 2.0, nu=nu, rule=1)[0]
    assert orc.rotation(1.0, 4.0, nu * 2.1, nu=nu, rule=1)[0]


@pytest.mark.parametrize("precision,u", [("f64", OMEGA), ("f32", UPSILON)])
def test_random_pivots_annihilate(orc, precision, u):
    """1000 random pivots (SPEC acceptance 1): c^2+s^2 = 1 within 4u,
    |theta| <= pi/4 (c >= 1/sqrt2 - 4u), and J^T A J has a zero (p,q) entry
    to within 8u (|a_pp|+|a_qq|+|a_pq|) -- computed independently in numpy."""
    rng = np.random.default_rng(7)
    for _ in range(1000):
        app, aqq = rng.standard_normal(2) * 10 ** rng.uniform(-3, 3, 2)
        apq = rng.standard_normal() * 10 ** rng.uniform(-6, 2)
        if precision == "f32":
            app, aqq, apq = (float(np.float32(v)) for v in (app, aqq, apq))
        rot, t, s, tau = orc.rotation(app, aqq, apq, precision=precision)
        assert rot
        c = 1.0 / np.sqrt(1.0 + t * t)      # independent of the oracle's c
        assert abs(s - t * c) <= 4 * u * abs(s)
        assert abs(c * c + s * s - 1) <= 6 * u
        assert abs(tau - s / (1 + c)) <= 6 * u * abs(tau)
        assert c >= 2 ** -0.5 - 4 * u
        A = np.array([[app, apq], [apq, aqq]])
        J = np.array([[c, s], [-s, c]])
        B = J.T @ A @ J
        assert abs(B[0, 1]) <= 8 * u * (abs(app) + abs(aqq) + abs(apq)) * 4


def test_large_mu_branch_matches_exact_t(orc):
    """Reading R4: for |mu| >= 2^26 the oracle uses t = 1/(2 mu).  Compare with
    t = 1/(mu + sqrt(1+mu^2)) evaluated in 60-digit decimal arithmetic."""
    getcontext().prec = 60
    for mu in (2.0 ** 26, 2.0 ** 26 + 1, 3.1e9, -7.7e12, 1e160, -1e200):
        app, apq = 0.0, 1.0
        aqq = 2.0 * mu  # mu = (aqq - app)/(2 apq)
        rot, t, s, tau = orc.rotation(app, aqq, apq)
        m = Decimal(mu)
        r = (1 + m * m).sqrt()
        t_ex = 1 / (m + r) if m >= 0 else 1 / (m - r)
        assert rot
        assert abs(Decimal(t) - t_ex) <= Decimal(2 * OMEGA) * abs(t_ex)


def test_round_equals_dense_product(orc):
    """One round of n/2 disjoint rotations == J^T T J with J the dense product
    of the round's rotations (built in numpy from the schedule), and V == J.
    This pins rows/columns, signs and the mirror of the tile update."""
    for n, b in ((8, 1), (12, 2), (16, 4)):
        T0 = rand_sym(n, 100 + n)
        P, Q = orc.schedule(n, b)
        J = np.eye(n)
        for p, q in zip(P[0], Q[0]):
            rot, t, s, tau = orc.rotation(T0[p, p], T0[q, q], T0[p, q], nu=20 * OMEGA)
            c = 1.0 / np.sqrt(1.0 + t * t) if rot else 1.0
            J[p, p] = c; J[q, q] = c; J[p, q] = s; J[q, p] = -s
        ref = J.T @ T0 @ J
        for p, q in zip(P[0], Q[0]):
            ref[p, q] = ref[q, p] = 0.0
        r = orc.jacobi_evd(T0, b=b, tol=0.0, max_sweeps=1, max_rounds=1)
        assert np.max(np.abs(r.T - ref)) <= 16 * OMEGA * np.linalg.norm(T0)
        assert np.max(np.abs(r.V - J)) <= 8 * OMEGA
        assert np.array_equal(r.T, r.T.T)  # exact symmetry (reading R7)


def test_round_offnorm_decrement(orc):
    """Eq. (3.2) per rotation, summed over a round of disjoint rotations:
    ||off(B)||^2 = ||off(A)||^2 - 2 sum a_pq^2, within 32 n omega ||A||_F^2."""
    for n, b in ((16, 1), (32, 4), (64, 8)):
        T0 = rand_sym(n, 5 + n)
        P, Q = orc.schedule(n, b)
        for r_idx in (0, 1, 2):
            T = T0.copy()
            if r_idx:
                T = orc.jacobi_evd(T0, b=b, tol=0.0, max_sweeps=1, max_rounds=r_idx).T
            before = orc.off(T) ** 2
            dec = 2 * sum(T[p, q] ** 2 for p, q in zip(P[r_idx], Q[r_idx]))
            after_T = orc.jacobi_evd(T0, b=b, tol=0.0, max_sweeps=1, max_rounds=r_idx + 1).T
            after = orc.off(after_T) ** 2
            assert abs(after - (before - dec)) <= 32 * n * OMEGA * np.linalg.norm(T0) ** 2
