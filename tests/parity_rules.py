"""Sweep-count parity rules (readings R20 / R23), shared by the GPU
parity tests.  Identical counts are the rule; the allowances below cover only
stop decisions taken at the rounding-noise level, where any two valid
evaluation orders of the same rotations may decide differently."""
import numpy as np

OMEGA = 2.0 ** -53


def sweeps_match(sw_a, hist_a, sw_b, hist_b, tol):
    """R20 (EVD): counts may differ by one when, at the sweep where the runs
    part, both off-norms ||off(T)||_F lie within 10x of tol = eps ||A||_F."""
    if sw_a == sw_b:
        return True
    if abs(sw_a - sw_b) != 1:
        return False
    k = min(sw_a, sw_b)
    return hist_a[k] <= 10 * tol and hist_b[k] <= 10 * tol


def svd_sweeps_match(res, ref, A, early=2e-4):
    """R23 (SVD, Alg. 5): identical fp64 sweep counts, except that they may
    differ by one when the decision after the sweep where the runs part was
    taken at a threshold in BOTH runs:
      * both relative off-norms ||off(C^T C)||_F / ||C^T C||_F at the rounding
        floor of the Gram matrix (<= 100 eps = 10 omega; the paper's eps =
        0.1 omega lies below that floor, which is why P:678 adds the early
        stop), where the rotate test |gamma| > omega sqrt(alpha beta)
        decides on rounding noise in the columns' last bits; or
      * both sweeps' rotations / N within a factor 2 of the early-stop ratio
        (P:678).
    res: the GPU result (report.off_hist absolute, report.rot_hist ints);
    ref: the oracle's (report.off_hist relative, report.rot_hist)."""
    a, b = res.sweeps, ref.report.sweeps
    if a == b:
        return True
    if abs(a - b) != 1:
        return False
    k = min(a, b)
    n = A.shape[1]
    N = n * (n - 1) / 2
    tot = np.linalg.norm(A.T @ A)                  # ||C^T C||_F = ||A^T A||_F (C = A Q, Q orthogonal)
    eps = 0.1 * OMEGA
    off_g = res.report.off_hist[k] / tot
    off_o = ref.report.off_hist[k]
    if off_g <= 100 * eps and off_o <= 100 * eps:
        return True
    rg = res.report.rot_hist[k - 1] / N
    ro = ref.report.rot_hist[k - 1] / N
    return early / 2 <= rg <= 2 * early and early / 2 <= ro <= 2 * early
