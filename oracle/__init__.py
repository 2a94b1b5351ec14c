"""ctypes wrapper around oracle/mpj_oracle.c.

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs are the only allowed callers.  The product
package paper_2211_03339_b200 never imports this module, and this module never
imports the product package.

Every array is float64 (or float32 for the low-precision stage) in column-major
(Fortran) order, matching the C code.  See mpj_oracle.c for the citation of
each function to /root/reference/PAPER.md.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

# libgomp reads these once, at load: passive waiting avoids a collapse when the
# host is oversubscribed (measured 18 s vs 0.3 s on an 8-core box).
os.environ.setdefault("OMP_WAIT_POLICY", "passive")
os.environ.setdefault("OMP_NUM_THREADS", str(max(1, len(os.sched_getaffinity(0)))))

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mpj_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OMEGA = 2.0 ** -53
UPSILON = 2.0 ** -24

GCC_FLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", "-std=gnu11"]


def threads() -> int:
    """OpenMP threads the oracle uses (reported as cpu_baseline.cores)."""
    return int(os.environ["OMP_NUM_THREADS"])


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no contraction: -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *GCC_FLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int)
_llp = C.POINTER(C.c_longlong)


class Cfg(C.Structure):
    _fields_ = [
        ("eps_factor", C.c_double), ("nu_factor", C.c_double),
        ("eps_low_factor", C.c_double), ("nu_low_factor", C.c_double),
        ("early_stop", C.c_double), ("max_sweeps", C.c_int), ("max_sweeps_low", C.c_int),
        ("rule", C.c_int), ("b", C.c_int), ("low_solver", C.c_int),
    ]


class Report(C.Structure):
    _fields_ = [
        ("sweeps", C.c_int), ("sweeps_low", C.c_int), ("status", C.c_int), ("status_low", C.c_int),
        ("rotations", C.c_longlong), ("rotations_low", C.c_longlong),
        ("normA", C.c_double), ("off0", C.c_double), ("off_hist", C.c_double * 64),
        ("rot_hist", C.c_double * 64),
    ]


def _declare(L):
    L.orc_padded_n.restype = C.c_int
    L.orc_padded_n.argtypes = [C.c_int, C.c_int]
    L.orc_schedule.restype = C.c_int
    L.orc_schedule.argtypes = [C.c_int, C.c_int, _ip, _ip]
    for nm, tp in (("orc_fro_f64", _dp), ("orc_fro_f32", _fp)):
        getattr(L, nm).restype = C.c_double
        getattr(L, nm).argtypes = [tp, C.c_int, C.c_int, C.c_int]
    for nm, tp in (("orc_off_f64", _dp), ("orc_off_f32", _fp)):
        getattr(L, nm).restype = C.c_double
        getattr(L, nm).argtypes = [tp, C.c_int, C.c_int]
    L.orc_rotation_f64.restype = C.c_int
    L.orc_rotation_f64.argtypes = [C.c_double] * 4 + [C.c_int, _dp, _dp, _dp]
    L.orc_rotation_f32.restype = C.c_int
    L.orc_rotation_f32.argtypes = [C.c_float] * 4 + [C.c_int, _fp, _fp, _fp]
    for nm, tp in (("orc_jacobi_evd_f64", _dp), ("orc_jacobi_evd_f32", _fp)):
        f = getattr(L, nm)
        f.restype = C.c_int
        f.argtypes = [tp, tp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                      C.c_longlong, _ip, _llp, _dp]
    L.orc_jacobi_rowcyclic_f64.restype = C.c_int
    L.orc_jacobi_rowcyclic_f64.argtypes = [_dp, _dp, C.c_int, C.c_double, C.c_double, C.c_int,
                                           C.c_int, _ip, _llp, _dp]
    L.orc_mgs_f64.restype = C.c_int
    L.orc_mgs_f64.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp]
    L.orc_gemm_f64.restype = None
    L.orc_gemm_f64.argtypes = [C.c_int, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int]
    L.orc_qtaq_f64.restype = None
    L.orc_qtaq_f64.argtypes = [_dp, _dp, C.c_int, _dp]
    L.orc_sort_desc.restype = None
    L.orc_sort_desc.argtypes = [_dp, C.c_int, _ip]
    L.orc_low_evd.restype = C.c_int
    L.orc_low_evd.argtypes = [_dp, C.c_int, C.POINTER(Cfg), _fp, C.POINTER(Report)]
    L.orc_mp_evd.restype = C.c_int
    L.orc_mp_evd.argtypes = [_dp, C.c_int, C.POINTER(Cfg), _fp, _dp, _dp, C.POINTER(Report)]
    L.orc_plain_evd.restype = C.c_int
    L.orc_plain_evd.argtypes = [_dp, C.c_int, C.POINTER(Cfg), _dp, _dp, C.POINTER(Report)]
    for nm, tp in (("orc_jacobi_svd_f64", _dp), ("orc_jacobi_svd_f32", _fp)):
        f = getattr(L, nm)
        f.restype = C.c_int
        f.argtypes = [tp, tp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                      C.c_int, _ip, _llp, _dp, _dp]
    L.orc_gram_offnorm.restype = None
    L.orc_gram_offnorm.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp]
    L.orc_mp_svd.restype = C.c_int
    L.orc_mp_svd.argtypes = [_dp, C.c_int, C.c_int, C.POINTER(Cfg), _fp, _dp, _dp, _dp,
                             C.POINTER(Report)]
    L.orc_plain_svd.restype = C.c_int
    L.orc_plain_svd.argtypes = [_dp, C.c_int, C.c_int, C.POINTER(Cfg), _dp, _dp, _dp,
                                C.POINTER(Report)]
    L.orc_mp_evd_batched.restype = C.c_int
    L.orc_mp_evd_batched.argtypes = [_dp, C.c_int, C.c_int, C.POINTER(Cfg), _dp, _dp, _ip, _ip]
    L.orc_sytrd_f32.restype = C.c_int
    L.orc_sytrd_f32.argtypes = [_fp, C.c_int, _fp, _fp, _fp]
    L.orc_orgtr_f32.restype = None
    L.orc_orgtr_f32.argtypes = [_fp, C.c_int, _fp, _fp]
    L.orc_tridiag_qr_f32.restype = C.c_int
    L.orc_tridiag_qr_f32.argtypes = [_fp, _fp, C.c_int, _fp]
    L.orc_low_evd_symqr.restype = C.c_int
    L.orc_low_evd_symqr.argtypes = [_dp, C.c_int, _fp, _fp, C.POINTER(Report)]
    L.orc_block_jacobi_evd_f64.restype = C.c_int
    L.orc_block_jacobi_evd_f64.argtypes = [_dp, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                           C.c_int, _ip, _llp, _dp]
    L.orc_report_size.restype = C.c_size_t
    L.orc_cfg_size.restype = C.c_size_t
    assert L.orc_report_size() == C.sizeof(Report)
    assert L.orc_cfg_size() == C.sizeof(Cfg)


def _f64(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _f32(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float32))


def _p(a):
    if a is None:
        return None
    if a.dtype == np.float64:
        return a.ctypes.data_as(_dp)
    if a.dtype == np.float32:
        return a.ctypes.data_as(_fp)
    if a.dtype == np.int32:
        return a.ctypes.data_as(_ip)
    raise TypeError(a.dtype)


LOW_SYMQR, LOW_JACOBI = 2, 1


def default_cfg(kind: str = "eig", b: int = 32, **kw) -> Cfg:
    """The paper's settings: eps = 0.1 omega; nu = 20 omega (EVD) or
    omega (SVD, with the 2e-4 early stop).  EVD step 1 (reading R12'):
    low_solver 0 / LOW_SYMQR = symmetric QR in binary32, LOW_JACOBI =
    the fp32 parallel Jacobi, whose stop rule is eps_low = max(10, 1.25
    sqrt(n)) upsilon (eps_low_factor = 0 selects the rule), nu_low = 20
    upsilon (EVD) / upsilon (SVD, whose low stage is always one-sided Jacobi;
    its eps_low is SPEC's 10 upsilon, S:281 -- DESIGN R12, measured best for
    Alg. 5)."""
    c = Cfg()
    c.eps_factor = 0.1
    c.nu_factor = 20.0 if kind == "eig" else 1.0
    c.eps_low_factor = 0.0 if kind == "eig" else 10.0
    c.nu_low_factor = 20.0 if kind == "eig" else 1.0
    c.early_stop = 0.0 if kind == "eig" else 2e-4
    c.max_sweeps = 60
    c.max_sweeps_low = 60
    c.rule = 0
    c.b = b
    c.low_solver = 0
    for k, v in kw.items():
        setattr(c, k, v)
    return c


# ------------------------------------------------------------------ ordering
def padded_n(n: int, b: int) -> int:
    return lib().orc_padded_n(n, b)


def schedule(n: int, b: int):
    """(P, Q) int arrays of shape (n_p - 1, n_p / 2): pair (P[r,k], Q[r,k]) of
    round r over the padded index range."""
    np_ = padded_n(n, b)
    h = np_ // 2
    P = np.zeros((max(np_ - 1, 0), h), dtype=np.int32)
    Q = np.zeros_like(P)
    r = lib().orc_schedule(n, b, _p(P), _p(Q))
    if r != np_ - 1:
        raise ValueError(f"bad ordering block size b={b}")
    return P, Q


# ------------------------------------------------------------------ norms
def off(T) -> float:
    T = np.asfortranarray(T)
    if T.dtype == np.float32:
        return lib().orc_off_f32(_p(T), T.shape[0], T.shape[0])
    T = _f64(T)
    return lib().orc_off_f64(_p(T), T.shape[0], T.shape[0])


def fro(A) -> float:
    A = np.asfortranarray(A)
    if A.dtype == np.float32:
        return lib().orc_fro_f32(_p(A), A.shape[0], A.shape[1], A.shape[0])
    A = _f64(A)
    return lib().orc_fro_f64(_p(A), A.shape[0], A.shape[1], A.shape[0])


def rotation(app, aqq, apq, nu=0.0, rule=0, precision="f64"):
    """Lemma 3.1 parameters: (rotate?, t, s, tau)."""
    if precision == "f64":
        t, s, u = C.c_double(), C.c_double(), C.c_double()
        r = lib().orc_rotation_f64(app, aqq, apq, nu, rule, C.byref(t), C.byref(s), C.byref(u))
    else:
        t, s, u = C.c_float(), C.c_float(), C.c_float()
        r = lib().orc_rotation_f32(app, aqq, apq, nu, rule, C.byref(t), C.byref(s), C.byref(u))
    return bool(r), t.value, s.value, u.value


# ------------------------------------------------------------------ Jacobi
@dataclass
class JacobiResult:
    T: np.ndarray
    V: np.ndarray
    sweeps: int
    rotations: int
    status: int
    off_hist: np.ndarray = field(default_factory=lambda: np.zeros(0))


def jacobi_evd(T, V=None, *, b=32, tol=0.0, nu=20 * OMEGA, rule=0, max_sweeps=60,
               max_rounds=-1, precision="f64") -> JacobiResult:
    """Alg. 2 / Alg. 3 steps 4-11 with the block merry-go-round ordering.
    ``tol`` is the absolute threshold eps*||A||_F of the while test."""
    if precision == "f64":
        T = _f64(T).copy(order="F")
        V = np.eye(T.shape[0]) if V is None else V
        V = _f64(V).copy(order="F")
        fn = lib().orc_jacobi_evd_f64
    else:
        T = _f32(T).copy(order="F")
        V = np.eye(T.shape[0], dtype=np.float32) if V is None else V
        V = _f32(V).copy(order="F")
        fn = lib().orc_jacobi_evd_f32
    n = T.shape[0]
    sw, rot = C.c_int(), C.c_longlong()
    hist = np.zeros(64)
    st = fn(_p(T), _p(V), n, b, tol, nu, rule, max_sweeps, max_rounds, C.byref(sw), C.byref(rot),
            _p(hist))
    return JacobiResult(T, V, sw.value, rot.value, st, hist[: min(sw.value + 1, 64)].copy())


def block_jacobi(T, V=None, *, b=32, tol=0.0, nu=20 * OMEGA, rule=0, max_sweeps=60,
                 max_inner=30) -> JacobiResult:
    """Classic block Jacobi with full inner diagonalisation of the 2b x 2b
    blocks (reading R26); rotations = inner rotations."""
    T = _f64(T).copy(order="F")
    n = T.shape[0]
    V = _f64(np.eye(n) if V is None else V).copy(order="F")
    sw, rot = C.c_int(), C.c_longlong()
    hist = np.zeros(64)
    st = lib().orc_block_jacobi_evd_f64(_p(T), _p(V), n, b, tol, nu, rule, max_sweeps, max_inner, C.byref(sw),
                                        C.byref(rot), _p(hist))
    return JacobiResult(T, V, sw.value, rot.value, st, hist[: min(sw.value + 1, 64)].copy())


def jacobi_rowcyclic(T, V=None, *, tol=0.0, nu=20 * OMEGA, rule=0, max_sweeps=60) -> JacobiResult:
    """Alg. 2 literally (row-cyclic)."""
    T = _f64(T).copy(order="F")
    n = T.shape[0]
    V = _f64(np.eye(n) if V is None else V).copy(order="F")
    sw, rot = C.c_int(), C.c_longlong()
    hist = np.zeros(64)
    st = lib().orc_jacobi_rowcyclic_f64(_p(T), _p(V), n, tol, nu, rule, max_sweeps, C.byref(sw),
                                        C.byref(rot), _p(hist))
    return JacobiResult(T, V, sw.value, rot.value, st, hist[: min(sw.value + 1, 64)].copy())


def mgs(Z):
    """Alg. 3 step 2: (Q, R, status)."""
    Z = _f64(Z)
    m, n = Z.shape
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n), order="F")
    st = lib().orc_mgs_f64(_p(Z), m, n, _p(Q), _p(R))
    return Q, R, st


def gemm(A, B, transA=False):
    A, B = _f64(A), _f64(B)
    if transA:
        k, m = A.shape
    else:
        m, k = A.shape
    n = B.shape[1]
    Cm = np.zeros((m, n), order="F")
    lib().orc_gemm_f64(int(transA), _p(A), _p(B), _p(Cm), m, n, k)
    return Cm


def qtaq(A, Q):
    """Alg. 3 step 3: symmetrised Q^T A Q."""
    A, Q = _f64(A), _f64(Q)
    n = A.shape[0]
    T = np.zeros((n, n), order="F")
    lib().orc_qtaq_f64(_p(A), _p(Q), n, _p(T))
    return T


def sort_desc(keys):
    keys = np.ascontiguousarray(keys, dtype=np.float64)
    perm = np.zeros(len(keys), dtype=np.int32)
    lib().orc_sort_desc(_p(keys), len(keys), _p(perm))
    return perm


def low_evd(A, cfg: Cfg | None = None):
    """Alg. 3 step 1 by the fp32 parallel Jacobi (reading R12, low_solver =
    LOW_JACOBI).  Returns (Z fp32, Report)."""
    A = _f64(A)
    n = A.shape[0]
    cfg = cfg or default_cfg("eig")
    Z = np.zeros((n, n), dtype=np.float32, order="F")
    rep = Report()
    lib().orc_low_evd(_p(A), n, C.byref(cfg), _p(Z), C.byref(rep))
    return Z, rep


def sytrd(A32):
    """Householder tridiagonalisation in binary32 (GvL Alg. 8.3.1, LAPACK
    reflector convention): (d, e, tau, Aout) with the reflectors v_k(1:) in
    Aout(k+2:, k)."""
    A = _f32(A32).copy(order="F")
    n = A.shape[0]
    d = np.zeros(n, dtype=np.float32)
    e = np.zeros(max(n - 1, 1), dtype=np.float32)
    tau = np.zeros(n, dtype=np.float32)
    lib().orc_sytrd_f32(_p(A), n, _p(d), _p(e), _p(tau))
    return d, e[: max(n - 1, 0)], tau, A


def orgtr(Aout, tau):
    """Q = H_0 ... H_{n-3} from sytrd's output (binary32)."""
    Aout = _f32(Aout)
    n = Aout.shape[0]
    Q = np.zeros((n, n), dtype=np.float32, order="F")
    lib().orc_orgtr_f32(_p(Aout), n, _p(np.ascontiguousarray(tau, dtype=np.float32)), _p(Q))
    return Q


def tridiag_qr(d, e, Z=None):
    """Symmetric QR algorithm (GvL Alg. 8.3.3, Wilkinson shift) on the
    tridiagonal (d, e) in binary32, rotations accumulated into Z (default I).
    Returns (eigenvalues unsorted, Z, implicit QR steps or -1)."""
    n = len(d)
    dd = np.ascontiguousarray(d, dtype=np.float32).copy()
    ee = np.zeros(max(n, 1), dtype=np.float32)
    ee[: n - 1] = e
    Z = _f32(np.eye(n, dtype=np.float32) if Z is None else Z).copy(order="F")
    steps = lib().orc_tridiag_qr_f32(_p(dd), _p(ee), n, _p(Z))
    return dd, Z, steps


def low_evd_symqr(A):
    """Alg. 3 step 1 by symmetric QR on fl32(A): (Z fp32 columns in
    descending eigenvalue order, lam32, Report)."""
    A = _f64(A)
    n = A.shape[0]
    Z = np.zeros((n, n), dtype=np.float32, order="F")
    lam = np.zeros(n, dtype=np.float32)
    rep = Report()
    lib().orc_low_evd_symqr(_p(A), n, _p(Z), _p(lam), C.byref(rep))
    return Z, lam, rep


@dataclass
class EvdResult:
    lam: np.ndarray
    V: np.ndarray
    status: int
    report: Report


def mp_evd(A, cfg: Cfg | None = None, Z=None) -> EvdResult:
    """Alg. 3 end to end."""
    A = _f64(A)
    n = A.shape[0]
    cfg = cfg or default_cfg("eig")
    lam = np.zeros(n)
    V = np.zeros((n, n), order="F")
    rep = Report()
    Zp = None if Z is None else _f32(Z)
    st = lib().orc_mp_evd(_p(A), n, C.byref(cfg), _p(Zp), _p(lam), _p(V), C.byref(rep))
    return EvdResult(lam, V, st, rep)


def plain_evd(A, cfg: Cfg | None = None) -> EvdResult:
    """Alg. 2 from T = A, P = I."""
    A = _f64(A)
    n = A.shape[0]
    cfg = cfg or default_cfg("eig")
    lam = np.zeros(n)
    V = np.zeros((n, n), order="F")
    rep = Report()
    st = lib().orc_plain_evd(_p(A), n, C.byref(cfg), _p(lam), _p(V), C.byref(rep))
    return EvdResult(lam, V, st, rep)


def jacobi_svd(Cm, V=None, *, b=32, eps_rel=0.1 * OMEGA, nu=OMEGA, early_stop=2e-4, max_sweeps=60,
               precision="f64") -> JacobiResult:
    """Alg. 4 loop (one-sided) with the block merry-go-round ordering."""
    if precision == "f64":
        Cm = _f64(Cm).copy(order="F")
        n = Cm.shape[1]
        V = _f64(np.eye(n) if V is None else V).copy(order="F")
        fn = lib().orc_jacobi_svd_f64
    else:
        Cm = _f32(Cm).copy(order="F")
        n = Cm.shape[1]
        V = _f32(np.eye(n, dtype=np.float32) if V is None else V).copy(order="F")
        fn = lib().orc_jacobi_svd_f32
    m = Cm.shape[0]
    sw, rot = C.c_int(), C.c_longlong()
    hist = np.zeros(64)
    rh = np.zeros(64)
    st = fn(_p(Cm), _p(V), m, n, b, eps_rel, nu, early_stop, max_sweeps, C.byref(sw),
            C.byref(rot), _p(hist), _p(rh))
    res = JacobiResult(Cm, V, sw.value, rot.value, st, hist[: min(sw.value + 1, 64)].copy())
    res.rot_hist = rh[: min(sw.value, 64)].copy()
    return res


def gram_offnorm(Cm):
    """(||off(C^T C)||_F, ||C^T C||_F) in long double."""
    Cm = _f64(Cm)
    o, t = C.c_double(), C.c_double()
    lib().orc_gram_offnorm(_p(Cm), Cm.shape[0], Cm.shape[1], C.byref(o), C.byref(t))
    return o.value, t.value


@dataclass
class SvdResult:
    sigma: np.ndarray
    U: np.ndarray
    V: np.ndarray
    status: int
    report: Report


def mp_svd(A, cfg: Cfg | None = None, Z=None) -> SvdResult:
    """Alg. 5 end to end."""
    A = _f64(A)
    m, n = A.shape
    cfg = cfg or default_cfg("svd")
    sig = np.zeros(n)
    U = np.zeros((m, n), order="F")
    V = np.zeros((n, n), order="F")
    rep = Report()
    Zp = None if Z is None else _f32(Z)
    st = lib().orc_mp_svd(_p(A), m, n, C.byref(cfg), _p(Zp), _p(sig), _p(U), _p(V), C.byref(rep))
    return SvdResult(sig, U, V, st, rep)


def plain_svd(A, cfg: Cfg | None = None) -> SvdResult:
    """Alg. 4 from C = A, V = I."""
    A = _f64(A)
    m, n = A.shape
    cfg = cfg or default_cfg("svd")
    sig = np.zeros(n)
    U = np.zeros((m, n), order="F")
    V = np.zeros((n, n), order="F")
    rep = Report()
    st = lib().orc_plain_svd(_p(A), m, n, C.byref(cfg), _p(sig), _p(U), _p(V), C.byref(rep))
    return SvdResult(sig, U, V, st, rep)


def mp_evd_batched(A, cfg: Cfg | None = None):
    """A: (batch, n, n) with each matrix column-major in A[k].T order, i.e.
    A[k] is the row-major image of the column-major matrix (symmetric inputs
    make the distinction moot).  Returns (lam (batch,n), V (batch,n,n) in the
    same convention, sweeps, sweeps_low, status)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    batch, n, _ = A.shape
    cfg = cfg or default_cfg("eig")
    lam = np.zeros((batch, n))
    V = np.zeros((batch, n, n))
    sw = np.zeros(batch, dtype=np.int32)
    swl = np.zeros(batch, dtype=np.int32)
    st = lib().orc_mp_evd_batched(_p(A), n, batch, C.byref(cfg), _p(lam), _p(V), _p(sw), _p(swl))
    return lam, V, sw, swl, st
