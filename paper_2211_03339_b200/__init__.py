"""Python binding of the mixed-precision Jacobi C ABI (include/mpjacobi.h).

Argument marshalling only: every step of the method runs in the CUDA kernels of
libmpjacobi.so (built in-tree by ``paper_2211_03339_b200.build.build()``).  The
binding fails loudly when the library is missing -- there is no CPU fallback.

Matrices are column-major on the C side.  A torch tensor ``X`` of shape
(rows, cols) is passed as-is when it is already column-major
(``X.stride() == (1, ld)``, e.g. ``Y.T`` for a contiguous ``Y``); otherwise a
column-major copy is made.  Outputs are returned as column-major tensors viewed
in math orientation (``out[i, j]`` is entry (i, j)).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpjacobi.so")

OMEGA = 2.0 ** -53
UPSILON = 2.0 ** -24

MPJ_OK, MPJ_ERR_INVALID, MPJ_ERR_NOCONV, MPJ_ERR_RANKDEF = 0, 1, 2, 3
MPJ_ERR_NONFINITE, MPJ_ERR_CUDA, MPJ_ERR_NCCL, MPJ_ERR_NOMEM = 4, 5, 6, 7
VARIANT_AUTO, VARIANT_SCALAR, VARIANT_BLOCK, VARIANT_BLOCK_FULL = 0, 1, 2, 3
LOW_AUTO, LOW_JACOBI, LOW_SYMQR = 0, 1, 2
ORTH_AUTO, ORTH_HOUSEHOLDER, ORTH_CGS, ORTH_SERIES = 0, 1, 2, 3

STATUS_NAMES = {0: "OK", 1: "INVALID", 2: "NOCONV", 3: "RANKDEF", 4: "NONFINITE", 5: "CUDA",
                6: "NCCL", 7: "NOMEM"}


class MpjError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"mpjacobi: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class mpj_config(C.Structure):
    _fields_ = [
        ("eps_factor", C.c_double), ("nu_factor", C.c_double), ("eps_low_factor", C.c_double),
        ("nu_low_factor", C.c_double), ("early_stop_ratio", C.c_double), ("max_sweeps", C.c_int),
        ("max_sweeps_low", C.c_int), ("stop_rule", C.c_int), ("variant", C.c_int), ("block_b", C.c_int),
        ("low_solver", C.c_int), ("orth", C.c_int),
    ]


class mpj_report(C.Structure):
    _fields_ = [
        ("sweeps", C.c_int), ("sweeps_low", C.c_int), ("status", C.c_int), ("status_low", C.c_int),
        ("rotations", C.c_longlong), ("rotations_low", C.c_longlong), ("norm_a", C.c_double),
        ("off0", C.c_double), ("off_hist", C.c_double * 64), ("t_low", C.c_double),
        ("t_orth", C.c_double), ("t_precond", C.c_double), ("t_jacobi", C.c_double),
        ("t_extract", C.c_double), ("t_total", C.c_double), ("n_padded", C.c_int), ("block_b", C.c_int),
        ("variant", C.c_int), ("launches", C.c_longlong), ("off_hist_low", C.c_double * 64),
        ("rot_hist", C.c_longlong * 64),
    ]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("off_hist", "off_hist_low", "rot_hist")}
        d["rot_hist"] = list(self.rot_hist[: self.sweeps])
        d["off_hist"] = list(self.off_hist[: max(self.sweeps + 1, 1)])
        d["off_hist_low"] = list(self.off_hist_low[: max(self.sweeps_low + 1, 1)])
        return d


_lib = None
_vp, _i64, _dp = C.c_void_p, C.c_int64, C.c_double


def lib():
    """Load libmpjacobi.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the CUDA library is the only implementation; there is no fallback)")
        L = C.CDLL(LIB_PATH)
        cfgp, repp = C.POINTER(mpj_config), C.POINTER(mpj_report)
        L.mpj_config_default_eig.argtypes = [cfgp]
        L.mpj_config_default_svd.argtypes = [cfgp]
        L.mpjacobi_last_error.restype = C.c_char_p
        L.mpjacobi_launch_count.restype = C.c_longlong
        L.mpjacobi_eig_workspace.restype = C.c_size_t
        L.mpjacobi_eig_workspace.argtypes = [_i64, cfgp]
        eig_args = [_vp, _i64, _i64, _vp, _vp, _i64, C.POINTER(C.c_int), _vp, C.c_size_t, _vp, cfgp, repp]
        for nm in ("mpjacobi_eig", "mpjacobi_eig_plain"):
            getattr(L, nm).restype = C.c_int
            getattr(L, nm).argtypes = eig_args
        L.mpjacobi_eig_z.restype = C.c_int
        L.mpjacobi_eig_z.argtypes = eig_args[:3] + [_vp, _vp, _i64] + eig_args[3:]
        for nm in ("mpjacobi_jacobi_f64", "mpjacobi_jacobi_f32"):
            getattr(L, nm).restype = C.c_int
            getattr(L, nm).argtypes = [_vp, _i64, _vp, _i64, _i64, _dp, _dp, C.c_int, _i64,
                                       C.POINTER(C.c_int), C.POINTER(C.c_longlong), C.POINTER(C.c_double),
                                       _vp, cfgp]
        L.mpjacobi_sytrd.restype = C.c_int
        L.mpjacobi_sytrd.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp]
        L.mpjacobi_tridiag_eig.restype = C.c_int
        L.mpjacobi_tridiag_eig.argtypes = [_vp, _vp, _i64, _vp, _vp, _i64, _vp]
        L.mpjacobi_orth_householder.restype = C.c_int
        L.mpjacobi_orth_householder.argtypes = [_vp, _vp, _i64, _vp]
        L.mpjacobi_orth_series.restype = C.c_int
        L.mpjacobi_orth_series.argtypes = [_vp, _vp, _i64, _vp]
        L.mpjacobi_orth.restype = C.c_int
        L.mpjacobi_orth.argtypes = [_vp, _vp, _i64, _vp]
        L.mpjacobi_precond.restype = C.c_int
        L.mpjacobi_precond.argtypes = [_vp, _vp, _vp, _i64, _vp]
        L.mpjacobi_dgemm.restype = C.c_int
        L.mpjacobi_dgemm.argtypes = [C.c_int, _vp, _vp, _vp, _i64, _i64, _i64, _vp]
        L.mpjacobi_profile_enable.argtypes = [C.c_int]
        L.mpjacobi_profile_get.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_longlong)]
        if hasattr(L, "mpjacobi_svd"):
            L.mpjacobi_svd_workspace.restype = C.c_size_t
            L.mpjacobi_svd_workspace.argtypes = [_i64, _i64, cfgp]
            L.mpjacobi_svd.restype = C.c_int
            L.mpjacobi_svd.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _i64,
                                       C.POINTER(C.c_int), _vp, C.c_size_t, _vp, cfgp, repp]
            L.mpjacobi_svd_z.restype = C.c_int
            L.mpjacobi_svd_z.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _i64,
                                         C.POINTER(C.c_int), _vp, C.c_size_t, _vp, cfgp, repp]
        L.mpjacobi_eig_mg.restype = C.c_int
        L.mpjacobi_eig_mg.argtypes = [_vp, _i64, _i64, _vp, _vp, _i64, C.POINTER(C.c_int), _vp, C.c_int, C.c_int,
                                      C.c_int, _vp, cfgp, repp]
        L.mpjacobi_svd_mg.restype = C.c_int
        L.mpjacobi_svd_mg.argtypes = [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _i64, C.POINTER(C.c_int), _vp,
                                      C.c_int, C.c_int, C.c_int, _vp, cfgp, repp]
        L.mpjacobi_svd_mg_plan.restype = C.c_int
        L.mpjacobi_svd_mg_plan.argtypes = [_i64, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), _vp, _vp, _vp]
        L.mpjacobi_mg_plan.restype = C.c_int
        L.mpjacobi_mg_plan.argtypes = [_i64, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), _vp, _vp, _vp]
        L.mpjacobi_nccl_unique_id.restype = C.c_int
        L.mpjacobi_nccl_unique_id.argtypes = [_vp, C.c_size_t]
        if hasattr(L, "mpjacobi_eig_batched"):
            L.mpjacobi_eig_batched.restype = C.c_int
            L.mpjacobi_eig_batched.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, cfgp]
            L.mpjacobi_eig_batched_z.restype = C.c_int
            L.mpjacobi_eig_batched_z.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, cfgp]
        _lib = L
    return _lib


EXPORTED = (
    "mpj_config_default_eig", "mpj_config_default_svd", "mpjacobi_eig_workspace", "mpjacobi_eig",
    "mpjacobi_eig_plain", "mpjacobi_jacobi_f64", "mpjacobi_jacobi_f32", "mpjacobi_orth",
    "mpjacobi_precond", "mpjacobi_dgemm", "mpjacobi_svd_workspace", "mpjacobi_svd",
    "mpjacobi_eig_batched", "mpjacobi_last_error", "mpjacobi_launch_count",
    "mpjacobi_profile_enable", "mpjacobi_profile_reset", "mpjacobi_profile_get",
    "mpjacobi_eig_mg", "mpjacobi_nccl_unique_id", "mpjacobi_mg_plan", "mpjacobi_eig_z", "mpjacobi_svd_z",
    "mpjacobi_sytrd", "mpjacobi_tridiag_eig", "mpjacobi_orth_householder", "mpjacobi_eig_batched_z",
    "mpjacobi_svd_mg", "mpjacobi_svd_mg_plan", "mpjacobi_orth_series",
)


def _check(status, ok=(MPJ_OK,)):
    if status not in ok:
        raise MpjError(status, lib().mpjacobi_last_error().decode())
    return status


def default_config(kind: str = "eig", **kw) -> mpj_config:
    c = mpj_config()
    (lib().mpj_config_default_eig if kind == "eig" else lib().mpj_config_default_svd)(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def launch_count() -> int:
    return lib().mpjacobi_launch_count()


def profile_enable(on: bool = True):
    """Time the library's dominant kernels with CUDA events on their own stream."""
    lib().mpjacobi_profile_enable(1 if on else 0)


def profile_reset():
    lib().mpjacobi_profile_reset()


def profile_get(kernel: str):
    """(seconds, launches) accumulated for a kernel name (see mpjacobi.h)."""
    sec, n = C.c_double(0), C.c_longlong(0)
    lib().mpjacobi_profile_get(kernel.encode(), C.byref(sec), C.byref(n))
    return sec.value, n.value


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def colmajor(x: torch.Tensor) -> torch.Tensor:
    """Column-major version of x (rows, cols): a view when already column-major."""
    if x.dim() != 2:
        raise ValueError("expected a matrix")
    if x.stride(0) == 1 and x.stride(1) >= max(1, x.shape[0]):
        return x
    return x.T.contiguous().T


def empty_colmajor(rows, cols, dtype=torch.float64, device="cuda", pin=False):
    if device == "cpu":
        return torch.empty((cols, rows), dtype=dtype, pin_memory=pin).T
    return torch.empty((cols, rows), dtype=dtype, device=device).T


@dataclass
class EigResult:
    lam: torch.Tensor
    V: torch.Tensor
    sweeps: int
    report: mpj_report
    Z: torch.Tensor | None = None


def _z_args(n, Z_in, Z_out, dev):
    """(Z_in column-major or None, Z_out tensor or None, ldz) for the *_z entry points."""
    zi = None
    if Z_in is not None:
        if Z_in.shape != (n, n) or Z_in.dtype != torch.float32:
            raise ValueError("Z_in must be an (n, n) float32 matrix")
        zi = colmajor(Z_in)
    zo = empty_colmajor(n, n, dtype=torch.float32, device=dev.type, pin=(dev.type == "cpu")) if Z_out else None
    ld = zi.stride(1) if zi is not None else n
    if zi is not None and zo is not None and ld != n:
        zi = zi.T.contiguous().T
        ld = n
    return zi, zo, max(ld, n)


def mpjacobi_eig(A, cfg: mpj_config | None = None, *, plain=False, workspace=None, out=None,
                 allow_noconv=False, Z_in=None, Z_out=False) -> EigResult:
    """Alg. 3 (or Alg. 2 with plain=True).  A: (n, n) float64 tensor on the GPU
    or on the host (host tensors are staged by the library; pin them for async
    copies).  Returns descending eigenvalues and column-major eigenvectors.
    Z_in (n, n) float32 replaces the low-precision stage's output (step 1,
    P:188); Z_out=True returns the Z step 2 consumed in ``.Z``
    (mpjacobi_eig_z)."""
    n = A.shape[0]
    if A.shape != (n, n) or A.dtype != torch.float64:
        raise ValueError("A must be a square float64 matrix")
    Acm = colmajor(A)
    dev = Acm.device
    if out is None:
        lam = torch.empty(n, dtype=torch.float64, device=dev, pin_memory=(dev.type == "cpu"))
        V = empty_colmajor(n, n, device=dev.type, pin=(dev.type == "cpu"))
    else:
        lam, V = out
    cfg = cfg or default_config("eig")
    rep = mpj_report()
    sw = C.c_int(0)
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        ws_ptr, ws_bytes = _ptr(workspace), workspace.numel() * workspace.element_size()
    zo = None
    if Z_in is not None or Z_out:
        if plain:
            raise ValueError("Z_in / Z_out apply to Alg. 3 only")
        zi, zo, ldz = _z_args(n, Z_in, Z_out, dev)
        st = lib().mpjacobi_eig_z(_ptr(Acm), n, Acm.stride(1), _ptr(zi), _ptr(zo), ldz, _ptr(lam), _ptr(V),
                                  V.stride(1), C.byref(sw), ws_ptr, ws_bytes, _stream(), C.byref(cfg), C.byref(rep))
    else:
        fn = lib().mpjacobi_eig_plain if plain else lib().mpjacobi_eig
        st = fn(_ptr(Acm), n, Acm.stride(1), _ptr(lam), _ptr(V), V.stride(1), C.byref(sw), ws_ptr, ws_bytes,
                _stream(), C.byref(cfg), C.byref(rep))
    _check(st, (MPJ_OK, MPJ_ERR_NOCONV) if allow_noconv else (MPJ_OK,))
    return EigResult(lam, V, sw.value, rep, zo)


def eig_workspace(n, cfg: mpj_config | None = None, device="cuda"):
    nbytes = lib().mpjacobi_eig_workspace(n, C.byref(cfg or default_config("eig")))
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


@dataclass
class JacobiResult:
    sweeps: int
    rotations: int
    status: int
    off_hist: list


def mpjacobi_jacobi(T, V, *, tol=0.0, nu=20 * OMEGA, max_sweeps=60, max_rounds=-1,
                    cfg: mpj_config | None = None) -> JacobiResult:
    """Alg. 2 / Alg. 3 steps 4-11 in place on device T (symmetric) and V.
    float64 or float32 tensors, column-major (symmetric T makes either layout
    valid; V must be column-major or is copied back)."""
    n = T.shape[0]
    fn = lib().mpjacobi_jacobi_f64 if T.dtype == torch.float64 else lib().mpjacobi_jacobi_f32
    Vc = colmajor(V)
    Tc = colmajor(T)
    sw, rot = C.c_int(0), C.c_longlong(0)
    hist = (C.c_double * 64)()
    st = fn(_ptr(Tc), Tc.stride(1), _ptr(Vc), Vc.stride(1), n, tol, nu, max_sweeps, max_rounds,
            C.byref(sw), C.byref(rot), hist, _stream(), C.byref(cfg) if cfg is not None else None)
    _check(st, (MPJ_OK, MPJ_ERR_NOCONV))
    if Vc.data_ptr() != V.data_ptr():
        V.copy_(Vc)
    if Tc.data_ptr() != T.data_ptr():
        T.copy_(Tc)
    return JacobiResult(sw.value, rot.value, st, list(hist[: min(sw.value + 1, 64)]))


def mpjacobi_sytrd(A32):
    """Alg. 3 step 1, part 1: binary32 Householder tridiagonalisation
    of a symmetric float32 CUDA matrix.  Returns (d, e, tau, Aout) with the
    reflectors in Aout (LAPACK lower layout)."""
    n = A32.shape[0]
    ld = (n + 3) // 4 * 4      # leading dimension a multiple of 4 (16-byte TMA strides)
    buf = torch.zeros((n, ld), dtype=torch.float32, device=A32.device)
    buf[:, :n] = A32.T         # buf row j = column j of A (column-major with ld)
    d = torch.empty(n, dtype=torch.float32, device=A32.device)
    e = torch.empty(max(n - 1, 1), dtype=torch.float32, device=A32.device)
    tau = torch.empty(n, dtype=torch.float32, device=A32.device)
    _check(lib().mpjacobi_sytrd(_ptr(buf), n, ld, _ptr(d), _ptr(e), _ptr(tau), _stream()))
    return d, e[: n - 1], tau, buf[:, :n].T


def mpjacobi_tridiag_eig(d, e):
    """Eigenpairs (binary64) of the tridiagonal (d, e) (float32 CUDA vectors):
    (lam descending, Y column-major)."""
    n = d.shape[0]
    lam = torch.empty(n, dtype=torch.float64, device=d.device)
    Y = empty_colmajor(n, n, device=d.device.type)
    ee = e if n > 1 else torch.zeros(1, dtype=torch.float32, device=d.device)
    _check(lib().mpjacobi_tridiag_eig(_ptr(d.contiguous()), _ptr(ee.contiguous()), n, _ptr(lam), _ptr(Y), n,
                                      _stream()))
    return lam, Y


def mpjacobi_orth(Z, method="cgs"):
    """Alg. 3 step 2: the QR factor Q of a square column-major device matrix
    (method "cgs": blocked CGS + CholeskyQR2; "householder": blocked
    Householder QR; "series": Cholesky QR with the fixed-point factor, R10b)."""
    n = Z.shape[0]
    Zc = colmajor(Z)
    if Zc.stride(1) != n:
        Zc = Zc.T.contiguous().T
    Q = empty_colmajor(n, n)
    fn = {"householder": lib().mpjacobi_orth_householder, "series": lib().mpjacobi_orth_series,
          "cgs": lib().mpjacobi_orth}[method]
    _check(fn(_ptr(Zc), _ptr(Q), n, _stream()))
    return Q


def mpjacobi_precond(A, Q):
    """Alg. 3 step 3: symmetrised Q^T A Q (device, fp64)."""
    n = A.shape[0]
    Ac = colmajor(A)
    Qc = colmajor(Q)
    if Ac.stride(1) != n:
        Ac = Ac.T.contiguous().T
    if Qc.stride(1) != n:
        Qc = Qc.T.contiguous().T
    T = empty_colmajor(n, n)
    _check(lib().mpjacobi_precond(_ptr(Ac), _ptr(Qc), _ptr(T), n, _stream()))
    return T


def mpjacobi_dgemm(A, B, transa=False):
    """C = op(A) B with the library's DMMA GEMM (parity tests)."""
    Ac, Bc = colmajor(A).T.contiguous().T, colmajor(B).T.contiguous().T
    m = Ac.shape[1] if transa else Ac.shape[0]
    k = Ac.shape[0] if transa else Ac.shape[1]
    n = Bc.shape[1]
    Cm = empty_colmajor(m, n)
    _check(lib().mpjacobi_dgemm(1 if transa else 0, _ptr(Ac), _ptr(Bc), _ptr(Cm), m, n, k, _stream()))
    return Cm


@dataclass
class SvdResult:
    sigma: torch.Tensor   # (n,) descending
    U: torch.Tensor       # (m, n) column-major, math orientation
    V: torch.Tensor       # (n, n) column-major, math orientation
    sweeps: int
    report: mpj_report
    Z: torch.Tensor | None = None


def mpjacobi_svd(A, cfg: mpj_config | None = None, *, workspace=None, out=None,
                 allow_noconv=False, Z_in=None, Z_out=False) -> SvdResult:
    """Alg. 5: A (m, n), m >= n, float64, on the GPU or the host.
    Z_in / Z_out as in eig() (step 1's n x n Z; mpjacobi_svd_z)."""
    m, n = A.shape
    if A.dtype != torch.float64 or m < n:
        raise ValueError("A must be float64 with m >= n")
    Acm = colmajor(A)
    dev = Acm.device
    pin = dev.type == "cpu"
    if out is None:
        sig = torch.empty(n, dtype=torch.float64, device=dev, pin_memory=pin)
        U = empty_colmajor(m, n, device=dev.type, pin=pin)
        V = empty_colmajor(n, n, device=dev.type, pin=pin)
    else:
        sig, U, V = out
    cfg = cfg or default_config("svd")
    rep = mpj_report()
    sw = C.c_int(0)
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        ws_ptr, ws_bytes = _ptr(workspace), workspace.numel() * workspace.element_size()
    zo = None
    if Z_in is not None or Z_out:
        zi, zo, ldz = _z_args(n, Z_in, Z_out, dev)
        st = lib().mpjacobi_svd_z(_ptr(Acm), m, n, Acm.stride(1), _ptr(zi), _ptr(zo), ldz, _ptr(sig), _ptr(U),
                                  U.stride(1), _ptr(V), V.stride(1), C.byref(sw), ws_ptr, ws_bytes, _stream(),
                                  C.byref(cfg), C.byref(rep))
    else:
        st = lib().mpjacobi_svd(_ptr(Acm), m, n, Acm.stride(1), _ptr(sig), _ptr(U), U.stride(1), _ptr(V),
                                V.stride(1), C.byref(sw), ws_ptr, ws_bytes, _stream(), C.byref(cfg), C.byref(rep))
    _check(st, (MPJ_OK, MPJ_ERR_NOCONV) if allow_noconv else (MPJ_OK,))
    return SvdResult(sig, U, V, sw.value, rep, zo)


def svd_workspace(m, n, cfg: mpj_config | None = None, device="cuda"):
    nbytes = lib().mpjacobi_svd_workspace(m, n, C.byref(cfg or default_config("svd")))
    return torch.empty(nbytes, dtype=torch.uint8, device=device)


@dataclass
class BatchedResult:
    lam: torch.Tensor          # (batch, n), descending per matrix
    V: torch.Tensor            # (batch, n, n), V[k][i, j] = entry (i, j) of matrix k's eigenvectors
    sweeps: torch.Tensor       # (batch,) int32 fp64 sweeps
    sweeps_low: torch.Tensor   # (batch,) int32 fp32 sweeps
    status: int
    Z: torch.Tensor | None = None   # (batch, n, n) float32 step-1 output (Z_out=True)


def mpjacobi_eig_batched(A, cfg: mpj_config | None = None, allow_noconv=False, Z_in=None,
                         Z_out=False) -> BatchedResult:
    """Batched Alg. 3, one matrix per CTA (n <= 64).  A: (batch, n, n) float64
    CUDA tensor; A[k] is matrix k (symmetric, so either memory order is its
    column-major image).  Outputs are column-major per matrix, returned as
    math-orientation views.  Z_in: (batch, n, n) float32 CUDA tensor, step 1's
    output Z[k] (math orientation) -- step 1 is skipped; Z_out: return the Z
    step 2 consumed (mpjacobi_eig_batched_z)."""
    if A.dim() != 3 or A.shape[1] != A.shape[2] or A.dtype != torch.float64 or not A.is_cuda:
        raise ValueError("A must be a (batch, n, n) float64 CUDA tensor")
    batch, n, _ = A.shape
    Ac = A.transpose(1, 2).contiguous()          # memory of matrix k = column-major image of A[k]
    lam = torch.empty((batch, n), dtype=torch.float64, device=A.device)
    V = torch.empty((batch, n, n), dtype=torch.float64, device=A.device)
    sw = torch.empty(batch, dtype=torch.int32, device=A.device)
    swl = torch.empty(batch, dtype=torch.int32, device=A.device)
    zi = None
    if Z_in is not None:
        if Z_in.shape != A.shape or Z_in.dtype != torch.float32 or not Z_in.is_cuda:
            raise ValueError("Z_in must be a (batch, n, n) float32 CUDA tensor")
        zi = Z_in.transpose(1, 2).contiguous()   # column-major per matrix
    zo = torch.empty((batch, n, n), dtype=torch.float32, device=A.device) if Z_out else None
    st = lib().mpjacobi_eig_batched_z(_ptr(Ac), n, batch, _ptr(zi) if zi is not None else None,
                                      _ptr(zo) if zo is not None else None, _ptr(lam), _ptr(V), _ptr(sw),
                                      _ptr(swl), _stream(), C.byref(cfg or default_config("eig")))
    _check(st, (MPJ_OK, MPJ_ERR_NOCONV) if allow_noconv else (MPJ_OK,))
    return BatchedResult(lam, V.transpose(1, 2), sw, swl, st, zo.transpose(1, 2) if zo is not None else None)


def svd_mg_plan(n: int, nranks: int):
    """The partition plan of mpjacobi_svd_mg (host-only, no GPU): (n_p,
    pairs[rounds, mb, 2], moves: list per round transition of (blk, src, dst))."""
    import numpy as np
    npd, rounds = C.c_int(0), C.c_int(0)
    _check(lib().mpjacobi_svd_mg_plan(n, nranks, C.byref(npd), C.byref(rounds), None, None, None))
    mb = npd.value // 64
    pairs = np.zeros((rounds.value, mb, 2), dtype=np.int32)
    mv = np.zeros((max(rounds.value - 1, 1), 4 * nranks, 3), dtype=np.int32)
    nm = np.zeros(max(rounds.value - 1, 1), dtype=np.int32)
    _check(lib().mpjacobi_svd_mg_plan(n, nranks, None, None, pairs.ctypes.data, mv.ctypes.data, nm.ctypes.data))
    return npd.value, pairs, [mv[r, : nm[r]].tolist() for r in range(rounds.value - 1)]


def mg_plan(n: int, nranks: int):
    """The partition plan of one sweep of eig_mg (host-only, no GPU):
    (n_p, slots[rounds, mb, 4], xfers: list per round of (src, sphys, dst, dphys))."""
    import numpy as np
    npd, rounds = C.c_int(0), C.c_int(0)
    _check(lib().mpjacobi_mg_plan(n, nranks, C.byref(npd), C.byref(rounds), None, None, None))
    mb = npd.value // 64
    slots = np.zeros((rounds.value, mb, 4), dtype=np.int32)
    xf = np.zeros((rounds.value, 4 * nranks, 4), dtype=np.int32)
    nx = np.zeros(rounds.value, dtype=np.int32)
    _check(lib().mpjacobi_mg_plan(n, nranks, None, None, slots.ctypes.data, xf.ctypes.data, nx.ctypes.data))
    return npd.value, slots, [xf[r, : nx[r]].tolist() for r in range(rounds.value)]


def nccl_unique_id() -> bytes:
    """128-byte NCCL id (rank 0 creates it, then broadcasts it)."""
    buf = C.create_string_buffer(128)
    _check(lib().mpjacobi_nccl_unique_id(buf, 128))
    return buf.raw


def mpjacobi_eig_mg(A, cfg: mpj_config | None = None, *, nccl_id: bytes | None = None, rank: int = 0,
                    nranks: int = 1, emulate_ranks: int = 1, out=None, allow_noconv=False) -> EigResult:
    """Multi-GPU Alg. 3 (column-block partition).  With nccl_id (bytes from
    nccl_unique_id() on rank 0, broadcast with torch.distributed), one call per
    rank/GPU; without it, `emulate_ranks` ranks run inside this process on the
    current GPU.  A (full, every rank) and the replicated outputs as in eig()."""
    n = A.shape[0]
    Acm = colmajor(A)
    dev = Acm.device
    if out is None:
        lam = torch.empty(n, dtype=torch.float64, device=dev, pin_memory=(dev.type == "cpu"))
        V = empty_colmajor(n, n, device=dev.type, pin=(dev.type == "cpu"))
    else:
        lam, V = out
    cfg = cfg or default_config("eig")
    rep = mpj_report()
    sw = C.c_int(0)
    idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    st = lib().mpjacobi_eig_mg(_ptr(Acm), n, Acm.stride(1), _ptr(lam), _ptr(V), V.stride(1), C.byref(sw), idbuf,
                               rank, nranks, emulate_ranks, _stream(), C.byref(cfg), C.byref(rep))
    _check(st, (MPJ_OK, MPJ_ERR_NOCONV) if allow_noconv else (MPJ_OK,))
    return EigResult(lam, V, sw.value, rep)


def mpjacobi_svd_mg(A, cfg: mpj_config | None = None, *, nccl_id: bytes | None = None, rank: int = 0,
                    nranks: int = 1, emulate_ranks: int = 1, allow_noconv=False) -> SvdResult:
    """Multi-GPU Alg. 5 (column partition of the one-sided rotations,
    SURVEY 8(f) row 2): one call per rank with nccl_id, or `emulate_ranks`
    ranks inside this process.  A (m, n), m >= n, float64 (host or device, the
    same on every rank); Sigma, U, V returned on the current GPU, replicated."""
    m, n = A.shape
    if A.dtype != torch.float64 or m < n:
        raise ValueError("A must be float64 with m >= n")
    Acm = colmajor(A)
    sig = torch.empty(n, dtype=torch.float64, device="cuda")
    U = empty_colmajor(m, n, device="cuda")
    V = empty_colmajor(n, n, device="cuda")
    cfg = cfg or default_config("svd")
    rep = mpj_report()
    sw = C.c_int(0)
    idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    st = lib().mpjacobi_svd_mg(_ptr(Acm), m, n, Acm.stride(1), _ptr(sig), _ptr(U), U.stride(1), _ptr(V), V.stride(1),
                               C.byref(sw), idbuf, rank, nranks, emulate_ranks, _stream(), C.byref(cfg), C.byref(rep))
    _check(st, (MPJ_OK, MPJ_ERR_NOCONV) if allow_noconv else (MPJ_OK,))
    return SvdResult(sig, U, V, sw.value, rep, None)


# short aliases
svd_mg = mpjacobi_svd_mg
eig_mg = mpjacobi_eig_mg
eig_batched = mpjacobi_eig_batched
svd = mpjacobi_svd
eig = mpjacobi_eig
jacobi = mpjacobi_jacobi
orth = mpjacobi_orth
sytrd = mpjacobi_sytrd
tridiag_eig = mpjacobi_tridiag_eig
precond = mpjacobi_precond
dgemm = mpjacobi_dgemm
