"""Experiment (not product code): does a LAPACK-class low-precision stage
(the paper's own step 1: symmetric QR / ssyevd) save fp64
sweeps over the fp32 Jacobi stage (reading R12)?  Z from torch.linalg.eigh in
float32 (cuSOLVER syevd) is fed to mpjacobi_eig_z; optionally refined by fp32
Jacobi sweeps on fl32(Z^T A Z) first.  Prints one JSON line per case."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2211_03339_b200 as mpj  # noqa: E402
import workloads as W  # noqa: E402

UPS = 2.0 ** -24


def run(n, mode, kappa):
    A, lam = W.example1_torch(n, kappa, mode, W.seed_for(4, mode, kappa))
    A = A.T  # column-major view (symmetric)
    out = []
    torch.cuda.synchronize()
    r = mpj.eig(A, Z_out=True)
    torch.cuda.synchronize()
    t0 = time.time(); r = mpj.eig(A, Z_out=True); torch.cuda.synchronize(); t = time.time() - t0
    rep = r.report
    out.append(dict(case="jacobi32", n=n, mode=mode, kappa=kappa, sweeps=r.sweeps, sweeps_low=rep.sweeps_low,
                    off0=rep.off0 / rep.norm_a, t=t, t_low=rep.t_low, t_jac=rep.t_jacobi,
                    hist=[x / rep.norm_a for x in rep.off_hist[: r.sweeps + 1]]))
    torch.cuda.synchronize()
    t0 = time.time()
    w, Z = torch.linalg.eigh(A.float())
    torch.cuda.synchronize()
    t_eigh = time.time() - t0
    Z = Z.flip(1).contiguous()
    Zc = Z.T.contiguous().T
    r2 = mpj.eig(A, Z_in=Zc)
    torch.cuda.synchronize()
    t0 = time.time(); r2 = mpj.eig(A, Z_in=Zc); torch.cuda.synchronize(); t = time.time() - t0
    rep = r2.report
    out.append(dict(case="ssyevd", n=n, mode=mode, kappa=kappa, sweeps=r2.sweeps, off0=rep.off0 / rep.norm_a,
                    t=t, t_eigh=t_eigh, t_jac=rep.t_jacobi,
                    hist=[x / rep.norm_a for x in rep.off_hist[: r2.sweeps + 1]]))
    # refine: fp32 Jacobi on fl32(Z^T A Z) accumulating into Z
    for epsf in (0.0, 1000.0):
        A32 = A.float()
        T = (Z.T @ A32 @ Z)
        T = 0.5 * (T + T.T)
        T = T.T.contiguous().T
        V = Z.clone().T.contiguous().T
        nA32 = torch.linalg.norm(A32).item()
        ef = epsf if epsf > 0 else max(10.0, 1.25 * n ** 0.5)
        torch.cuda.synchronize(); t0 = time.time()
        jr = mpj.jacobi(T, V, tol=ef * UPS * nA32, nu=float(torch.tensor(20 * UPS, dtype=torch.float32)),
                        max_sweeps=60)
        torch.cuda.synchronize(); tj = time.time() - t0
        r3 = mpj.eig(A, Z_in=V)
        rep = r3.report
        out.append(dict(case=f"ssyevd+jacobi32(eps={ef:.0f}u)", n=n, mode=mode, kappa=kappa, sweeps=r3.sweeps,
                        refine_sweeps=jr.sweeps, t_refine=tj, off0=rep.off0 / rep.norm_a, t_jac=rep.t_jacobi,
                        hist=[x / rep.norm_a for x in rep.off_hist[: r3.sweeps + 1]]))
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        n, mode, kappa = spec.split(",")
        run(int(n), int(mode), float(kappa))
