"""Per-call timings of mpj.eig (MP and plain) at n = 1024 (config 2 rows)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_03339_b200 as mpj
import workloads as W

n = 1024
for kind, gen, mode in (("uniform", W.example1, 4), ("clustered", W.example2, 4), ("one large", W.example1, 1)):
    kappa = 1e3
    A, _ = gen(n, kappa, mode, W.seed_for(2, mode, kappa))
    At = torch.from_numpy(A).cuda()
    for plain in (False, True):
        ts = []
        for i in range(5):
            mpj.profile_reset(); mpj.profile_enable(True)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            r = mpj.eig(At, plain=plain)
            torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
            mpj.profile_enable(False)
        rep = r.report
        ks = {k: round(1e3 * mpj.profile_get(k)[0], 2) for k in ("block_apply_f64", "block_solve_f64", "block_apply_f32",
                                                                  "block_solve_f32", "symqr_sytrd", "symqr_trieig",
                                                                  "symqr_backtransform")}
        print(kind, "plain" if plain else "mp", "ms/call", [round(t, 1) for t in ts], "sweeps", r.sweeps, rep.sweeps_low,
              "stages", round(rep.t_low * 1e3, 1), round(rep.t_orth * 1e3, 1), round(rep.t_precond * 1e3, 1), round(rep.t_jacobi * 1e3, 1), ks, flush=True)
