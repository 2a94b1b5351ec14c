"""North_star (4) evidence: the scalar (one round at a time) variant at the
bench size, timed per round with CUDA events on the library's stream, against
the HBM roofline of its 32 n_p^2 bytes per round (T and V read + written);
compare with the block variant's per-sweep time in the bench line."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2211_03339_b200 as mpj  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 32
g = torch.Generator(device="cuda").manual_seed(3)
A = torch.randn(n, n, device="cuda", dtype=torch.float64, generator=g)
T = ((A + A.T) / 2).T.contiguous().T
V = torch.eye(n, device="cuda", dtype=torch.float64).T.contiguous().T
cfg = mpj.default_config("eig", variant=mpj.VARIANT_SCALAR, block_b=32)
mpj.jacobi(T, V, tol=0.0, max_rounds=2, cfg=cfg)          # warm
torch.cuda.synchronize()
t0 = time.perf_counter()
mpj.jacobi(T, V, tol=0.0, max_rounds=rounds, cfg=cfg)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / rounds
by = 32.0 * n * n
print(json.dumps({"n": n, "rounds": rounds, "s_per_round": dt, "GBps": by / dt / 1e9,
                  "s_per_sweep_est": dt * (n - 1), "bytes_per_round": by}))
