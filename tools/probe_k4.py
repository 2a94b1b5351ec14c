"""A few fp64 block rounds at n = 8192 (diag + 1e-6 random: every pair
rotates) for ncu captures of the fp64 apply kernel; MPJ_F64_APPLY selects it."""
import os
import sys

sys.path.insert(0, os.environ.get("MPJ_PKG_DIR", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_2211_03339_b200 as mpj

n = int(os.environ.get("N", "8192"))
g = torch.Generator(device="cuda").manual_seed(1)
R = torch.randn(n, n, device="cuda", dtype=torch.float64, generator=g)
T = torch.diag(torch.linspace(1, 2, n, device="cuda", dtype=torch.float64)) + 1e-6 * (R + R.T) / 2
del R
V = torch.eye(n, device="cuda", dtype=torch.float64)
cfg = mpj.default_config("eig", variant=mpj.VARIANT_BLOCK, block_b=32)
rounds = 63 + 32 * int(os.environ.get("BROUNDS", "4"))
mpj.profile_reset()
mpj.profile_enable(True)
r = mpj.jacobi(T, V, tol=0.0, max_sweeps=1, max_rounds=rounds, cfg=cfg)
torch.cuda.synchronize()
mpj.profile_enable(False)
sec, cnt = mpj.profile_get("block_apply_f64")
print(f"K4 fp64 ({os.environ.get('MPJ_F64_APPLY', 'default')}): {1e3 * sec / max(cnt, 1):.4f} ms/launch over {cnt}")
