"""Is the fp64 apply power-bound?  One fp64 block sweep at n = 8192 on (a) a
dense random symmetric matrix and (b) diag + 1e-6 random (every pair still
rotates, U ~ I): same work, different operand bit patterns.  Reports the
average K4 launch time and the SM clock / power sampled every 50 ms."""
import os
import statistics
import subprocess
import sys
import threading

sys.path.insert(0, os.environ.get("MPJ_PKG_DIR", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_2211_03339_b200 as mpj


def sample(stop, rows):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    for line in p.stdout:
        rows.append(line.strip())
        if stop.is_set():
            break
    p.terminate()


n = 8192
g = torch.Generator(device="cuda").manual_seed(1)
R = torch.randn(n, n, device="cuda", dtype=torch.float64, generator=g)
cases = {
    "dense_random": (R + R.T) / 2,
    "diag_plus_1e-6": torch.diag(torch.linspace(1, 2, n, device="cuda", dtype=torch.float64)) + 1e-6 * (R + R.T) / 2,
}
cfg = mpj.default_config("eig", variant=mpj.VARIANT_BLOCK, block_b=32)
for name, T0 in cases.items():
    for rep in range(2):
        T = T0.clone()
        V = torch.eye(n, device="cuda", dtype=torch.float64)
        torch.cuda.synchronize()
        rows, stop = [], threading.Event()
        th = threading.Thread(target=sample, args=(stop, rows), daemon=True)
        th.start()
        mpj.profile_reset()
        mpj.profile_enable(True)
        r = mpj.jacobi(T, V, tol=0.0, max_sweeps=1, cfg=cfg)
        torch.cuda.synchronize()
        mpj.profile_enable(False)
        stop.set()
        th.join(timeout=2)
        sec, cnt = mpj.profile_get("block_apply_f64")
        clk = [float(x.split(",")[0]) for x in rows if x and x.split(",")[0].strip().replace(".", "").isdigit()]
        pw = [float(x.split(",")[1]) for x in rows if x and len(x.split(",")) > 1 and x.split(",")[1].strip().replace(".", "").isdigit()]
        cap = sum(1 for x in rows if x.endswith("Active"))
        print(f"{name} rep{rep}: K4 fp64 {1e3 * sec / max(cnt, 1):.4f} ms/launch ({cnt} launches), rotations {r.rotations}, "
              f"sm MHz min/med {min(clk) if clk else None}/{statistics.median(clk) if clk else None}, "
              f"power W med/max {statistics.median(pw) if pw else None}/{max(pw) if pw else None}, "
              f"power-cap samples {cap}/{len(rows)}", flush=True)
