"""Per-CTA timeline of the last fp64 apply (K4) launch, from a diagnostics
build (MPJ_NVCC_EXTRA=-DMPJ_K4_TRACE): n = 8192, a few block rounds of the
first sweep (every item computed).  Prints the launch span, the spread of
CTA start / end times and the mean fraction of the span the CTA slots are
occupied (ncu's achieved-occupancy question: tail or ramp?)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import runpy

os.environ.setdefault("BROUNDS", "3")
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe_k4.py"))
import paper_2211_03339_b200 as mpj  # noqa: E402

buf = np.zeros(1024 * 3, dtype=np.uint64)
assert mpj.lib().mpjacobi_debug_k4_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong))) == 0
t = buf.reshape(1024, 3)
G = int((t[:, 0] > 0).sum())
t = t[:G].astype(np.float64)
t0 = t[:, 0].min()
st, en, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, t[:, 2].astype(int)
span = en.max()
print(f"CTAs {G}, span {span:.1f} us")
print(f"start: min {st.min():.1f} median {np.median(st):.1f} max {st.max():.1f} us")
print(f"end:   min {en.min():.1f} p10 {np.percentile(en, 10):.1f} median {np.median(en):.1f} p90 {np.percentile(en, 90):.1f} max {en.max():.1f} us")
print(f"CTA slot occupancy over the span: {((en - st).sum() / (G * span)):.3f}")
per_sm = {}
for i in range(G):
    per_sm.setdefault(sm[i], []).append((st[i], en[i], i))
spread = [max(e for _, e, _ in v) - min(e for _, e, _ in v) for v in per_sm.values()]
print(f"SMs {len(per_sm)}, CTAs per SM {sorted(set(len(v) for v in per_sm.values()))}, "
      f"end spread within an SM: median {np.median(spread):.1f} max {max(spread):.1f} us")
order = np.argsort(en)
print("earliest finishers (cta, sm, start, end):", [(int(i), int(sm[i]), round(st[i], 1), round(en[i], 1)) for i in order[:6]])
print("latest finishers:", [(int(i), int(sm[i]), round(st[i], 1), round(en[i], 1)) for i in order[-6:]])
