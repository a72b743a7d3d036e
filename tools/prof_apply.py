"""Profiling driver: one filter apply on a BASELINE-shaped operator (for ncu captures of the step
kernel). Usage: python tools/prof_apply.py [config] [applies]; config 1 = swiss roll n=2e5, 64
columns; config 2 = R^30 mixture n=1e6, 8 columns; config 4s / 4 = R^30 mixture n=1e6 / 4e6, 16 columns;
config 3 / 3s = swiss roll n=2e7 / 2e6, one column, 32-bit mode."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2211_00805_b200 as gs  # noqa: E402
from paper_2211_00805_b200 import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = gs.Context.default(0)
if cfg == "1":
    roll = workloads.swiss_roll(200_000, 1)
    pts, k, t, B = roll.points, 10, 1.0, 64
elif cfg in ("2", "4s", "4"):
    mix = workloads.gaussian_mixture(4_000_000 if cfg == "4" else 1_000_000, 30, 20 if cfg == "2" else 40, 3)
    pts, k, t, B = mix.points, 15, 0.5, 8 if cfg == "2" else 16
elif cfg in ("3", "3s"):
    roll = workloads.swiss_roll(20_000_000 if cfg == "3" else 2_000_000, 1)
    pts, k, t, B = roll.points, 10, 1.0, 1
else:
    raise SystemExit("config")
fp32 = cfg in ("3", "3s")
t0 = time.time()
A, _ = gs.knn_gaussian_graph(pts, k, ctx=ctx)
lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
f = gs.HeatFilter(lap, t, 30)
n = pts.shape[0]
X = np.abs(np.sin(np.arange(n)[:, None] * (np.arange(B)[None, :] + 1.0))) + 0.1
if B == 1:
    X = X[:, 0]
print("setup", time.time() - t0, flush=True)
Y = f.apply(X, fp32=fp32)  # warm-up (builds the layout / schedule)
ctx.set_timing(True)
for _ in range(reps):
    Y = f.apply(X, fp32=fp32)
nst, ms = ctx.timing(0)
ctx.set_timing(False)
print(f"apply done: {nst} step launches, avg step {1e3 * ms / max(nst, 1):.1f} us", float(np.abs(Y).sum()))
