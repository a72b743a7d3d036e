"""Profiling driver: config 0 (n = 2000 swiss roll, one pair, 100 sweeps) through gs_sinkhorn."""
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2211_00805_b200 as gs  # noqa: E402
from paper_2211_00805_b200 import workloads  # noqa: E402

ctx = gs.Context.default(0)
roll = workloads.swiss_roll(2000, 1)
A, _ = gs.knn_gaussian_graph(roll.points, 10, ctx=ctx)
f = gs.HeatFilter(gs.laplacian(A, gs.LaplacianKind.combinatorial), 1.0, 30)
mu = gs.Distribution(workloads.bump_in_s(roll, 2 * math.pi, 0.5), validate=False)
nu = gs.Distribution(workloads.bump_in_s(roll, 2 * math.pi + 0.5, 0.5), validate=False)
a = np.full(2000, 1.0 / 2000)
p = gs.SinkhornParams(100, 5e-324)
gs.geodesic_sinkhorn(f, mu, nu, a, p)
ctx.set_timing(True)
t0 = time.perf_counter()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for _ in range(reps):
    r = gs.geodesic_sinkhorn(f, mu, nu, a, p)
dt = time.perf_counter() - t0
n0, ms0 = ctx.timing(0)
n1, ms1 = ctx.timing(1)
print(f"{reps} runs: {1e3 * dt / reps:.2f} ms/run wall, class0 {n0} launches {ms0 / reps:.3f} ms/run, "
      f"class1 {n1} launches {ms1 / reps:.3f} ms/run, cost {r.cost}")
