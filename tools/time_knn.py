"""Times the device kNN graph build on a config-2/4-shaped cloud (R^30 Gaussian mixture).
Usage: python tools/time_knn.py n comps [mode ...]   (mode: tc | brute; GS_KNN)"""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_2211_00805_b200 as gs  # noqa: E402
from paper_2211_00805_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
comps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
modes = sys.argv[3:] or ["tc"]
mix = workloads.gaussian_mixture(n, 30, comps, 3)
ctx = gs.Context.default(0)
for mode in modes:
    os.environ["GS_KNN"] = mode
    t0 = time.perf_counter()
    A, sigma = gs.knn_gaussian_graph(mix.points, 15)
    dt = time.perf_counter() - t0
    print(f"n={n} d=30 k=15 comps={comps} GS_KNN={mode}: graph {dt:.2f}s nnz={A.stored_entries()} "
          f"sigma={sigma!r} fallback_queries={ctx.lib.gs_ctx_knn_fallback(ctx.handle)}", flush=True)
