"""Times the device kNN graph build on a config-2-shaped cloud (R^30 Gaussian mixture)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2211_00805_b200 as gs  # noqa: E402
from paper_2211_00805_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
comps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mix = workloads.gaussian_mixture(n, 30, comps, 3)
t0 = time.perf_counter()
A, sigma = gs.knn_gaussian_graph(mix.points, 15)
print(f"n={n} d=30 k=15 graph {time.perf_counter() - t0:.1f}s nnz={A.stored_entries()}")
