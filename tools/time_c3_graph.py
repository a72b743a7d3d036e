"""Times the config 3 graph build (20M-point swiss roll, k = 10, grid kNN) on the device."""
import sys
import time

sys.path.insert(0, ".")
import paper_2211_00805_b200 as gs  # noqa: E402
from paper_2211_00805_b200 import workloads  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
t0 = time.perf_counter()
roll = workloads.swiss_roll(n, 1)
t1 = time.perf_counter()
A, sigma = gs.knn_gaussian_graph(roll.points, 10)
t2 = time.perf_counter()
lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
t3 = time.perf_counter()
f = gs.HeatFilter(lap, 1.0, 30)
t4 = time.perf_counter()
print(f"n={n} points {t1-t0:.1f}s graph {t2-t1:.1f}s nnz={A.stored_entries()} laplacian+lambda {t3-t2:.1f}s "
      f"(rounds {lap.power_rounds}) filter {t4-t3:.1f}s sigma={sigma:.4g}")
