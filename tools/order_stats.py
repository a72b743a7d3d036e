"""Tuning tool: bandwidth profile of the filter's locality order on the config-1 graph."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2211_00805_b200 as gs
from paper_2211_00805_b200 import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
cfg = workloads.config1(n, 2)
A, sigma = gs.knn_gaussian_graph(cfg.roll.points, 10)
lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
f = gs.HeatFilter(lap, 1.0, 30)
order = f.vertex_order()
newpos = np.empty(n, np.int64); newpos[order] = np.arange(n)
S = lap.matrix
offs, cols = S.row_offsets(), S.col_indices()
rows = np.repeat(np.arange(n), np.diff(offs))
d = np.abs(newpos[rows] - newpos[cols])
print("n", n, "nnz", cols.size, "bandwidth max", d.max(), "p99", np.percentile(d, 99), "p90", np.percentile(d, 90), "mean", d.mean())
for R in (32, 64, 128, 256, 512):
    pr = newpos[rows] // R
    key = pr * n + newpos[cols]
    u = np.unique(key)
    cnt = np.bincount(u // n)
    span = []
    print(f"R={R}: unique neighbour rows per block mean {cnt.mean():.1f} (x{cnt.mean()/R:.2f}), max {cnt.max()}")
