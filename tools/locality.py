"""Mean / median |newpos(i) - newpos(j)| over CSR entries in the filter's Cuthill-McKee order."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2211_00805_b200 as gs  # noqa: E402
from paper_2211_00805_b200 import workloads  # noqa: E402


def stat(name, A):
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    f = gs.HeatFilter(lap, 1.0, 30)
    L = f.scaled_laplacian()
    offs, cols = L.row_offsets(), L.col_indices()
    order = f.vertex_order()
    n = order.size
    newpos = np.empty(n, np.int64)
    newpos[order] = np.arange(n)
    rows = np.repeat(np.arange(n), np.diff(offs))
    span = np.abs(newpos[rows] - newpos[cols])
    print(f"{name}: n={n} nnz={cols.size} mean span {span.mean():.0f} median {np.median(span):.0f} "
          f"p90 {np.percentile(span, 90):.0f} frac<=256 {(span <= 256).mean():.3f}")


stat("swiss200k", gs.knn_gaussian_graph(workloads.swiss_roll(200_000, 1).points, 10)[0])
stat("swiss2M", gs.knn_gaussian_graph(workloads.swiss_roll(2_000_000, 1).points, 10)[0])
stat("mix20_400k", gs.knn_gaussian_graph(workloads.gaussian_mixture(400_000, 30, 20, 3).points, 15)[0])
stat("mix40_400k", gs.knn_gaussian_graph(workloads.gaussian_mixture(400_000, 30, 40, 5).points, 15)[0])
