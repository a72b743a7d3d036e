"""Stage-by-stage engine vs oracle comparison on the kNN benchmark's default inputs."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np, pyoracle as po
import paper_2211_00805_b200 as gs
from paper_2211_00805_b200 import knn_bench as kb
s = kb.make_swiss_roll(15, 1000, 3.0, 10, 1)
nb, eps = gs.select_knn(s.ambient, 5)
nbo = np.empty_like(nb); epso = np.empty_like(eps)
nbo, epso = po.knn(s.ambient, 5)
print("knn equal", np.array_equal(nb, nbo), "eps equal", np.array_equal(eps, epso),
      "rows differing", int((nb != nbo).any(1).sum()))
A = gs.knn_alpha_decay_graph(s.ambient, 5, 40.0)
Ao = po.knn_graph(s.ambient, 5, 0, 40.0)[0]
print("graph equal", np.array_equal(A.row_offsets(), Ao.offs) and np.array_equal(A.col_indices(), Ao.cols),
      "vals equal", np.array_equal(A.values(), Ao.vals) if A.stored_entries() == Ao.nnz else None)
lap = gs.laplacian(A, gs.LaplacianKind.normalized)
Lo, lam, rounds = po.laplacian(Ao, 1)
print("lambda", lap.lambda_max_bound, lam, "rounds", lap.power_rounds, rounds)
f = gs.HeatFilter(lap, 20.0, 100)
fo = po.Filter(Lo, 1, lam, 20.0, 100)
print("coeffs equal", np.array_equal(f.coefficients(), fo.coeffs), "t_eff", f.effective_time(), fo.t_eff)
x = np.random.default_rng(0).standard_normal((15000, 3))
print("apply equal", np.array_equal(f.apply(x), fo.apply(x)))
