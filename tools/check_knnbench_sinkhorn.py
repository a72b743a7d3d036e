"""Engine Sinkhorn on the oracle's exact graph vs the oracle (kNN benchmark default inputs)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np, pyoracle as po
import paper_2211_00805_b200 as gs
from paper_2211_00805_b200 import knn_bench as kb
s = kb.make_swiss_roll(15, 1000, 3.0, 10, 1)
A = gs.knn_alpha_decay_graph(s.ambient, 5, 40.0)
Ao = po.knn_graph(s.ambient, 5, 0, 40.0)[0]
rd = np.abs(A.values() - Ao.vals) / np.abs(Ao.vals)
print("alpha-decay weights: max rel diff", rd.max(), "entries differing", int((rd > 0).sum()), "of", rd.size)
Ae = gs.SparseSymMatrix.from_csr(Ao.n, Ao.offs, Ao.cols, Ao.vals)  # the oracle's graph on the device
lap = gs.laplacian(Ae, gs.LaplacianKind.normalized)
Lo, lam, _ = po.laplacian(Ao, 1)
f = gs.HeatFilter(lap, 20.0, 100)
fo = po.Filter(Lo, 1, lam, 20.0, 100)
x = np.random.default_rng(0).standard_normal((15000, 3))
print("apply on the oracle graph equal", np.array_equal(f.apply(x), fo.apply(x)))
n = Ao.n
groups = [np.flatnonzero(s.labels == c) for c in range(15)]
mus, nus = [], []
for i in range(15):
    for j in range(i + 1, 15):
        mus.append(gs.Distribution.indicator(n, groups[i])); nus.append(gs.Distribution.indicator(n, groups[j]))
a = np.full(n, 1.0 / n)
try:
    res = gs.geodesic_sinkhorn_batch(f, mus, nus, a, gs.SinkhornParams(500, 1e-6))
    print("engine on oracle graph: converged", [r.iterations for r in res][:12])
except gs.Error as e:
    print("engine on oracle graph:", e)
