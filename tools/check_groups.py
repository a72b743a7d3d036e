import sys; sys.path.insert(0,'.'); sys.path.insert(0,'./oracle'); sys.path.insert(0,'./tests')
import numpy as np, pyoracle as po
import paper_2211_00805_b200 as gs
from helpers import acceptance_graph, engine_filter, oracle_filter, random_distribution
from paper_2211_00805_b200.rng import Rng
n = 150
r, c, v = acceptance_graph(n, 1001)
f, _ = engine_filter(r, c, v, n, 1, 1.0, 30)
fo = oracle_filter(r, c, v, n, 1, 1.0, 30)
for P in (65, 70, 105, 130):
    rng = Rng(P)
    mus = [random_distribution(n, rng) for _ in range(P)]
    nus = [random_distribution(n, rng) for _ in range(P)]
    a = np.full(n, 1.0 / n)
    try:
        res = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m) for m in mus], [gs.Distribution(x) for x in nus], a, gs.SinkhornParams(300, 1e-9))
        e = None
    except gs.Error as ex:
        res, e = None, str(ex)
    try:
        ref = po.sinkhorn_batch(fo, a, np.array(mus), np.array(nus), 300, 1e-9); re_ = None
    except po.OracleError as ex:
        ref, re_ = None, str(ex)
    if e or re_:
        print(P, "engine:", e, "oracle:", re_); continue
    bad = [p for p in range(P) if not (np.array_equal(res[p].v, ref["v"][p]) and res[p].iterations == ref["iterations"][p])]
    print(P, "mismatched pairs:", bad[:10], len(bad), "iters", [res[p].iterations for p in bad[:3]], [int(ref["iterations"][p]) for p in bad[:3]])
