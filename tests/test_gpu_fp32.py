"""GPU: the optional fp32 mode against the fp64 oracle (north_star: 1e-4 relative; DESIGN.md
lists the fp32 constants: floor FLT_MIN, positivity slack 64 FLT_EPSILON)."""
import numpy as np
import pytest

import pyoracle as po
from helpers import (acceptance_graph, engine_filter, oracle_filter, random_connected_graph,
                     random_distribution)

pytestmark = pytest.mark.gpu
TOL32 = 1e-4


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


@pytest.mark.parametrize("width", [1, 3, 8, 64])
def test_filter_apply_fp32(gs, width):
    n = 300
    r, c, v = acceptance_graph(n, 1300)
    f, _ = engine_filter(r, c, v, n, 0, 1.0, 30)
    fo = oracle_filter(r, c, v, n, 0, 1.0, 30)
    X = np.abs(np.random.default_rng(width).standard_normal((n, width)))
    ref = fo.apply(X)
    out = f.apply(X, fp32=True)
    assert np.max(np.abs(out - ref)) <= TOL32 * np.max(np.abs(ref))


def test_sinkhorn_fp32(gs):
    n = 200
    r, c, v = random_connected_graph(n, 21)
    f, _ = engine_filter(r, c, v, n, 1, 0.9, 30)
    fo = oracle_filter(r, c, v, n, 1, 0.9, 30)
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(7)
    mus = [random_distribution(n, rng) for _ in range(8)]
    nus = [random_distribution(n, rng) for _ in range(8)]
    a = np.full(n, 1.0 / n)
    res = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m) for m in mus],
                                     [gs.Distribution(x) for x in nus], a,
                                     gs.SinkhornParams(60, 5e-324), no_stagnation_abort=True,
                                     fp32=True)
    ref = po.sinkhorn_batch(fo, a, np.array(mus), np.array(nus), 60, 5e-324, flags=1)
    for p in range(8):
        assert abs(res[p].cost - ref["cost"][p]) <= TOL32 * abs(ref["cost"][p])


def test_barycenter_fp32(gs):
    n = 120
    r, c, v = random_connected_graph(n, 12)
    f, _ = engine_filter(r, c, v, n, 1, 0.8, 30)
    fo = oracle_filter(r, c, v, n, 1, 0.8, 30)
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(9)
    members = [random_distribution(n, rng) for _ in range(4)]
    a = np.full(n, 1.0 / n)
    fam = gs.DistributionFamily([gs.Distribution(x) for x in members])
    res = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(40, 5e-324), fp32=True)
    ref = po.barycenter(fo, a, np.array(members), None, 40, 5e-324)
    b = res.barycenter.weights
    assert np.max(np.abs(b - ref["barycenter"]) / ref["barycenter"]) <= TOL32
