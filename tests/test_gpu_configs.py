"""GPU parity on the BASELINE.json configurations (seeded synthetic inputs).

config 0 runs at its full size (n = 2000); configs 1 and 2 at reduced sizes the CPU oracle
finishes in seconds (same construction, same code paths); full-size config 1 is checked through
size-independent properties in bench-scale runs (mass/marginal identities below)."""
import math

import numpy as np
import pytest

import pyoracle as po
from helpers import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


def _graph_pair(gs, points, k, kernel):
    """Engine graph (device kNN) and oracle graph for the same points."""
    if kernel == 1:
        A, sigma = gs.knn_gaussian_graph(points, k)
    else:
        A, sigma = gs.knn_alpha_decay_graph(points, k, 40.0), None
    Ao, sigma_o = po.knn_graph(points, k, kernel, 40.0)
    return A, Ao, sigma, sigma_o


def test_config0_graph_lambda_and_disconnected(gs):
    """Config 0: n=2000 swiss roll, k=10 Gaussian-median graph, t=1, K=30, bumps at 2pi / 4pi
    (width 0.5), 100 sweeps. The bump centres are farther apart than K hops, so the reference
    raises Disconnected at sweep 50: the engine must raise it at the same sweep."""
    from paper_2211_00805_b200 import workloads
    roll = workloads.swiss_roll(2000, 1)
    A, Ao, sigma, sigma_o = _graph_pair(gs, roll.points, 10, 1)
    assert sigma == sigma_o
    assert np.array_equal(A.row_offsets(), Ao.offs) and np.array_equal(A.col_indices(), Ao.cols)
    assert rel(A.values(), Ao.vals) <= 1e-14
    # downstream parity on the oracle's graph is bit-exact (uploaded as a trusted CSR)
    Au = gs.SparseSymMatrix.from_csr(2000, Ao.offs, Ao.cols, Ao.vals)
    lap = gs.laplacian(Au, gs.LaplacianKind.combinatorial)
    Lo, lam_o, rounds_o = po.laplacian(Ao, 0)
    assert lap.lambda_max_bound == lam_o and lap.power_rounds == rounds_o
    f = gs.HeatFilter(lap, 1.0, 30)
    fo = po.Filter(Lo, 0, lam_o, 1.0, 30)
    mu = workloads.bump_in_s(roll, 2 * math.pi, 0.5)
    nu = workloads.bump_in_s(roll, 4 * math.pi, 0.5)
    a = np.full(2000, 1.0 / 2000)
    with pytest.raises(po.OracleError) as eo:
        po.sinkhorn_batch(fo, a, mu[None], nu[None], 100, 5e-324, single_style=True)
    with pytest.raises(gs.Error) as eg:
        gs.geodesic_sinkhorn(f, gs.Distribution(mu, validate=False), gs.Distribution(nu, validate=False),
                             a, gs.SinkhornParams(100, 5e-324))
    assert eo.value.code == "Disconnected" and eg.value.code == gs.errc.disconnected
    assert str(eg.value) == str(eo.value)


def test_config0_companion_converges(gs):
    """Well-posed companion of config 0 (nu at 2pi + 0.5): 100 sweeps, cost within 1e-9."""
    from paper_2211_00805_b200 import workloads
    roll = workloads.swiss_roll(2000, 1)
    A, Ao, _, _ = _graph_pair(gs, roll.points, 10, 1)
    for use_engine_graph in (False, True):
        G = A if use_engine_graph else gs.SparseSymMatrix.from_csr(2000, Ao.offs, Ao.cols, Ao.vals)
        lap = gs.laplacian(G, gs.LaplacianKind.combinatorial)
        f = gs.HeatFilter(lap, 1.0, 30)
        Lo, lam_o, _ = po.laplacian(Ao, 0)
        fo = po.Filter(Lo, 0, lam_o, 1.0, 30)
        mu = workloads.bump_in_s(roll, 2 * math.pi, 0.5)
        nu = workloads.bump_in_s(roll, 2 * math.pi + 0.5, 0.5)
        a = np.full(2000, 1.0 / 2000)
        res = gs.geodesic_sinkhorn(f, gs.Distribution(mu, validate=False),
                                   gs.Distribution(nu, validate=False), a, gs.SinkhornParams(100, 5e-324))
        ref = po.sinkhorn_batch(fo, a, mu[None], nu[None], 100, 5e-324, single_style=True)
        assert res.iterations == ref["iterations"][0] == 100
        assert rel(res.cost, ref["cost"][0]) <= 1e-9
        assert rel(res.kl, ref["kl"][0]) <= 1e-9
        if not use_engine_graph:
            assert np.array_equal(res.v, ref["v"][0])


def test_config1_shape_reduced(gs):
    """Config 1 construction at n = 6000, 16 pairs, 25 sweeps, stagnation abort disabled (the
    bench's documented deviation) on both sides."""
    from paper_2211_00805_b200 import workloads
    cfg = workloads.config1(6000, 16, seed=1, pair_seed=2)
    A, Ao, sigma, sigma_o = _graph_pair(gs, cfg.roll.points, 10, 1)
    Au = gs.SparseSymMatrix.from_csr(6000, Ao.offs, Ao.cols, Ao.vals)
    lap = gs.laplacian(Au, gs.LaplacianKind.combinatorial)
    f = gs.HeatFilter(lap, 1.0, 30)
    Lo, lam_o, _ = po.laplacian(Ao, 0)
    fo = po.Filter(Lo, 0, lam_o, 1.0, 30)
    a = np.full(6000, 1.0 / 6000)
    res = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m, validate=False) for m in cfg.mus],
                                     [gs.Distribution(x, validate=False) for x in cfg.nus], a,
                                     gs.SinkhornParams(25, 5e-324), no_stagnation_abort=True)
    ref = po.sinkhorn_batch(fo, a, cfg.mus, cfg.nus, 25, 5e-324, flags=1)
    for p in range(16):
        assert np.array_equal(res[p].v, ref["v"][p]) and np.array_equal(res[p].w, ref["w"][p])
        assert rel(res[p].cost, ref["cost"][p]) <= 1e-9
        assert rel(res[p].marginal_error, ref["marginal_error"][p]) <= 1e-9


def test_config2_shape_reduced(gs):
    """Config 2 construction at n = 4000 in R^30 (20-component mixture, k = 15, t = 0.5), 8
    members on random 60% subsets of 4 clusters, 30 sweeps. The graph splits into one component
    per cluster, so the barycenter is floor-dominated: parity checks that the
    1e-300 / 1e300 clamp semantics are reproduced."""
    from paper_2211_00805_b200 import workloads
    mix = workloads.gaussian_mixture(4000, 30, 20, 3)
    members = workloads.cluster_subset_members(mix, 8, 4, 0.6, 4)
    A, Ao, sigma, sigma_o = _graph_pair(gs, mix.points, 15, 1)
    assert np.array_equal(A.col_indices(), Ao.cols)
    Au = gs.SparseSymMatrix.from_csr(4000, Ao.offs, Ao.cols, Ao.vals)
    lap = gs.laplacian(Au, gs.LaplacianKind.combinatorial)
    f = gs.HeatFilter(lap, 0.5, 30)
    Lo, lam_o, _ = po.laplacian(Ao, 0)
    fo = po.Filter(Lo, 0, lam_o, 0.5, 30)
    a = np.full(4000, 1.0 / 4000)
    fam = gs.DistributionFamily([gs.Distribution(m, validate=False) for m in members])
    res = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(30, 1e-9))
    ref = po.barycenter(fo, a, members, None, 30, 1e-9)
    assert res.iterations == ref["iterations"]
    assert rel(res.barycenter.weights[ref["barycenter"] > 1e-200],
               ref["barycenter"][ref["barycenter"] > 1e-200]) <= 1e-9
    assert np.array_equal(res.barycenter.weights <= 1e-200, ref["barycenter"] <= 1e-200)
    assert rel(res.marginal_error, ref["marginal_error"]) <= 1e-9


def _mixture_filters(gs, mix, k, t):
    A, Ao, _, _ = _graph_pair(gs, mix.points, k, 1)
    n = mix.points.shape[0]
    Au = gs.SparseSymMatrix.from_csr(n, Ao.offs, Ao.cols, Ao.vals)
    lap = gs.laplacian(Au, gs.LaplacianKind.combinatorial)
    Lo, lam_o, _ = po.laplacian(Ao, 0)
    assert lap.lambda_max_bound == lam_o
    return gs.HeatFilter(lap, t, 30), po.Filter(Lo, 0, lam_o, t, 30)


def test_config2_shape_companion_shared_clusters(gs):
    """Well-posed companion of config 2 (SURVEY §7 hard part 1): R^30 mixture with overlapping
    clusters (means ~ N(0, 1), so the k = 15 graph is connected), 8 members uniform over random
    60% subsets of 4 clusters drawn from a shared pool of 6; the barycenter converges instead of
    hitting the 1e-300 floor. Every barycenter weight and V within 1e-9 of the oracle."""
    from paper_2211_00805_b200 import workloads
    mix = workloads.gaussian_mixture(4000, 30, 20, 3, mean_scale=1.0)
    members = workloads.cluster_subset_members(mix, 8, 4, 0.6, 4, cluster_pool=range(6))
    f, fo = _mixture_filters(gs, mix, 15, 0.5)
    a = np.full(4000, 1.0 / 4000)
    fam = gs.DistributionFamily([gs.Distribution(m, validate=False) for m in members])
    res = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(200, 1e-9))
    ref = po.barycenter(fo, a, members, None, 200, 1e-9)
    assert res.iterations == ref["iterations"]
    assert res.barycenter.weights.min() > 1e-200  # not floor-dominated
    assert rel(res.barycenter.weights, ref["barycenter"]) <= 1e-9
    # the converged marginal error (~1e-9) is a difference of O(1) quantities: absolute bound
    assert abs(res.marginal_error - ref["marginal_error"]) <= 1e-12


def test_config4_shape_barycentric_distance(gs):
    """Config-4 shape at reduced size (R^30, 40 overlapping clusters, k = 15, t = 0.5): two
    6-member groups as specified (group B with 20% of its mass shifted onto clusters 20-39), both
    barycenters and the geodesic Sinkhorn distance between them (barycenter.cpp:101-107) within
    1e-9 of the oracle."""
    from paper_2211_00805_b200 import workloads
    n, m = 3000, 6
    mix = workloads.gaussian_mixture(n, 30, 40, 5, mean_scale=1.0)
    cfg = workloads.config4_from_mixture(mix, m, member_seed=6)
    f, fo = _mixture_filters(gs, mix, 15, 0.5)
    a = np.full(n, 1.0 / n)
    params = gs.SinkhornParams(200, 1e-9)
    fa = gs.DistributionFamily([gs.Distribution(x, validate=False) for x in cfg.group_a])
    fb = gs.DistributionFamily([gs.Distribution(x, validate=False) for x in cfg.group_b])
    ba = gs.sinkhorn_barycenter(f, fa, a, params)
    bb = gs.sinkhorn_barycenter(f, fb, a, params)
    d = gs.barycentric_distance(f, fa, fb, a, params)
    ra = po.barycenter(fo, a, cfg.group_a, None, 200, 1e-9)
    rb = po.barycenter(fo, a, cfg.group_b, None, 200, 1e-9)
    assert rel(ba.barycenter.weights, ra["barycenter"]) <= 1e-9
    assert rel(bb.barycenter.weights, rb["barycenter"]) <= 1e-9
    rd = po.sinkhorn_batch(fo, a, ra["barycenter"][None], rb["barycenter"][None], 200, 1e-9,
                           single_style=True)
    assert np.isfinite(d) and d > 0
    assert rel(d, rd["cost"][0]) <= 1e-9
