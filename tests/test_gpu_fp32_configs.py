"""GPU: the optional 32-bit mode on the BASELINE swiss-roll constructions (configs 0, 1, 3) against
the fp64 oracle. north_star: distances within 1e-4 relative in fp32.

The 32-bit mode stores every Chebyshev-vector word as the upper half of the fp64 word (sign, the
11-bit fp64 exponent, 20 fraction bits) and computes in fp64 (DESIGN.md §4 "Precision"): binary32's
exponent cannot hold the scaling vectors of long-range transport (profiles/r02_fp32_range.md).
Where the reference's result is not finite (or the stagnation rule fires) the 32-bit mode must
report the same errc, never a non-finite value."""
import math

import numpy as np
import pytest

import pyoracle as po
from part_comm import ThreadGroup

pytestmark = pytest.mark.gpu
TOL32 = 1e-4


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


def _filters(gs, points, k=10, t=1.0):
    """Engine filter on the oracle's graph (uploaded as a trusted CSR) and the oracle filter."""
    Ao, _ = po.knn_graph(points, k, 1, 0.0)
    Au = gs.SparseSymMatrix.from_csr(Ao.n, Ao.offs, Ao.cols, Ao.vals)
    lap = gs.laplacian(Au, gs.LaplacianKind.combinatorial)
    Lo, lam_o, _ = po.laplacian(Ao, 0)
    assert lap.lambda_max_bound == lam_o
    return gs.HeatFilter(lap, t, 30), po.Filter(Lo, 0, lam_o, t, 30)


def _dists(gs, X):
    return [gs.Distribution(x, validate=False) for x in X]


def test_config0_companion_fp32(gs):
    """Config 0 (n = 2000) with nu at 2pi + 0.5: 100 fp32 sweeps vs the fp64 oracle."""
    from paper_2211_00805_b200 import workloads
    roll = workloads.swiss_roll(2000, 1)
    f, fo = _filters(gs, roll.points)
    mu = workloads.bump_in_s(roll, 2 * math.pi, 0.5)
    nu = workloads.bump_in_s(roll, 2 * math.pi + 0.5, 0.5)
    a = np.full(2000, 1.0 / 2000)
    ref = po.sinkhorn_batch(fo, a, mu[None], nu[None], 100, 5e-324, single_style=True)
    res = gs.geodesic_sinkhorn(f, gs.Distribution(mu, validate=False), gs.Distribution(nu, validate=False),
                               a, gs.SinkhornParams(100, 5e-324), fp32=True)
    assert res.iterations == 100
    assert abs(res.cost - ref["cost"][0]) <= TOL32 * abs(ref["cost"][0])


@pytest.mark.parametrize("n,pairs", [(6000, 16), (20000, 8)])
def test_config1_companions_fp32(gs, n, pairs):
    """Config 1 construction with well-posed companion pairs (workloads.bump_mixture_companions:
    every target bump a geodesic offset <= 0.5 from its source bump), 200 sweeps: every fp32
    cost finite and within 1e-4 of the fp64 oracle's."""
    from paper_2211_00805_b200 import workloads
    roll = workloads.swiss_roll(n, 1)
    mus, nus = workloads.bump_mixture_companions(roll, pairs, 2)
    f, fo = _filters(gs, roll.points)
    a = np.full(n, 1.0 / n)
    ref = po.sinkhorn_batch(fo, a, mus, nus, 200, 5e-324)
    res = gs.geodesic_sinkhorn_batch(f, _dists(gs, mus), _dists(gs, nus), a,
                                     gs.SinkhornParams(200, 5e-324), fp32=True)
    cost = np.array([r.cost for r in res])
    assert np.all(np.isfinite(cost))
    assert np.max(np.abs(cost - ref["cost"]) / np.abs(ref["cost"])) <= TOL32
    assert all(r.iterations == 200 for r in res)
    err = np.array([r.marginal_error for r in res])
    assert np.max(np.abs(err - ref["marginal_error"])) <= 1e-3 * np.max(ref["marginal_error"]) + 1e-9


def test_config1_as_specified_fp32_error_semantics(gs):
    """Config 1 as specified (random 3-bump mixtures, most pairs beyond the K-hop reach) with the
    stagnation abort on: the fp64 reference raises Disconnected for the first stagnating pair;
    the fp32 mode raises the same errc for the same pair at the same sweep."""
    from paper_2211_00805_b200 import workloads
    cfg = workloads.config1(6000, 16, seed=1, pair_seed=2)
    f, fo = _filters(gs, cfg.roll.points)
    a = np.full(6000, 1.0 / 6000)
    with pytest.raises(po.OracleError) as eo:
        po.sinkhorn_batch(fo, a, cfg.mus, cfg.nus, 100, 5e-324)
    with pytest.raises(gs.Error) as eg:
        gs.geodesic_sinkhorn_batch(f, _dists(gs, cfg.mus), _dists(gs, cfg.nus), a,
                                   gs.SinkhornParams(100, 5e-324), fp32=True)
    assert eo.value.code == "Disconnected" and eg.value.code == gs.errc.disconnected
    assert str(eg.value) == str(eo.value)  # same pair index in the message


def test_config1_as_specified_fp32_never_nonfinite(gs):
    """With the abort disabled (the bench's deviation) the fp64 reference returns -inf costs for
    pairs whose v underflows; the fp32 mode must not return a non-finite value: it either
    matches a finite fp64 cost within 1e-4 or raises numerical_underflow."""
    from paper_2211_00805_b200 import workloads
    cfg = workloads.config1(6000, 8, seed=1, pair_seed=2)
    f, fo = _filters(gs, cfg.roll.points)
    a = np.full(6000, 1.0 / 6000)
    try:
        res = gs.geodesic_sinkhorn_batch(f, _dists(gs, cfg.mus), _dists(gs, cfg.nus), a,
                                         gs.SinkhornParams(60, 5e-324), no_stagnation_abort=True,
                                         fp32=True)
    except gs.Error as e:
        assert e.code == gs.errc.numerical_underflow
        return
    assert all(np.isfinite(r.cost) and np.isfinite(r.marginal_error) for r in res)


@pytest.mark.parametrize("nparts", [1, 2, 4])
def test_config3_shape_fp32_row_partitioned(gs, nparts):
    """Config 3 construction at reduced n (swiss roll, k = 10, t = 1, K = 30, fp32, one pair:
    config 0's bump at 2pi against its companion at 2pi + 0.5, 100 sweeps), rows partitioned
    over 1/2/4 parts (threads with an in-process comm, one GPU): the stitched v, w equal the
    unpartitioned fp32 run bit for bit, and the cost is within 1e-4 of the fp64 oracle."""
    from paper_2211_00805_b200 import workloads
    n = 20000
    roll = workloads.swiss_roll(n, 1)
    f, fo = _filters(gs, roll.points)
    mu = workloads.bump_in_s(roll, 2 * math.pi, 0.5)
    nu = workloads.bump_in_s(roll, 2 * math.pi + 0.5, 0.5)
    a = np.full(n, 1.0 / n)
    params = gs.SinkhornParams(100, 5e-324)
    full = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(mu, validate=False)],
                                      [gs.Distribution(nu, validate=False)], a, params, fp32=True)[0]
    ref = po.sinkhorn_batch(fo, a, mu[None], nu[None], 100, 5e-324)
    assert abs(full.cost - ref["cost"][0]) <= TOL32 * abs(ref["cost"][0])
    parts = [None] * nparts

    def body(r, comm):
        ctx = gs.Context(0)
        part = gs.RowPartition(f, nparts, r, ctx=ctx)
        parts[r] = part
        vid = part.vertices
        return part.sinkhorn([mu[vid]], [nu[vid]], a[vid], params,
                             comm=comm.comm if nparts > 1 else None, fp32=True)[0]

    res = ThreadGroup(nparts).run(body)
    v = np.zeros(n)
    w = np.zeros(n)
    for p, q in zip(parts, res):
        v[p.vertices] = q.v
        w[p.vertices] = q.w
    assert np.array_equal(v, full.v) and np.array_equal(w, full.w)
    assert abs(res[0].cost - full.cost) <= 1e-12 * abs(full.cost)


def test_config1_companions_fp32_windowed_64_columns(gs, monkeypatch):
    """64 companion pairs in the 32-bit mode: 256-byte rows run the windowed kernel
    (k_cheb_win<float, 64>); every cost within 1e-4 of the fp64 oracle, and v / w bit-identical
    to the register-gather kernel (GS_WIN=0: same storage words, same fp64 chains; the cost sums
    run over the two layouts' vertex orders, so they agree to rounding)."""
    from paper_2211_00805_b200 import workloads
    n, pairs = 6000, 64
    roll = workloads.swiss_roll(n, 1)
    mus, nus = workloads.bump_mixture_companions(roll, pairs, 3)
    f, fo = _filters(gs, roll.points)
    a = np.full(n, 1.0 / n)
    params = gs.SinkhornParams(100, 5e-324)
    res = gs.geodesic_sinkhorn_batch(f, _dists(gs, mus), _dists(gs, nus), a, params, fp32=True)
    ref = po.sinkhorn_batch(fo, a, mus, nus, 100, 5e-324)
    cost = np.array([r.cost for r in res])
    assert np.all(np.isfinite(cost))
    assert np.max(np.abs(cost - ref["cost"]) / np.abs(ref["cost"])) <= TOL32
    monkeypatch.setenv("GS_WIN", "0")
    reg = gs.geodesic_sinkhorn_batch(f, _dists(gs, mus), _dists(gs, nus), a, params, fp32=True)
    for p in range(pairs):
        assert np.array_equal(res[p].v, reg[p].v) and np.array_equal(res[p].w, reg[p].w)
        assert abs(res[p].cost - reg[p].cost) <= 1e-14 * abs(reg[p].cost)
