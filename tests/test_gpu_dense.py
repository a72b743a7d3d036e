"""Dense entropic Sinkhorn on the device (gs_dense.cu; transport.cpp:271-311) and the kNN
benchmark's dense baselines (bench.cpp:311-331) against the oracle restatement
(go_dense_sinkhorn / go_squared_distances), plus the reference's own dense-Sinkhorn tests
(test_transport.cpp:77-96, 208-215; test_bench.cpp:160-192). Products and sums follow the
oracle's order bit for bit; exp / log are libdevice vs glibc, so results are held to 1e-9."""
import numpy as np
import pytest

import pyoracle as po
from helpers import random_connected_graph, random_distribution

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


@pytest.mark.parametrize("r,c,lam,seed", [(3, 3, 0.7, 1), (37, 53, 0.5, 2), (200, 150, 2.0, 3)])
def test_dense_sinkhorn_matches_oracle(gs, r, c, lam, seed):
    from paper_2211_00805_b200.rng import Rng
    g = np.random.default_rng(seed)
    X, Y = g.standard_normal((r, 4)), g.standard_normal((c, 4))
    cost = po.squared_distances(X, Y)
    mu, nu = random_distribution(r, Rng(seed)), random_distribution(c, Rng(seed + 100))
    res = gs.dense_sinkhorn(cost, gs.Distribution(mu), gs.Distribution(nu), lam, gs.SinkhornParams(400, 1e-10))
    ref = po.dense_sinkhorn(cost, mu, nu, lam, 400, 1e-10)
    assert res.iterations == ref["iterations"] and res.converged == ref["converged"]
    assert rel(res.cost, ref["cost"]) <= TOL and rel(res.kl, ref["kl"]) <= TOL
    assert rel(res.v, ref["v"]) <= TOL and rel(res.w, ref["w"]) <= TOL
    assert abs(res.marginal_error - ref["marginal_error"]) <= 1e-12


def test_dense_zero_cost_gives_product_plan(gs):
    """test_transport.cpp:208-215."""
    mu, nu = np.array([0.5, 0.3, 0.2]), np.array([0.2, 0.2, 0.6])
    res = gs.dense_sinkhorn(np.zeros((3, 3)), gs.Distribution(mu), gs.Distribution(nu), 0.7,
                            gs.SinkhornParams(500, 1e-12))
    assert res.converged
    plan = res.v[:, None] * np.ones((3, 3)) * res.w[None, :]
    assert np.abs(plan - np.outer(mu, nu)).max() <= 1e-10


def test_dense_matches_geodesic_proposition_1(gs):
    """test_transport.cpp:77-96: geodesic Sinkhorn cost == dense Sinkhorn dual cost on
    -4t log(exact heat kernel), within 1e-6."""
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(42)
    for seed in (11, 12):
        n = 40 + (seed % 3) * 25
        r, c, v = random_connected_graph(n, seed)
        A = gs.SparseSymMatrix.from_arrays(n, r, c, v)
        lap = gs.laplacian(A, gs.LaplacianKind.normalized)
        t = 0.5 + 0.25 * (seed % 4)
        f = gs.HeatFilter(lap, t, 50)
        mu, nu = random_distribution(n, rng), random_distribution(n, rng)
        geo = gs.geodesic_sinkhorn(f, gs.Distribution(mu), gs.Distribution(nu), np.ones(n),
                                   gs.SinkhornParams(3000, 1e-10))
        Ld = lap.matrix.to_dense()
        lam_, U = np.linalg.eigh(Ld)
        H = (U * np.exp(-t * lam_)) @ U.T
        cost = -4.0 * t * np.log(H)
        dense = gs.dense_sinkhorn(cost, gs.Distribution(mu), gs.Distribution(nu), 4.0 * t,
                                  gs.SinkhornParams(3000, 1e-10))
        assert geo.converged and dense.converged
        assert abs(geo.cost - dense.dual_cost()) <= 1e-6 * abs(geo.cost)


def test_dense_validation(gs):
    mu = gs.Distribution(np.array([0.5, 0.5]))
    with pytest.raises(gs.Error) as e:
        gs.dense_sinkhorn(np.array([[0.0, np.inf], [1.0, 0.0]]), mu, mu, 1.0)
    assert e.value.code == gs.errc.invalid_argument
    with pytest.raises(gs.Error) as e:
        gs.dense_sinkhorn(np.zeros((2, 2)), mu, mu, 0.0)
    assert e.value.code == gs.errc.invalid_argument
    with pytest.raises(gs.Error) as e:
        gs.dense_sinkhorn(np.zeros((2, 3)), mu, mu, 1.0)
    assert e.value.code == gs.errc.length_mismatch
    with pytest.raises(gs.Error) as e:  # exp(-1e8) underflows: every kernel entry is zero
        gs.dense_sinkhorn(np.full((2, 2), 1e5), mu, mu, 1e-3)
    assert e.value.code == gs.errc.numerical_underflow
    assert "row underflowed" in str(e.value)


@pytest.mark.parametrize("squared,lam", [(False, 2.0), (True, 20.0)])
def test_dense_groups_match_oracle(gs, squared, lam):
    """bench.cpp:311-331: every cluster pair of a benchmark sample, one device call, against the
    oracle's per-pair squared_distances + dense_sinkhorn."""
    from paper_2211_00805_b200 import knn_bench as kb
    sample = kb.make_swiss_roll(5, 90, 3.0, 10, 4)
    groups = [np.flatnonzero(sample.labels == c) for c in range(5)]
    pairs = [(i, j) for i in range(5) for j in range(i + 1, 5)]
    prm = gs.SinkhornParams(500, 1e-6)
    runs = gs.dense_sinkhorn_groups(sample.ambient, groups, pairs, squared, lam, prm)
    for (i, j), run in zip(pairs, runs):
        C = po.squared_distances(sample.ambient[groups[i]], sample.ambient[groups[j]])
        if not squared:
            C = np.sqrt(C)
        ref = po.dense_sinkhorn(C, np.full(len(groups[i]), 1.0 / len(groups[i])),
                                np.full(len(groups[j]), 1.0 / len(groups[j])), lam, 500, 1e-6)
        assert run.iterations == ref["iterations"] and run.converged == ref["converged"]
        assert rel(run.cost, ref["cost"]) <= TOL and rel(run.kl, ref["kl"]) <= TOL


def test_knn_benchmark_dense_rows(gs):
    """test_bench.cpp:160-192: every method's distance matrix is symmetric with a zero diagonal
    and finite; metrics in range."""
    from paper_2211_00805_b200 import knn_bench as kb
    cfg = kb.KnnBenchConfig(n_distributions=8, samples_per_dist=60, noise_sigma=4.0, ambient_dim=3,
                            seeds=[5], k=5, t=10.0, degree=64, euler_steps=10,
                            sinkhorn=gs.SinkhornParams(400, 1e-6),
                            methods=["geodesic_sinkhorn", "dense_sinkhorn_w1", "dense_sinkhorn_w2"],
                            no_stagnation_abort=True)
    res = kb.knn_benchmark(cfg)
    for name, d in res["per_seed"][0]["distances"].items():
        assert d.shape == (8, 8)
        assert np.abs(d - d.T).max() <= 1e-12 and np.abs(np.diag(d)).max() == 0.0
        assert np.isfinite(d).all()
    for name, rep in res["mean_report"].items():
        assert rep["total"] >= rep["distance"] and abs(rep["spearman"]) <= 1.0
        assert 0.0 <= rep["p_at_5"] <= 1.0
