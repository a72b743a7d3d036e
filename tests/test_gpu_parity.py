"""GPU parity: the CUDA engine (through its C ABI) against the CPU oracle on the same seeded
inputs. Integer/index work and every + - * / sqrt fma path must be bit-exact; paths through
log/exp/pow (libdevice vs glibc) are held to the north-star tolerance, 1e-9 relative in fp64."""
import numpy as np
import pytest

import pyoracle as po
from helpers import (acceptance_graph, engine_filter, oracle_filter, path_graph,
                     random_connected_graph, random_distribution, random_signal, rel)

pytestmark = pytest.mark.gpu

TOL = 1e-9  # north_star: distances and barycenters within 1e-9 relative in fp64


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


# --------------------------------------------------------------------------- coefficients
@pytest.mark.parametrize("t,deg", [(0.5, 30), (1.0, 30), (5.0, 50), (20.0, 110), (7.95, 30),
                                   (15.33, 30), (50.3, 30), (1e-12, 10), (0.0, 5)])
def test_coefficients_bit_exact(gs, t, deg):
    dev = gs.heat_chebyshev_coefficients(t, deg)
    ref = po.heat_coefficients(t, deg)
    assert np.array_equal(dev, ref)


def test_coefficient_validation(gs):
    with pytest.raises(gs.Error) as e:
        gs.heat_chebyshev_coefficients(1.0, 0)
    assert e.value.code == gs.errc.invalid_argument
    with pytest.raises(gs.Error) as e:
        gs.heat_chebyshev_coefficients(-1.0, 5)
    assert e.value.code == gs.errc.non_positive_time


# --------------------------------------------------------------------------- sparse / laplacian
@pytest.mark.parametrize("n,seed", [(3, 1), (50, 3), (200, 7), (1000, 11)])
def test_from_triplets_and_laplacian_bit_exact(gs, n, seed):
    r, c, v = random_connected_graph(n, seed)
    A = gs.SparseSymMatrix.from_arrays(n, r, c, v)
    Ao = po.from_triplets(n, r, c, v)
    assert np.array_equal(A.row_offsets(), Ao.offs)
    assert np.array_equal(A.col_indices(), Ao.cols)
    assert np.array_equal(A.values(), Ao.vals)
    for kind in (0, 1):
        lap = gs.laplacian(A, gs.LaplacianKind(kind))
        Lo, lam_o, rounds_o = po.laplacian(Ao, kind)
        assert np.array_equal(lap.matrix.row_offsets(), Lo.offs)
        assert np.array_equal(lap.matrix.col_indices(), Lo.cols)
        assert np.array_equal(lap.matrix.values(), Lo.vals)
        assert lap.lambda_max_bound == lam_o
        assert lap.power_rounds == rounds_o


def test_triplet_validation_and_duplicates(gs):
    with pytest.raises(gs.Error) as e:
        gs.SparseSymMatrix.from_triplets(2, [(0, 2, 1.0)])
    assert e.value.code == gs.errc.index_out_of_range
    with pytest.raises(gs.Error) as e:
        gs.SparseSymMatrix.from_triplets(2, [(0, 1, float("nan"))])
    assert e.value.code == gs.errc.invalid_argument
    with pytest.raises(gs.Error) as e:
        gs.SparseSymMatrix.from_triplets(2, [(0, 1, 1.0), (1, 0, 2.0)])
    assert "conflicting duplicate" in str(e.value)
    m = gs.SparseSymMatrix.from_triplets(3, [(0, 1, 1.0), (1, 0, 1.0), (1, 2, 0.0)])
    assert m.stored_entries() == 2  # agreeing duplicate merged, explicit zero dropped
    z = gs.SparseSymMatrix.from_triplets(4, [])
    assert z.stored_entries() == 0 and gs.estimate_lambda_max(z) == 0.0


def test_negative_weight_rejected(gs):
    A = gs.SparseSymMatrix.from_triplets(2, [(0, 1, -0.5)])
    with pytest.raises(gs.Error) as e:
        gs.laplacian(A, gs.LaplacianKind.combinatorial)
    assert e.value.code == gs.errc.negative_weight


def test_isolated_vertex_identity_row(gs):
    A = gs.SparseSymMatrix.from_triplets(3, [(0, 1, 2.0)])
    L = gs.laplacian(A, gs.LaplacianKind.normalized)
    assert L.matrix.coeff(2, 2) == 1.0 and L.matrix.coeff(2, 0) == 0.0


def test_spmm_and_gershgorin_bit_exact(gs):
    n = 300
    r, c, v = random_connected_graph(n, 5)
    A = gs.SparseSymMatrix.from_arrays(n, r, c, v)
    Ao = po.from_triplets(n, r, c, v)
    rng = np.random.default_rng(0)
    for width in (1, 3, 8, 17):
        x = rng.standard_normal((n, width)) if width > 1 else rng.standard_normal(n)
        assert np.array_equal(A.multiply(x), po.spmm(Ao, x))
    assert A.gershgorin_bound() == po.gershgorin(Ao)


# --------------------------------------------------------------------------- filter
@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("width", [1, 2, 3, 5, 8, 13, 64])
def test_filter_apply_bit_exact(gs, kind, width):
    n = 257
    r, c, v = acceptance_graph(n, 1000 + n)
    f, _ = engine_filter(r, c, v, n, kind, 1.0, 30)
    fo = oracle_filter(r, c, v, n, kind, 1.0, 30)
    assert np.array_equal(f.coefficients(), fo.coeffs)
    X = np.random.default_rng(width).standard_normal((n, width))
    if width == 1:
        X = X[:, 0]
    assert np.array_equal(f.apply(X), fo.apply(X))


@pytest.mark.parametrize("deg", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("width", [1, 8, 64])
def test_filter_apply_small_degree_bit_exact(gs, deg, width):
    """The step kernel defers acc updates (three steps at most, the last step always): every
    schedule boundary for K = 1..8, on the scalar, narrow and one-warp-per-row layouts."""
    n = 300
    r, c, v = acceptance_graph(n, 77 + deg)
    f, _ = engine_filter(r, c, v, n, 0, 0.7, deg)
    fo = oracle_filter(r, c, v, n, 0, 0.7, deg)
    X = np.random.default_rng(deg).standard_normal((n, width))
    if width == 1:
        X = X[:, 0]
    assert np.array_equal(f.apply(X), fo.apply(X))


@pytest.mark.parametrize("deg", [1, 2, 3, 4, 7])
def test_sinkhorn_small_degree_matches_oracle(gs, deg):
    """Fused last-step epilogues at the schedule boundaries: same outcome as the oracle (results
    bit for bit, or the same KernelNotPositive when a short expansion goes negative)."""
    n = 90
    r, c, v = acceptance_graph(n, 5 + deg)
    f, _ = engine_filter(r, c, v, n, 1, 0.5, deg)
    fo = oracle_filter(r, c, v, n, 1, 0.5, deg)
    mus, nus = _pairs(n, 3, 40 + deg)
    a = np.full(n, 1.0 / n)
    try:
        res = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m) for m in mus],
                                         [gs.Distribution(x) for x in nus], a, gs.SinkhornParams(60, 1e-10))
        err = None
    except gs.Error as e:
        res, err = None, e.code
    try:
        ref = po.sinkhorn_batch(fo, a, np.array(mus), np.array(nus), 60, 1e-10)
        ref_status = 0
    except po.OracleError as e:
        ref, ref_status = None, e.status
    if err is not None:
        assert ref_status == int(err) + 1
        return
    assert ref_status == 0
    for p, q in enumerate(res):
        assert np.array_equal(q.v, ref["v"][p]) and np.array_equal(q.w, ref["w"][p])
        assert q.iterations == ref["iterations"][p]


def test_two_vertex_closed_form(gs):
    """test_heat.cpp:135-150."""
    f, _ = engine_filter(np.array([0], np.int32), np.array([1], np.int32), np.array([1.0]), 2, 0,
                         1.0, 10)
    out = f.apply(np.array([1.0, 0.0]))
    assert abs(out[0] - 0.5676676416) <= 1e-6 * 0.5676676416
    assert abs(out[1] - 0.4323323584) <= 1e-6 * 0.4323323584
    p = 0.5 * (1 + np.exp(-2.0))
    q = 0.5 * (1 - np.exp(-2.0))
    assert np.max(np.abs(out - [p, q])) <= 1e-9


def test_batched_equals_single(gs):
    """test_heat.cpp:167-179: batched application equals per-signal application."""
    r, c, v = random_connected_graph(40, 9)
    f, _ = engine_filter(r, c, v, 40, 1, 1.2, 25)
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(10)
    batch = np.stack([random_signal(40, rng) for _ in range(7)], axis=1)
    out = f.apply(batch)
    for col in range(7):
        assert np.array_equal(out[:, col], f.apply(batch[:, col].copy()))


# --------------------------------------------------------------------------- Sinkhorn
def _pairs(n, P, seed):
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(seed)
    mus = [random_distribution(n, rng) for _ in range(P)]
    nus = [random_distribution(n, rng) for _ in range(P)]
    return mus, nus


@pytest.mark.parametrize("blk", ["0", "1"])
@pytest.mark.parametrize("P", [1, 4, 9, 40, 70])  # 40, 70: one warp per 64-column row, 1 / 2 groups
def test_sinkhorn_batch_matches_oracle(gs, P, blk, monkeypatch):
    monkeypatch.setenv("GS_BLK", blk)  # 1: the 8-row block kernel (opt-in) on the wide groups
    n = 120
    r, c, v = random_connected_graph(n, 21)
    f, _ = engine_filter(r, c, v, n, 1, 0.9, 30)
    fo = oracle_filter(r, c, v, n, 1, 0.9, 30)
    mus, nus = _pairs(n, P, 7)
    a = np.full(n, 1.0 / n)
    res = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m) for m in mus],
                                     [gs.Distribution(x) for x in nus], a, gs.SinkhornParams(400, 1e-9))
    ref = po.sinkhorn_batch(fo, a, np.array(mus), np.array(nus), 400, 1e-9)
    for p in range(P):
        assert res[p].iterations == ref["iterations"][p]
        assert res[p].converged == ref["converged"][p]
        assert rel(res[p].cost, ref["cost"][p]) <= TOL
        assert rel(res[p].kl, ref["kl"][p]) <= TOL
        assert np.array_equal(res[p].v, ref["v"][p])
        assert np.array_equal(res[p].w, ref["w"][p])
        assert rel(res[p].marginal_error, ref["marginal_error"][p]) <= 1e-6


def test_sinkhorn_mixed_convergence(gs):
    """Pairs converge at different sweeps: the compaction semantics (transport.cpp:210-226)."""
    n = 90
    r, c, v = random_connected_graph(n, 4)
    f, _ = engine_filter(r, c, v, n, 0, 1.0, 30)
    fo = oracle_filter(r, c, v, n, 0, 1.0, 30)
    mus, nus = _pairs(n, 6, 3)
    nus[2] = mus[2]  # self transport converges fast
    a = np.full(n, 1.0 / n)
    res = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m) for m in mus],
                                     [gs.Distribution(x) for x in nus], a, gs.SinkhornParams(60, 1e-8))
    ref = po.sinkhorn_batch(fo, a, np.array(mus), np.array(nus), 60, 1e-8)
    assert len(set(int(x) for x in ref["iterations"])) > 1
    for p in range(6):
        assert res[p].iterations == ref["iterations"][p]
        assert res[p].converged == ref["converged"][p]
        assert np.array_equal(res[p].v, ref["v"][p])
        assert rel(res[p].cost, ref["cost"][p]) <= TOL


def test_disconnected_raises_like_reference(gs):
    """test_transport.cpp:354-367 + batch message with the pair index."""
    f, _ = engine_filter(np.array([0, 2], np.int32), np.array([1, 3], np.int32), np.array([1.0, 1.0]),
                         4, 0, 1.0, 20)
    a = np.full(4, 0.25)
    mu = gs.Distribution.indicator(4, [0])
    nu = gs.Distribution.indicator(4, [3])
    with pytest.raises(gs.Error) as e:
        gs.geodesic_sinkhorn(f, mu, nu, a, gs.SinkhornParams(500, 1e-9))
    assert e.value.code == gs.errc.disconnected
    assert "same graph component" in str(e.value)
    ok = gs.Distribution.indicator(4, [1])
    with pytest.raises(gs.Error) as e:
        gs.geodesic_sinkhorn_batch(f, [mu, mu], [ok, nu], a, gs.SinkhornParams(500, 1e-9))
    assert e.value.code == gs.errc.disconnected
    assert str(e.value).endswith("for pair 1")


def test_kernel_not_positive(gs):
    """test_transport.cpp:369-382."""
    n = 40
    r, c, v = random_connected_graph(n, 40)
    f, _ = engine_filter(r, c, v, n, 1, 50.0, 3)
    a = np.full(n, 1.0 / n)
    with pytest.raises(gs.Error) as e:
        gs.geodesic_sinkhorn(f, gs.Distribution.indicator(n, [7]), gs.Distribution.indicator(n, [20]),
                             a, gs.SinkhornParams(100, 1e-9))
    assert e.value.code == gs.errc.kernel_not_positive


def test_distribution_validation(gs):
    n = 10
    r, c, v = random_connected_graph(n, 2)
    f, _ = engine_filter(r, c, v, n, 1, 1.0, 10)
    good = np.full(n, 0.1)
    bad = np.full(n, 0.2)
    with pytest.raises(gs.Error) as e:
        gs.geodesic_sinkhorn(f, gs.Distribution(good), gs.Distribution(bad, validate=False), good)
    assert "sum to 1" in str(e.value)
    with pytest.raises(gs.Error) as e:
        gs.geodesic_sinkhorn(f, gs.Distribution(good), gs.Distribution(good), -good)
    assert "vertex weights must be positive" in str(e.value)


# --------------------------------------------------------------------------- barycenter
@pytest.mark.parametrize("m,kind,blk", [(1, 1, "0"), (3, 1, "0"), (8, 0, "0"), (11, 1, "0"), (37, 0, "0"),
                                        (37, 0, "1")])
def test_barycenter_matches_oracle(gs, m, kind, blk, monkeypatch):
    monkeypatch.setenv("GS_BLK", blk)
    n = 100
    r, c, v = random_connected_graph(n, 12)
    f, _ = engine_filter(r, c, v, n, kind, 0.8, 30)
    fo = oracle_filter(r, c, v, n, kind, 0.8, 30)
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(8 + m)
    members = [random_distribution(n, rng) for _ in range(m)]
    a = np.full(n, 1.0 / n)
    fam = gs.DistributionFamily([gs.Distribution(x) for x in members])
    res = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(300, 1e-8))
    ref = po.barycenter(fo, a, np.array(members), None, 300, 1e-8)
    assert res.iterations == ref["iterations"]
    assert res.converged == ref["converged"]
    assert rel(res.barycenter.weights, ref["barycenter"]) <= TOL
    for cidx in range(m):
        assert rel(res.scalings[cidx][0], ref["V"][cidx]) <= TOL
        assert rel(res.scalings[cidx][1], ref["W"][cidx]) <= TOL


def test_barycentric_distance(gs):
    n = 30
    r, c, v = random_connected_graph(n, 14)
    f, _ = engine_filter(r, c, v, n, 1, 0.7, 30)
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(13)
    t_fam = gs.DistributionFamily([gs.Distribution(random_distribution(n, rng)) for _ in range(2)])
    c_fam = gs.DistributionFamily([gs.Distribution(random_distribution(n, rng)) for _ in range(2)])
    a = np.full(n, 1.0 / n)
    tc = gs.barycentric_distance(f, t_fam, c_fam, a, gs.SinkhornParams(500, 1e-8))
    ct = gs.barycentric_distance(f, c_fam, t_fam, a, gs.SinkhornParams(500, 1e-8))
    assert abs(tc - ct) <= 1e-8 * (1 + abs(tc))


# --------------------------------------------------------------------------- kNN
def test_knn_tie_break_lower_index(gs):
    """test_graph.cpp:50-58."""
    pts = np.array([[0, 0], [1, 0], [0, 1], [-1, 0], [0, -1]], np.float64)
    A = gs.knn_alpha_decay_graph(pts, 2, 2.0)
    assert A.coeff(2, 3) > 0.0
    assert A.coeff(3, 4) == 0.0
    assert A.coeff(1, 4) > 0.0


def test_knn_three_collinear(gs):
    """test_graph.cpp:41-48."""
    A = gs.knn_alpha_decay_graph(np.array([[0.0], [1.0], [2.0]]), 1, 2.0)
    assert abs(A.coeff(0, 1) - np.exp(-1.0)) <= 1e-12 * np.exp(-1.0)
    assert abs(A.coeff(1, 2) - np.exp(-1.0)) <= 1e-12 * np.exp(-1.0)
    assert A.coeff(0, 2) == 0.0 and A.coeff(0, 0) == 0.0


def test_knn_duplicates_raise(gs):
    with pytest.raises(gs.Error) as e:
        gs.knn_alpha_decay_graph(np.array([[1.0], [1.0]]), 1, 40.0)
    assert e.value.code == gs.errc.duplicate_points


@pytest.mark.parametrize("n,d,k", [(500, 3, 10), (700, 30, 15), (300, 2, 4)])
def test_knn_indices_bit_exact(gs, n, d, k):
    from paper_2211_00805_b200.rng import Rng
    pts = Rng(n + d).normals(n * d).reshape(n, d)
    nb, eps = gs.select_knn(pts, k)
    nbo, epso = po.knn(pts, k)
    assert np.array_equal(nb, nbo)
    assert np.array_equal(eps, epso)


@pytest.mark.parametrize("kernel", [0, 1])
def test_knn_graph_matches_oracle(gs, kernel):
    from paper_2211_00805_b200.rng import Rng
    n, d, k = 400, 3, 10
    pts = Rng(5).normals(n * d).reshape(n, d)
    if kernel == 0:
        A = gs.knn_alpha_decay_graph(pts, k, 40.0)
        sigma = None
    else:
        A, sigma = gs.knn_gaussian_graph(pts, k)
    Ao, sigma_o = po.knn_graph(pts, k, kernel, 40.0)
    assert np.array_equal(A.row_offsets(), Ao.offs)
    assert np.array_equal(A.col_indices(), Ao.cols)
    assert rel(A.values(), Ao.vals) <= 1e-13
    if sigma is not None:
        assert sigma == sigma_o


# --------------------------------------------------------------------------- §8(f) next items
def test_plan_rows_rebuild_marginals(gs):
    """acceptance.cpp:168-197 (criterion 4): plan rows of a converged run rebuild mu and nu."""
    n = 80
    r, c, v = acceptance_graph(n, 480)
    f, _ = engine_filter(r, c, v, n, 1, 1.0, 40)
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(4)
    mu, nu = random_distribution(n, rng), random_distribution(n, rng)
    a = np.full(n, 1.0 / n)
    res = gs.geodesic_sinkhorn(f, gs.Distribution(mu), gs.Distribution(nu), a, gs.SinkhornParams(5000, 1e-6))
    assert res.converged
    plan = gs.plan_rows(res, f, a, np.arange(n))
    assert np.abs(plan.sum(1) - mu).sum() <= 1e-6
    assert np.abs(plan.sum(0) - nu).sum() <= 1e-6
    assert np.array_equal(gs.plan_row(res, f, a, 7), plan[7])


def test_mccann_interpolation_on_device_plan_rows(gs):
    """mccann_interpolate (transport.cpp:326-376) over the geodesic plan's source x target block
    computed on the device in one batched call (bench.cpp:439-448): the block equals the oracle's
    plan rows (impulse applies, then v_i * column * a * w clamped at 0) within 1e-12, and the
    interpolation drawn from either block is the same point set."""
    n = 120
    r, c, v = acceptance_graph(n, 481)
    f, _ = engine_filter(r, c, v, n, 1, 1.0, 40)
    fo = oracle_filter(r, c, v, n, 1, 1.0, 40)
    src_v, tgt_v = np.arange(0, 60), np.arange(60, 120)
    mu = np.zeros(n)
    mu[src_v] = 1.0 / 60
    nu = np.zeros(n)
    nu[tgt_v] = 1.0 / 60
    a = np.full(n, 1.0 / n)
    res = gs.geodesic_sinkhorn(f, gs.Distribution(mu), gs.Distribution(nu), a, gs.SinkhornParams(3000, 1e-9))
    assert res.converged
    block = gs.geodesic_plan_rows(res, f, a, src_v, tgt_v)
    imp = np.zeros((n, 60))
    imp[src_v, np.arange(60)] = 1.0
    cols = fo.apply(imp)  # column i: H e_{src i}; symmetric operator, so row src_i of H
    ref = np.maximum(0.0, res.v[src_v][:, None] * (cols[tgt_v].T * (a[tgt_v] * res.w[tgt_v])[None, :]))
    assert np.max(np.abs(block - ref)) <= 1e-12 * np.max(np.abs(ref))
    pts = np.random.default_rng(5).standard_normal((n, 2))
    got = gs.mccann_interpolate(pts[src_v], pts[tgt_v], lambda i: block[i], 0.5, 60, 11)
    want = gs.mccann_interpolate(pts[src_v], pts[tgt_v], lambda i: ref[i], 0.5, 60, 11)
    assert got.shape == (60, 2)
    assert np.abs(got - want).max() <= 1e-12 or np.mean(np.all(np.isclose(got, want), axis=1)) >= 0.95


def test_graph_file_round_trip(gs, tmp_path):
    """test_graph.cpp:141-150: save/load is exact."""
    from paper_2211_00805_b200.rng import Rng
    pts = Rng(5).normals(40 * 2).reshape(40, 2)
    A = gs.knn_alpha_decay_graph(pts, 3, 40.0)
    path = str(tmp_path / "g.txt")
    gs.save_graph(A, path)
    B = gs.load_graph(path)
    assert B.size() == A.size() and B.stored_entries() == A.stored_entries()
    assert np.array_equal(B.to_dense(), A.to_dense())
    with pytest.raises(gs.Error) as e:
        gs.load_graph(str(tmp_path / "missing.txt"))
    assert e.value.code == gs.errc.io_error


@pytest.mark.parametrize("blk", ["1", "0"])
@pytest.mark.parametrize("n", [8, 61, 500])
def test_block_records_kernel_bit_exact(gs, n, blk, monkeypatch):
    """8-row block kernel (wide fp64 rows): records re-sorted by original column keep every row's
    CSR fma order -- applies on a shuffled-vertex graph (so new and original column orders differ)
    equal the oracle bit for bit, including a last partial block. GS_BLK=1 selects it (opt-in);
    GS_BLK=0 is the default warp-per-row kernel on the same inputs."""
    monkeypatch.setenv("GS_BLK", blk)
    r, c, v = acceptance_graph(n, 4242 + n) if n > 8 else random_connected_graph(n, 5)
    perm = np.random.default_rng(n).permutation(n)
    r, c = perm[np.asarray(r)].astype(np.int32), perm[np.asarray(c)].astype(np.int32)
    f, _ = engine_filter(r, c, v, n, 0, 1.3, 30)
    fo = oracle_filter(r, c, v, n, 0, 1.3, 30)
    for width in (33, 64, 100):
        X = np.random.default_rng(width + n).standard_normal((n, width))
        assert np.array_equal(f.apply(X), fo.apply(X))
        # fp32 wide rows (own rows staged by per-warp TMA copies; odd n leaves a one-row warp)
        X32 = X.astype(np.float32).astype(np.float64)
        ref = fo.apply(X32)
        assert np.max(np.abs(f.apply(X32, fp32=True) - ref)) <= 1e-4 * np.max(np.abs(ref))


@pytest.mark.parametrize("width", [1, 3, 8, 16, 64, 100])
def test_hub_rows_span_several_chunks(gs, width):
    """Rows longer than one CSR chunk (32 entries for 64-column rows, 8 for narrow rows): a hub
    joined to 150 vertices plus a ring, so the next-chunk prefetch and the chunk boundaries of
    every layout are exercised; bit-exact against the oracle."""
    from paper_2211_00805_b200.rng import Rng
    n = 400
    rng = Rng(99)
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i)
        cols.append((i + 1) % n)
        vals.append(rng.uniform(0.2, 1.0))
    for j in range(1, 151):
        rows.append(0)
        cols.append(2 * j + 1)
        vals.append(rng.uniform(0.1, 0.9))
    for i in range(5, n, 37):  # a few more medium-degree rows
        for d in (3, 11, 29, 47):
            rows.append(i)
            cols.append((i + d * 3) % n)
            vals.append(rng.uniform(0.1, 0.5))
    r, c, v = np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals)
    f, _ = engine_filter(r, c, v, n, 0, 0.9, 30)
    fo = oracle_filter(r, c, v, n, 0, 0.9, 30)
    X = np.random.default_rng(width).standard_normal((n, width))
    if width == 1:
        X = X[:, 0]
    assert np.array_equal(f.apply(X), fo.apply(X))
    X32 = np.asarray(X, np.float32).astype(np.float64)
    y32 = f.apply(X32, fp32=True)
    y64 = fo.apply(X32)
    assert np.max(np.abs(y32 - y64)) <= 1e-4 * np.max(np.abs(y64))


@pytest.mark.parametrize("m", [1, 8, 40, 64])
def test_barycenter_fused_log_mean_bit_identical(m, monkeypatch):
    """The log-domain geometric mean fused into the psi apply's last-step epilogue
    (barycenter.cpp:75-78; StepArgs::lb) gives bit-identical barycenters and scalings to the
    separate k_bary_lb / k_max_key passes (GS_BARY_UNFUSED=1), on every step-kernel layout
    (m = 1: warp-per-row kernel; 8: narrow rows; 40/64: windowed wide rows)."""
    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200.rng import Rng
    from helpers import engine_filter, random_connected_graph, random_distribution

    n = 700
    r, c, v = random_connected_graph(n, 91)
    f, _ = engine_filter(r, c, v, n, 1, 0.6, 30)
    rng = Rng(92)
    fam = gs.DistributionFamily([gs.Distribution(random_distribution(n, rng)) for _ in range(m)])
    a = np.full(n, 1.0 / n)
    fused = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(60, 1e-12))
    monkeypatch.setenv("GS_BARY_UNFUSED", "1")
    sep = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(60, 1e-12))
    assert fused.iterations == sep.iterations
    assert np.array_equal(fused.barycenter.weights, sep.barycenter.weights)
    for k in range(m):
        assert np.array_equal(fused.scalings[k][0], sep.scalings[k][0])
        assert np.array_equal(fused.scalings[k][1], sep.scalings[k][1])


@pytest.mark.parametrize("width,hub", [(64, 1500), (64, 300), (40, 1500)])
def test_windowed_kernel_hub_rows_and_fallback(width, hub):
    """Wide batches (>= 256-byte rows) run the windowed kernel unless a row alone needs more ring
    loads than a block may take (gs_win.cu build_schedule: W / 2 = 188 for 512-byte rows; hub
    degrees 300 and 1500 -> the register kernel). Either way the filter apply is bit-identical to
    the oracle."""
    from paper_2211_00805_b200.rng import Rng
    n = 2000
    r, c, v = random_connected_graph(n, 97, 0.5)
    rng = Rng(98)
    have = {(min(a, b), max(a, b)) for a, b in zip(r.tolist(), c.tolist())}
    extra = [(0, j) for j in range(1, hub) if (0, j) not in have]
    r = np.concatenate([r, np.array([e[0] for e in extra], np.int32)])
    c = np.concatenate([c, np.array([e[1] for e in extra], np.int32)])
    v = np.concatenate([v, np.array([rng.uniform(0.1, 0.5) for _ in extra])])
    f, _ = engine_filter(r, c, v, n, 1, 0.8, 30)
    fo = oracle_filter(r, c, v, n, 1, 0.8, 30)
    X = np.abs(np.sin(np.arange(n)[:, None] * (np.arange(width)[None, :] + 1.0))) + 0.05
    assert np.array_equal(f.apply(X), fo.apply(X))
