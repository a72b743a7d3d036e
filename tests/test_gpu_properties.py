"""The reference's property tests (SURVEY.md §4 "hot-path tests") restated on the device engine
directly -- the same fixtures as the reference's tests (test_util.hpp graphs and signals, seeded
through geosink::Rng) and the reference's tolerances. Bit-exact parity with the oracle is
covered elsewhere; these read like the reference's own suite."""
import numpy as np
import pytest

from helpers import path_graph, random_connected_graph, random_distribution, random_signal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


def _lap(gs, n, seed, kind, graph=None):
    r, c, v = graph(n, seed) if graph else random_connected_graph(n, seed)
    return gs.laplacian(gs.SparseSymMatrix.from_arrays(n, r, c, v), gs.LaplacianKind(kind))


def _filter(gs, n, seed, kind, t, K, graph=None):
    return gs.HeatFilter(_lap(gs, n, seed, kind, graph), t, K)


def test_filter_invariants(gs):
    """test_heat.cpp:122-149: constants fixed, mass conserved, non-negative outputs."""
    from paper_2211_00805_b200.rng import Rng
    f = _filter(gs, 35, 5, 0, 0.8, 30)
    assert np.abs(f.apply(np.ones(35)) - 1).max() <= 1e-9
    f = _filter(gs, 64, 6, 0, 1.5, 40)
    rng = Rng(7)
    for _ in range(10):
        x = np.abs(random_signal(64, rng))
        assert abs(f.apply(x).sum() - x.sum()) <= 1e-9 * x.sum()
    f = _filter(gs, 100, 8, 0, 1.0, 30)
    rng = Rng(9)
    for _ in range(5):
        assert f.apply(np.abs(random_signal(100, rng))).min() >= -1e-9


def test_filter_semigroup(gs):
    """test_heat.cpp:151-163: H_s H_t = H_{s+t} within 1e-6 (same lambda bound for all three)."""
    from paper_2211_00805_b200.rng import Rng
    lap = _lap(gs, 50, 4, 1)
    x = random_signal(50, Rng(3))
    a, b, ab = (gs.HeatFilter(lap, t, 60) for t in (0.4, 0.7, 1.1))
    assert np.abs(a.apply(b.apply(x)) - ab.apply(x)).max() <= 1e-6 * np.abs(x).max()


def test_laplacian_and_lambda(gs):
    """test_graph.cpp:71-131: edge Laplacian, L 1 = 0, PSD, lambda bracket vs the eigensolver."""
    A = gs.SparseSymMatrix.from_triplets(2, [(0, 1, 1.0)])
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    assert np.array_equal(lap.matrix.to_dense(), [[1, -1], [-1, 1]])
    assert 2.0 <= lap.lambda_max_bound <= 2.02 + 1e-12
    for seed in (1, 2, 3):
        lap = _lap(gs, 80, seed, 0)
        L = lap.matrix.to_dense()
        assert np.abs(L @ np.ones(80)).max() <= 1e-10 * np.abs(L).max()
        w = np.linalg.eigvalsh(L)
        assert w.min() >= -1e-10 and w.max() <= lap.lambda_max_bound <= 1.02 * w.max() + 1e-9


def test_knn_graph_structure(gs):
    """test_graph.cpp:60-69: symmetric, zero diagonal, at most 2 k n stored entries."""
    pts = np.random.default_rng(4).standard_normal((300, 3))
    A = gs.knn_alpha_decay_graph(pts, 6, 10.0)
    D = A.to_dense()
    assert np.array_equal(D, D.T) and np.all(np.diag(D) == 0)
    assert A.stored_entries() <= 2 * 6 * 300


def test_uniform_self_transport(gs):
    """test_transport.cpp:47-58: the uniform self-transport fixed point."""
    f = _filter(gs, 40, 2, 1, 1.0, 30)
    u = np.full(40, 1 / 40)
    res = gs.geodesic_sinkhorn(f, gs.Distribution(u), gs.Distribution(u), u, gs.SinkhornParams(500, 1e-10))
    assert res.converged and res.marginal_error <= 1e-10
    ratio = res.v / res.w
    assert np.abs(ratio / ratio.mean() - 1).max() <= 1e-6


def test_symmetry_and_relabelling(gs):
    """test_transport.cpp:98-144: W(mu, nu) = W(nu, mu) and invariance under vertex relabelling."""
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(5)
    f = _filter(gs, 30, 3, 1, 0.8, 30)
    mu, nu = random_distribution(30, rng), random_distribution(30, rng)
    a = np.full(30, 1 / 30)
    p = gs.SinkhornParams(2000, 1e-10)
    fwd = gs.geodesic_sinkhorn(f, gs.Distribution(mu), gs.Distribution(nu), a, p).cost
    bwd = gs.geodesic_sinkhorn(f, gs.Distribution(nu), gs.Distribution(mu), a, p).cost
    assert abs(fwd - bwd) <= 1e-8 * (1 + abs(fwd))
    n = 24
    rng = Rng(6)
    r, c, v = random_connected_graph(n, 8)
    mu, nu = random_distribution(n, rng), random_distribution(n, rng)
    perm = list(range(n))
    for i in range(n - 1, 0, -1):
        j = rng.below(i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    perm = np.array(perm)
    mu2, nu2 = np.empty(n), np.empty(n)
    mu2[perm], nu2[perm] = mu, nu
    a = np.full(n, 1 / n)
    out = []
    for rr, cc, m_, n_ in ((r, c, mu, nu), (perm[r], perm[c], mu2, nu2)):
        f = gs.HeatFilter(gs.laplacian(gs.SparseSymMatrix.from_arrays(n, rr.astype(np.int32), cc.astype(np.int32), v),
                                       gs.LaplacianKind.normalized), 0.7, 30)
        out.append(gs.geodesic_sinkhorn(f, gs.Distribution(m_), gs.Distribution(n_), a, p).cost)
    assert abs(out[0] - out[1]) <= 1e-10 * (1 + abs(out[0]))


def test_hop_ordering_and_batch_equals_single(gs):
    """test_transport.cpp:146-175."""
    f = _filter(gs, 6, 0, 0, 0.25, 40, graph=lambda n, s: path_graph(n))
    a = np.full(6, 1 / 6)
    e = np.eye(6)
    costs = [gs.geodesic_sinkhorn(f, gs.Distribution(e[0]), gs.Distribution(e[j]), a,
                                  gs.SinkhornParams(500, 1e-6)).cost for j in (1, 2, 3)]
    assert costs[0] < costs[1] < costs[2]
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(7)
    f = _filter(gs, 35, 10, 1, 0.9, 25)
    a = np.full(35, 1 / 35)
    mus = [random_distribution(35, rng) for _ in range(4)]
    nus = [random_distribution(35, rng) for _ in range(4)]
    p = gs.SinkhornParams(400, 1e-8)
    batch = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m) for m in mus], [gs.Distribution(x) for x in nus], a, p)
    for q in range(4):
        single = gs.geodesic_sinkhorn(f, gs.Distribution(mus[q]), gs.Distribution(nus[q]), a, p)
        assert batch[q].iterations == single.iterations
        assert abs(batch[q].cost - single.cost) <= 1e-12 * (1 + abs(single.cost))


def test_barycenter_properties(gs):
    """test_barycenter.cpp:60-126: automorphism of the 8-cycle, alpha = (1, 0) degeneracy."""
    r = np.arange(8, dtype=np.int32)
    f = _filter(gs, 8, 0, 0, 0.5, 30, graph=lambda n, s: (r, (r + 1) % 8, np.ones(8)))
    fam = gs.DistributionFamily([gs.Distribution(np.eye(8)[0]), gs.Distribution(np.eye(8)[4])])
    res = gs.sinkhorn_barycenter(f, fam, np.full(8, 1 / 8), gs.SinkhornParams(500, 1e-10))
    assert res.converged
    b = res.barycenter.weights
    assert np.abs(b - np.roll(b, 4)).max() <= 1e-8
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(5)
    f = _filter(gs, 20, 6, 1, 0.5, 25)
    a = np.full(20, 1 / 20)
    m0, m1 = random_distribution(20, rng), random_distribution(20, rng)
    p = gs.SinkhornParams(300, 1e-8)
    pair = gs.sinkhorn_barycenter(f, gs.DistributionFamily([gs.Distribution(m0), gs.Distribution(m1)],
                                                          np.array([1.0, 0.0])), a, p)
    solo = gs.sinkhorn_barycenter(f, gs.DistributionFamily([gs.Distribution(m0)]), a, p)
    assert np.abs(pair.barycenter.weights - solo.barycenter.weights).sum() <= 1e-9


def test_reruns_are_bit_identical(gs):
    """acceptance.cpp:356-446 (byte-identical reruns): the engine is deterministic run to run."""
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(11)
    f = _filter(gs, 500, 12, 1, 1.0, 30)
    a = np.full(500, 1 / 500)
    mus = [gs.Distribution(random_distribution(500, rng)) for _ in range(20)]
    nus = [gs.Distribution(random_distribution(500, rng)) for _ in range(20)]
    p = gs.SinkhornParams(200, 1e-9)
    one = gs.geodesic_sinkhorn_batch(f, mus, nus, a, p)
    two = gs.geodesic_sinkhorn_batch(f, mus, nus, a, p)
    for x, y in zip(one, two):
        assert np.array_equal(x.v, y.v) and np.array_equal(x.w, y.w)
        assert (x.cost, x.kl, x.iterations, x.marginal_error) == (y.cost, y.kl, y.iterations, y.marginal_error)


def test_caller_locality_order_is_result_neutral(gs):
    """gs_filter_set_order: any vertex order of either layout gives bit-identical applies and
    Sinkhorn scalings (rows keep their entries in the original column order); a non-permutation
    is rejected with invalid_argument."""
    from paper_2211_00805_b200.rng import Rng
    n = 300
    f = _filter(gs, n, 11, 0, 1.0, 30)
    X = np.stack([random_signal(n, Rng(20 + q)) for q in range(64)], axis=1)
    X8 = X[:, :8].copy()
    mus = [random_distribution(n, Rng(40 + p)) for p in range(3)]
    nus = [random_distribution(n, Rng(50 + p)) for p in range(3)]
    a = np.full(n, 1.0 / n)
    prm = gs.SinkhornParams(60, 1e-11)

    def run():
        res = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m) for m in mus],
                                         [gs.Distribution(x) for x in nus], a, prm)
        return f.apply(X), f.apply(X8), [(r.v.copy(), r.w.copy(), r.cost, r.iterations) for r in res]

    base = run()
    perm = np.random.default_rng(3).permutation(n).astype(np.int32)
    f.set_vertex_order(perm, 0)
    f.set_vertex_order(perm[::-1].copy(), 1)
    got = run()
    assert np.array_equal(base[0], got[0]) and np.array_equal(base[1], got[1])
    for (v0, w0, c0, i0), (v1, w1, c1, i1) in zip(base[2], got[2]):
        # v, w and the sweep count are bit-identical; the cost is a tree sum over vertices in
        # layout order, so it may move by an ulp
        assert np.array_equal(v0, v1) and np.array_equal(w0, w1) and i0 == i1
        assert abs(c0 - c1) <= 1e-14 * abs(c0)
    bad = perm.copy()
    bad[0] = bad[1]
    with pytest.raises(gs.Error) as e:
        f.set_vertex_order(bad, 0)
    assert e.value.code == gs.errc.invalid_argument
    assert np.array_equal(f.apply(X), base[0])  # the identity fallback is still a valid order
