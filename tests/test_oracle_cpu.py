"""CPU-only: the oracle (oracle/geosink_oracle.c) pinned against the reference's own RNG output,
independent closed forms / scipy / dense eigendecomposition oracles, and the reference test
suite's known-answer and property tests (restated, cited per test)."""
import os

import numpy as np
import pytest

import pyoracle as po
from helpers import (acceptance_graph, from_weights, path_graph, random_connected_graph,
                     random_distribution, random_signal)
from paper_2211_00805_b200.rng import Rng

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def approx(a, b, eps):
    """doctest::Approx(b).epsilon(eps) (scale 1): |a - b| < eps * (1 + max(|a|, |b|))."""
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


def _golden(name):
    return np.load(os.path.join(GOLDEN, name))


# --------------------------------------------------------------------------- RNG (rng.hpp)
def test_rng_matches_reference_rng_hpp_fixture():
    g = _golden("rng_reference.npz")
    for seed in (0, 1, 42, 0x5EED1A4B, 2**63 + 5):
        assert np.array_equal(po.rng_bits(seed, 700), g[f"bits_{seed}"])
        assert np.array_equal(po.rng_uniform(seed, 700), g[f"uniform_{seed}"])
        assert np.array_equal(po.rng_normal(seed, 701), g[f"normal_{seed}"])
        assert np.array_equal(po.rng_below(seed, 97, 300), g[f"below97_{seed}"])
        r = Rng(seed)  # the engine's host RNG (gs_rng_*) must agree too
        assert np.array_equal(r.normals(701), g[f"normal_{seed}"])
    mix = [po.lib().go_rng_seed_mix(a, b) for a in (0, 1, 7, 2**40) for b in (0, 3, 11)]
    assert np.array_equal(np.array(mix, np.uint64), g["seed_mix"])


def test_rng_matches_live_reference_when_built():
    R = po.ref_rng()
    if R is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    z = np.empty(1001)
    R.ref_rng_normal(12345, 1001, z)
    assert np.array_equal(po.rng_normal(12345, 1001), z)


# --------------------------------------------------------------------------- coefficients
def test_coefficients_match_bessel_closed_form():
    """tests/test_heat.cpp:87-100 (1e-12 for b0, 1e-11 for b_k) against scipy.special.ive."""
    g = _golden("bessel_ive.npz")
    for key in g.files:
        t = float(key[2:])
        ref = g[key]
        b = po.heat_coefficients(t, ref.size - 1)
        assert approx(b[0], ref[0], 1e-12)
        for k in range(1, min(ref.size - 1, 40) + 1):
            assert approx(b[k], ref[k], 1e-11), (t, k)


@pytest.mark.parametrize("t", [0.3, 2.0, 7.0])
def test_series_reproduces_exponential(t):
    """tests/test_heat.cpp:102-113."""
    deg = 4 * int(np.ceil(t)) + 30
    b = po.heat_coefficients(t, deg)
    for x in (0.0, 0.17, 0.5, 1.0, 1.43, 2.0):
        theta = np.arccos(np.clip(x - 1.0, -1, 1))
        acc = b[0] / 2 + sum(b[k] * np.cos(k * theta) for k in range(1, deg + 1))
        assert approx(acc, np.exp(-t * x), 1e-11)


def test_vanishing_time_identity():
    """tests/test_heat.cpp:115-125."""
    b = po.heat_coefficients(1e-12, 10)
    assert abs(b[0] - 2.0) <= 2e-11 and np.abs(b[1:]).max() < 1e-11
    A = po.from_triplets(2, [0], [1], [1.0])
    L, lam, _ = po.laplacian(A, 0)
    f = po.Filter(L, 0, lam, 1e-12, 10)
    x = np.array([0.3, -1.7])
    assert np.abs(f.apply(x) - x).max() <= 1e-8 * 1.7


@pytest.mark.parametrize("t", [0.5, 2.0, 10.0])
def test_coefficient_tail_decay(t):
    """tests/test_heat.cpp:127-133."""
    kmin = int(np.ceil(4 * t)) + 20
    b = po.heat_coefficients(t, kmin + 5)
    assert np.all(np.abs(b[kmin:]) <= 1e-12 * abs(b[0]))


def test_coefficient_validation():
    with pytest.raises(po.OracleError) as e:
        po.heat_coefficients(1.0, 0)
    assert e.value.code == "InvalidArgument"
    with pytest.raises(po.OracleError) as e:
        po.heat_coefficients(float("nan"), 3)
    assert e.value.code == "NonPositiveTime"


# --------------------------------------------------------------------------- filter
def test_two_vertex_closed_form():
    """tests/test_heat.cpp:135-150."""
    A = po.from_triplets(2, [0], [1], [1.0])
    L, lam, _ = po.laplacian(A, 0)
    assert 2.0 <= lam <= 2.02 + 1e-12
    f = po.Filter(L, 0, lam, 1.0, 10)
    out = f.apply(np.array([1.0, 0.0]))
    assert abs(out[0] - 0.5676676416) <= 1e-6 and abs(out[1] - 0.4323323584) <= 1e-6
    p, q = 0.5 * (1 + np.exp(-2.0)), 0.5 * (1 - np.exp(-2.0))
    H = np.array([[p, q], [q, p]])
    assert np.abs(out - H[:, 0]).max() <= 1e-9
    x = np.array([0.25, 0.75])
    assert np.abs(f.apply(x) - H @ x).max() <= 1e-9


def test_filter_vs_dense_oracle_acceptance_criterion_1():
    """tests/acceptance/acceptance.cpp:73-97 at n in {20, 100} (fixture), K=30, <= 1e-8."""
    g = _golden("heat_dense.npz")
    worst = 0.0
    for n in (20, 100):
        r, c, v = acceptance_graph(n, 1000 + n)
        A = po.from_triplets(n, r, c, v)
        for kind in (0, 1):
            L, lam, _ = po.laplacian(A, kind)
            for t in (0.1, 1.0, 5.0):
                f = po.Filter(L, kind, lam, t, 30)
                H = g[f"H_{n}_{kind}_{t}"]
                rng = Rng(77 + n)
                X = np.stack([random_signal(n, rng) for _ in range(20)], axis=1)
                worst = max(worst, np.abs(f.apply(X) - H @ X).max())
    assert worst <= 1e-8, worst


@pytest.mark.parametrize("kind", [0, 1])
def test_filter_vs_eigh_random_graph(kind):
    """tests/test_heat.cpp:152-165: n=50 random graph, 1e-10."""
    r, c, v = random_connected_graph(50, 3)
    A = po.from_triplets(50, r, c, v)
    L, lam, _ = po.laplacian(A, kind)
    t = 0.5 if kind == 1 else 0.5 / lam * 2.0
    f = po.Filter(L, kind, lam, t, 30)
    w, U = np.linalg.eigh(L.to_dense())
    H = (U * np.exp(-t * w)) @ U.T
    rng = Rng(4)
    for _ in range(10):
        x = random_signal(50, rng)
        assert np.abs(f.apply(x) - H @ x).max() <= 1e-10


def test_filter_properties():
    """tests/test_heat.cpp:167-208: batch == single, constants fixed, mass conserved, >= -1e-9."""
    r, c, v = random_connected_graph(40, 9)
    A = po.from_triplets(40, r, c, v)
    L, lam, _ = po.laplacian(A, 1)
    f = po.Filter(L, 1, lam, 1.2, 25)
    rng = Rng(10)
    X = np.stack([random_signal(40, rng) for _ in range(7)], axis=1)
    Y = f.apply(X)
    for col in range(7):
        assert np.array_equal(Y[:, col], f.apply(X[:, col].copy()))
    r, c, v = random_connected_graph(35, 5)
    L, lam, _ = po.laplacian(po.from_triplets(35, r, c, v), 0)
    f = po.Filter(L, 0, lam, 0.8, 30)
    assert np.abs(f.apply(np.ones(35)) - 1).max() <= 1e-9
    r, c, v = random_connected_graph(64, 6)
    L, lam, _ = po.laplacian(po.from_triplets(64, r, c, v), 0)
    f = po.Filter(L, 0, lam, 1.5, 40)
    rng = Rng(7)
    for _ in range(10):
        x = np.abs(random_signal(64, rng))
        assert abs(f.apply(x).sum() - x.sum()) <= 1e-9 * x.sum()
    r, c, v = random_connected_graph(100, 8)
    L, lam, _ = po.laplacian(po.from_triplets(100, r, c, v), 0)
    f = po.Filter(L, 0, lam, 1.0, 30)
    rng = Rng(9)
    for _ in range(5):
        assert f.apply(np.abs(random_signal(100, rng))).min() >= -1e-9


def test_filter_validation():
    """tests/test_heat.cpp:288-298."""
    A = po.from_triplets(2, [0], [1], [1.0])
    L, lam, _ = po.laplacian(A, 0)
    for t, k, code in ((0.0, 10, "NonPositiveTime"), (-1.0, 10, "NonPositiveTime"),
                       (1.0, 0, "InvalidArgument")):
        with pytest.raises(po.OracleError) as e:
            po.Filter(L, 0, lam, t, k)
        assert e.value.code == code


# --------------------------------------------------------------------------- graph
def test_knn_tie_break_and_alpha_decay():
    """tests/test_graph.cpp:41-58."""
    A, _ = po.knn_graph(np.array([[0.0], [1.0], [2.0]]), 1, 0, 2.0)
    assert abs(A.coeff(0, 1) - np.exp(-1)) <= 1e-12 and abs(A.coeff(1, 2) - np.exp(-1)) <= 1e-12
    assert A.coeff(0, 2) == 0.0 and A.coeff(0, 0) == 0.0
    pts = np.array([[0, 0], [1, 0], [0, 1], [-1, 0], [0, -1]], np.float64)
    A, _ = po.knn_graph(pts, 2, 0, 2.0)
    assert A.coeff(2, 3) > 0 and A.coeff(3, 4) == 0 and A.coeff(1, 4) > 0


def test_knn_matches_bruteforce_exact_distances():
    rng = Rng(7)
    pts = rng.normals(120 * 3).reshape(120, 3)
    nb, eps = po.knn(pts, 4)
    d2 = ((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d2, np.inf)
    ref = np.argsort(d2, axis=1, kind="stable")[:, :4]
    assert np.array_equal(nb, ref)
    A, _ = po.knn_graph(pts, 4, 0, 10.0)
    D = A.to_dense()
    assert np.array_equal(D, D.T) and np.all(np.diag(D) == 0) and A.nnz <= 2 * 4 * 120


def test_knn_validation():
    with pytest.raises(po.OracleError) as e:
        po.knn_graph(np.array([[1.0], [1.0]]), 1, 0, 40.0)
    assert e.value.code == "DuplicatePoints"
    pts = Rng(3).normals(20).reshape(10, 2)
    for k, alpha in ((10, 40.0), (0, 40.0), (3, 0.0)):
        with pytest.raises(po.OracleError):
            po.knn_graph(pts, k, 0, alpha)


def test_laplacian_properties():
    """tests/test_graph.cpp:71-139."""
    A = po.from_triplets(2, [0], [1], [1.0])
    L, lam, _ = po.laplacian(A, 0)
    assert np.array_equal(L.to_dense(), [[1, -1], [-1, 1]]) and 2.0 <= lam <= 2.02 + 1e-12
    L, lam, _ = po.laplacian(A, 1)
    assert np.array_equal(L.to_dense(), [[1, -1], [-1, 1]]) and lam == 2.0
    r, c, v = random_connected_graph(60, 11)
    L, lam, _ = po.laplacian(po.from_triplets(60, r, c, v), 0)
    assert np.abs(po.spmm(L, np.ones(60))).max() <= 1e-10 * np.abs(L.vals).max()
    L3, _, _ = po.laplacian(po.from_triplets(3, [0], [1], [2.0]), 1)
    assert L3.coeff(2, 2) == 1.0 and L3.coeff(2, 0) == 0.0
    with pytest.raises(po.OracleError) as e:
        po.laplacian(po.from_triplets(2, [0], [1], [-0.5]), 0)
    assert e.value.code == "NegativeWeight"
    z, _ = po.lambda_max(po.from_triplets(4, [], [], []))
    assert z == 0.0
    for seed in (1, 2, 3):
        r, c, v = random_connected_graph(80, seed)
        L, lam, _ = po.laplacian(po.from_triplets(80, r, c, v), 0)
        lam_n = np.linalg.eigvalsh(L.to_dense()).max()
        assert lam_n <= lam <= 1.02 * lam_n + 1e-9


def test_from_triplets_semantics():
    """sparse.cpp:15-53: mirror, merge agreeing duplicates, drop zeros, reject conflicts."""
    m = po.from_triplets(3, [0, 1, 1], [1, 0, 2], [1.0, 1.0, 0.0])
    assert m.nnz == 2
    with pytest.raises(po.OracleError) as e:
        po.from_triplets(2, [0, 1], [1, 0], [1.0, 2.0])
    assert e.value.code == "InvalidArgument"
    with pytest.raises(po.OracleError) as e:
        po.from_triplets(2, [0], [2], [1.0])
    assert e.value.code == "IndexOutOfRange"


def test_detdot_blocked_order():
    """The documented blocked reduction is an exact restatement for small inputs."""
    x = np.arange(1, 10001, dtype=np.float64) * 1e-3
    y = np.ones_like(x)
    assert po.detdot(x, y) == pytest.approx(x.sum(), rel=1e-15)
    z = np.array([1e16, 1.0, -1e16, 3.0, 5.0])  # order-sensitive values
    assert po.detdot(z, np.ones(5)) == ((z[0] + z[4]) + z[2]) + (z[1] + z[3])


# --------------------------------------------------------------------------- transport
def dense_sinkhorn(C, mu, nu, lam, max_iter, tol):
    """transport.cpp:272-312 restated in numpy (test-only dense oracle)."""
    K = np.exp(-C / lam)
    w = np.ones(nu.size)
    phi = K @ w
    v = np.zeros(mu.size)
    err = np.inf
    conv = False
    for it in range(1, max_iter + 1):
        v = mu / np.maximum(phi, 1e-300)
        w = nu / np.maximum(K.T @ v, 1e-300)
        phi = K @ w
        err = np.abs(v * phi - mu).sum()
        if err <= tol:
            conv = True
            break
    kl = (mu[mu > 0] * np.log(np.maximum(v, 1e-300)[mu > 0])).sum() + \
         (nu[nu > 0] * np.log(np.maximum(w, 1e-300)[nu > 0])).sum() - 1.0
    return dict(v=v, w=w, kl=kl, converged=conv, dual_cost=lam * (1 + kl))


def _filter(n, seed, kind, t, K, graph=random_connected_graph):
    r, c, v = graph(n, seed)
    A = po.from_triplets(n, r, c, v)
    L, lam, _ = po.laplacian(A, kind)
    return po.Filter(L, kind, lam, t, K), L


def test_uniform_self_transport():
    """tests/test_transport.cpp:224-235."""
    f, _ = _filter(40, 2, 1, 1.0, 30)
    u = np.full(40, 1 / 40)
    res = po.sinkhorn_batch(f, u, u[None], u[None], 500, 1e-10, single_style=True)
    assert res["converged"][0] and res["marginal_error"][0] <= 1e-10
    ratio = res["v"][0] / res["w"][0]
    assert np.abs(ratio / ratio.mean() - 1).max() <= 1e-6


def test_proposition_1_equivalence():
    """tests/test_transport.cpp:254-273: cost == dense Sinkhorn dual cost on -4t ln H, 1e-6."""
    rng = Rng(42)
    for seed in (11, 12, 13, 14):
        n = 40 + (seed % 3) * 25
        t = 0.5 + 0.25 * (seed % 4)
        f, L = _filter(n, seed, 1, t, 50)
        mu = random_distribution(n, rng)
        nu = random_distribution(n, rng)
        geo = po.sinkhorn_batch(f, np.ones(n), mu[None], nu[None], 3000, 1e-10, single_style=True)
        w, U = np.linalg.eigh(L.to_dense())
        H = (U * np.exp(-t * w)) @ U.T
        dense = dense_sinkhorn(-4 * t * np.log(H), mu, nu, 4 * t, 3000, 1e-10)
        assert geo["converged"][0] and dense["converged"]
        assert abs(geo["cost"][0] - dense["dual_cost"]) <= 1e-6 * abs(geo["cost"][0])


def test_symmetry_and_relabelling():
    """tests/test_transport.cpp:275-321."""
    rng = Rng(5)
    f, _ = _filter(30, 3, 1, 0.8, 30)
    mu, nu = random_distribution(30, rng), random_distribution(30, rng)
    a = np.full(30, 1 / 30)
    fwd = po.sinkhorn_batch(f, a, mu[None], nu[None], 2000, 1e-10)
    bwd = po.sinkhorn_batch(f, a, nu[None], mu[None], 2000, 1e-10)
    assert abs(fwd["cost"][0] - bwd["cost"][0]) <= 1e-8 * (1 + abs(fwd["cost"][0]))
    n = 24
    rng = Rng(6)
    r, c, v = random_connected_graph(n, 8)
    mu, nu = random_distribution(n, rng), random_distribution(n, rng)
    perm = list(range(n))
    for i in range(n - 1, 0, -1):
        j = rng.below(i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    perm = np.array(perm)
    A1 = po.from_triplets(n, r, c, v)
    A2 = po.from_triplets(n, perm[r], perm[c], v)
    mu2, nu2 = np.empty(n), np.empty(n)
    mu2[perm], nu2[perm] = mu, nu
    a = np.full(n, 1 / n)
    out = []
    for A, m_, n_ in ((A1, mu, nu), (A2, mu2, nu2)):
        L, lam, _ = po.laplacian(A, 1)
        out.append(po.sinkhorn_batch(po.Filter(L, 1, lam, 0.7, 30), a, m_[None], n_[None], 2000,
                                     1e-10)["cost"][0])
    assert abs(out[0] - out[1]) <= 1e-10 * (1 + abs(out[0]))


def test_batch_equals_single():
    """tests/test_transport.cpp:335-352: same iterations, cost <= 1e-12."""
    rng = Rng(7)
    f, _ = _filter(35, 10, 1, 0.9, 25)
    a = np.full(35, 1 / 35)
    mus = np.array([random_distribution(35, rng) for _ in range(4)])
    nus = np.array([random_distribution(35, rng) for _ in range(4)])
    batch = po.sinkhorn_batch(f, a, mus, nus, 400, 1e-8)
    for p in range(4):
        single = po.sinkhorn_batch(f, a, mus[p:p + 1], nus[p:p + 1], 400, 1e-8, single_style=True)
        assert batch["iterations"][p] == single["iterations"][0]
        assert abs(batch["cost"][p] - single["cost"][0]) <= 1e-12 * (1 + abs(single["cost"][0]))


def test_hop_ordering_on_path():
    """tests/test_transport.cpp:323-333."""
    f, _ = _filter(6, 0, 0, 0.25, 40, graph=lambda n, s: path_graph(n))
    a = np.full(6, 1 / 6)
    e = np.eye(6)
    costs = [po.sinkhorn_batch(f, a, e[0][None], e[j][None], 500, 1e-6, single_style=True)["cost"][0]
             for j in (1, 2, 3)]
    assert costs[0] < costs[1] < costs[2]


def test_disconnected_and_kernel_not_positive():
    """tests/test_transport.cpp:354-382."""
    A = po.from_triplets(4, [0, 2], [1, 3], [1.0, 1.0])
    L, lam, _ = po.laplacian(A, 0)
    f = po.Filter(L, 0, lam, 1.0, 20)
    e = np.eye(4)
    with pytest.raises(po.OracleError) as ex:
        po.sinkhorn_batch(f, np.full(4, 0.25), e[0][None], e[3][None], 500, 1e-9, single_style=True)
    assert ex.value.code == "Disconnected" and "same graph component" in str(ex.value)
    with pytest.raises(po.OracleError) as ex:
        po.sinkhorn_batch(f, np.full(4, 0.25), np.stack([e[0], e[0]]), np.stack([e[1], e[3]]), 500,
                          1e-9)
    assert str(ex.value).endswith("for pair 1")
    f, _ = _filter(40, 40, 1, 50.0, 3)
    e = np.eye(40)
    with pytest.raises(po.OracleError) as ex:
        po.sinkhorn_batch(f, np.full(40, 1 / 40), e[7][None], e[20][None], 100, 1e-9)
    assert ex.value.code == "KernelNotPositive"


def test_two_vertex_vs_dense():
    """tests/test_transport.cpp:237-252."""
    A = po.from_triplets(2, [0], [1], [1.0])
    L, lam, _ = po.laplacian(A, 0)
    f = po.Filter(L, 0, lam, 1.0, 30)
    mu, nu = np.array([1.0, 0.0]), np.array([0.0, 1.0])
    geo = po.sinkhorn_batch(f, np.ones(2), mu[None], nu[None], 2000, 1e-12, single_style=True)
    p, q = 0.5 * (1 + np.exp(-2.0)), 0.5 * (1 - np.exp(-2.0))
    H = np.array([[p, q], [q, p]])
    dense = dense_sinkhorn(-4.0 * np.log(H), mu, nu, 4.0, 2000, 1e-12)
    assert geo["converged"][0]
    assert abs(geo["cost"][0] - dense["dual_cost"]) <= 1e-8 * abs(geo["cost"][0])


def test_plan_rows_rebuild_marginals():
    """acceptance criterion 4 (acceptance.cpp:168-197): plan rows diag(v) H diag(a w)."""
    n = 60
    f, _ = _filter(n, 460, 1, 1.0, 40, graph=acceptance_graph)
    rng = Rng(4)
    mu, nu = random_distribution(n, rng), random_distribution(n, rng)
    a = np.full(n, 1 / n)
    res = po.sinkhorn_batch(f, a, mu[None], nu[None], 5000, 1e-6, single_style=True)
    v, w = res["v"][0], res["w"][0]
    H = f.apply(np.eye(n))  # column i = H e_i
    plan = np.maximum(v[:, None] * H.T * (a * w)[None, :], 0.0)
    assert np.abs(plan.sum(1) - mu).sum() <= 1e-6
    assert np.abs(plan.sum(0) - nu).sum() <= 1e-6


# --------------------------------------------------------------------------- barycenter
def dense_barycenter(H, members, alphas, a, max_iter, tol):
    """tests/test_barycenter.cpp:17-52 restated."""
    m, n = members.shape
    app = lambda x: np.maximum(H @ (a * x), 1e-300)
    w = np.ones((m, n))
    phi = np.stack([app(w[i]) for i in range(m)])
    bary = np.full(n, 1 / n)
    for _ in range(max_iter):
        lb = np.zeros(n)
        v = members / phi
        psi = np.stack([app(v[i]) for i in range(m)])
        for i in range(m):
            lb += alphas[i] * np.log(psi[i])
        bary = np.exp(lb - lb.max())
        bary /= bary.sum()
        err = 0.0
        for i in range(m):
            w[i] = bary / psi[i]
            phi[i] = app(w[i])
            err = max(err, np.abs(v[i] * phi[i] - members[i]).sum())
        if err <= tol:
            break
    return bary / bary.sum()


def test_barycenter_path3_and_dense_oracle():
    """tests/test_barycenter.cpp:72-90 and 128-147."""
    f, L = _filter(3, 0, 0, 0.3, 30, graph=lambda n, s: path_graph(n))
    members = np.eye(3)[[0, 2]]
    a = np.full(3, 1 / 3)
    res = po.barycenter(f, a, members, None, 500, 1e-9)
    assert res["converged"]
    b = res["barycenter"]
    assert b[1] > b[0] and b[1] > b[2]
    w, U = np.linalg.eigh(L.to_dense())
    H = (U * np.exp(-0.3 * w)) @ U.T
    ref = dense_barycenter(H, members, [0.5, 0.5], a, 500, 1e-9)
    assert np.abs(b - ref).sum() <= 1e-8
    n = 60
    rng = Rng(8)
    f, L = _filter(n, 9, 1, 0.8, 40)
    members = np.array([random_distribution(n, rng) for _ in range(3)])
    a = np.full(n, 1 / n)
    res = po.barycenter(f, a, members, None, 400, 1e-8)
    assert res["converged"]
    w, U = np.linalg.eigh(L.to_dense())
    H = (U * np.exp(-0.8 * w)) @ U.T
    ref = dense_barycenter(H, members, np.full(3, 1 / 3), a, 400, 1e-8)
    assert np.abs(res["barycenter"] - ref).sum() <= 1e-5


def test_barycenter_degenerate_weights_and_automorphism():
    """tests/test_barycenter.cpp:92-126."""
    r = np.arange(8, dtype=np.int32)
    f, _ = _filter(8, 0, 0, 0.5, 30, graph=lambda n, s: (r, (r + 1) % 8, np.ones(8)))
    res = po.barycenter(f, np.full(8, 1 / 8), np.eye(8)[[0, 4]], None, 500, 1e-10)
    assert res["converged"]
    b = res["barycenter"]
    assert np.abs(b - np.roll(b, 4)).max() <= 1e-8
    rng = Rng(5)
    f, _ = _filter(20, 6, 1, 0.5, 25)
    a = np.full(20, 1 / 20)
    m0, m1 = random_distribution(20, rng), random_distribution(20, rng)
    pair = po.barycenter(f, a, np.stack([m0, m1]), np.array([1.0, 0.0]), 300, 1e-8)
    solo = po.barycenter(f, a, m0[None], None, 300, 1e-8)
    assert np.abs(pair["barycenter"] - solo["barycenter"]).sum() <= 1e-9


def test_barycenter_validation():
    f, _ = _filter(4, 0, 0, 0.5, 10, graph=lambda n, s: path_graph(n))
    with pytest.raises(po.OracleError):
        po.barycenter(f, np.full(4, 0.25), np.full((1, 4), 0.25), np.array([0.5, 0.5])[:1] * 3, 100,
                      1e-6)


# --------------------------------------------------------------------------- EulerHeat (f3)
def test_euler_system_and_dense_solve():
    """heat.cpp:133-219: the system equals I + (t/steps) L and the lockstep-CG apply matches
    (I + hL)^{-steps} X from a dense solve (CG residual tolerance 1e-10)."""
    from helpers import random_connected_graph
    n = 120
    r, c, v = random_connected_graph(n, 31)
    A = po.from_triplets(n, r, c, v)
    L, _, _ = po.laplacian(A, 0)
    t, steps = 0.8, 4
    S = po.euler_system(L, t, steps)
    Ld = np.zeros((n, n))
    for i in range(n):
        for p in range(L.offs[i], L.offs[i + 1]):
            Ld[i, L.cols[p]] = L.vals[p]
    Sd = np.zeros((n, n))
    for i in range(n):
        for p in range(S.offs[i], S.offs[i + 1]):
            Sd[i, S.cols[p]] = S.vals[p]
    assert np.allclose(Sd, np.eye(n) + (t / steps) * Ld, rtol=0, atol=1e-15)
    X = np.random.default_rng(2).standard_normal((n, 3))
    Y, it = po.euler_apply(S, steps, X)
    ref = X.copy()
    for _ in range(steps):
        ref = np.linalg.solve(Sd, ref)
    assert it > 0
    assert np.max(np.abs(Y - ref)) <= 1e-8 * np.max(np.abs(ref))
    y1, _ = po.euler_apply(S, steps, X[:, 1].copy())
    assert np.max(np.abs(y1 - ref[:, 1])) <= 1e-8 * np.max(np.abs(ref))


def test_euler_isolated_vertex_and_validation():
    n = 5  # vertex 4 isolated: its system row is the unit diagonal
    A = po.from_triplets(n, np.array([0, 1, 2], np.int32), np.array([1, 2, 3], np.int32),
                         np.array([1.0, 2.0, 0.5]))
    L, _, _ = po.laplacian(A, 0)
    S = po.euler_system(L, 1.0, 2)
    assert S.offs[5] - S.offs[4] == 1 and S.cols[S.offs[4]] == 4 and S.vals[S.offs[4]] == 1.0
    with pytest.raises(po.OracleError):
        po.euler_system(L, 0.0, 2)
    with pytest.raises(po.OracleError):
        po.euler_system(L, 1.0, 0)


# --------------------------------------------------------------------------- dense baselines
def test_oracle_squared_distances_and_dense_product_plan():
    """bench.cpp:32-39 against the direct formula; transport.cpp:271-311 on a zero cost gives the
    product plan (test_transport.cpp:208-215); validation as the reference (transport.cpp:274-280)."""
    import pyoracle as po
    g = np.random.default_rng(0)
    X, Y = g.standard_normal((7, 5)), g.standard_normal((9, 5))
    D = po.squared_distances(X, Y)
    assert np.abs(D - ((X[:, None] - Y[None]) ** 2).sum(-1)).max() <= 1e-12
    assert (po.squared_distances(X, X) >= 0).all()
    mu, nu = np.array([0.5, 0.3, 0.2]), np.array([0.2, 0.2, 0.6])
    r = po.dense_sinkhorn(np.zeros((3, 3)), mu, nu, 0.7, 500, 1e-12)
    assert r["converged"]
    assert np.abs(r["v"][:, None] * r["w"][None, :] - np.outer(mu, nu)).max() <= 1e-10
    with pytest.raises(po.OracleError, match="non-finite"):
        po.dense_sinkhorn(np.full((3, 3), np.nan), mu, nu, 0.7)
    with pytest.raises(po.OracleError, match="lambda"):
        po.dense_sinkhorn(np.zeros((3, 3)), mu, nu, -1.0)
    with pytest.raises(po.OracleError, match="row underflowed"):
        po.dense_sinkhorn(np.full((3, 3), 1e5), mu, nu, 1e-3)
