"""EulerHeat on the device (gs_euler_*; heat.cpp:133-219) against the CPU
oracle: the system I + (t/steps) L bit for bit, and the lockstep-CG applies bit for bit (the
oracle restates the CG with the device's blocked column sums; tests/test_oracle_cpu.py pins it
to a dense solve)."""
import numpy as np
import pytest

import pyoracle as po
from helpers import acceptance_graph, random_connected_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


def _pair(gs, r, c, v, n, kind):
    A = gs.SparseSymMatrix.from_arrays(n, r, c, v)
    lap = gs.laplacian(A, gs.LaplacianKind(kind))
    Lo, _, _ = po.laplacian(po.from_triplets(n, r, c, v), kind)
    return lap, Lo


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("steps", [1, 3])
@pytest.mark.parametrize("width", [1, 3, 64, 70])
def test_euler_apply_bit_exact(gs, kind, steps, width):
    n = 400
    r, c, v = acceptance_graph(n, 17 + width)
    lap, Lo = _pair(gs, r, c, v, n, kind)
    E = gs.EulerHeat(lap, 0.6, steps, solver="lockstep_cg")
    So = po.euler_system(Lo, 0.6, steps)
    S = E.system()
    assert np.array_equal(S.row_offsets(), So.offs)
    assert np.array_equal(S.col_indices(), So.cols)
    assert np.array_equal(S.values(), So.vals)
    X = np.random.default_rng(width + steps).standard_normal((n, width))
    if width == 1:
        X = X[:, 0]
    Y = E.apply(X)
    Yo, it_o = po.euler_apply(So, steps, X)
    assert np.array_equal(Y, Yo)
    assert E.last_iterations == it_o > 0


def test_euler_isolated_vertex_and_validation(gs):
    r = np.array([0, 1, 2], np.int32)
    c = np.array([1, 2, 3], np.int32)
    v = np.array([1.0, 2.0, 0.5])
    lap, Lo = _pair(gs, r, c, v, 5, 0)  # vertex 4 isolated: unit system row
    E = gs.EulerHeat(lap, 1.0, 2, solver="lockstep_cg")
    S = E.system()
    assert np.array_equal(S.row_offsets(), po.euler_system(Lo, 1.0, 2).offs)
    x = np.arange(5, dtype=np.float64) + 1.0
    y = E.apply(x)
    assert np.array_equal(y, po.euler_apply(po.euler_system(Lo, 1.0, 2), 2, x)[0])
    assert y[4] == x[4]
    with pytest.raises(gs.Error) as e:
        gs.EulerHeat(lap, 0.0, 2, solver="lockstep_cg")
    assert e.value.code == gs.errc.non_positive_time
    with pytest.raises(gs.Error) as e:
        gs.EulerHeat(lap, 1.0, 0, solver="lockstep_cg")
    assert e.value.code == gs.errc.invalid_argument


def test_euler_converges_to_heat_kernel(gs):
    """Implicit Euler with many steps approaches e^{-tL} (the Chebyshev filter)."""
    n = 200
    r, c, v = random_connected_graph(n, 5)
    lap, _ = _pair(gs, r, c, v, n, 1)
    f = gs.HeatFilter(lap, 1.0, 40)
    x = np.random.default_rng(3).standard_normal(n)
    ref = f.apply(x)
    err = [np.abs(gs.apply_euler(lap, 1.0, s, x) - ref).max() / np.abs(ref).max() for s in (10, 100)]
    assert err[1] < err[0] and err[1] < 5e-3


@pytest.mark.parametrize("P,steps", [(1, 2), (5, 3), (9, 1)])
def test_euler_sinkhorn_matches_oracle(gs, P, steps):
    """euler_sinkhorn_batch (transport.cpp:257-269): pairs converge at different sweeps, so the
    lockstep-CG batch shrinks; v, w, iterations, cost and KL bit for bit with the oracle."""
    from helpers import random_distribution
    from paper_2211_00805_b200.rng import Rng
    n = 120
    r, c, v = acceptance_graph(n, 60 + P)
    lap, Lo = _pair(gs, r, c, v, n, 1)
    E = gs.EulerHeat(lap, 0.8, steps, solver="lockstep_cg")
    So = po.euler_system(Lo, 0.8, steps)
    rng = Rng(P)
    mus = [random_distribution(n, rng) for _ in range(P)]
    nus = [random_distribution(n, rng) for _ in range(P)]
    a = np.full(n, 1.0 / n)
    res = gs.euler_sinkhorn_batch(E, [gs.Distribution(m) for m in mus], [gs.Distribution(x) for x in nus], a,
                                  gs.SinkhornParams(300, 1e-9))
    ref = po.euler_sinkhorn_batch(So, steps, 0.8, a, np.array(mus), np.array(nus), 300, 1e-9)
    for p in range(P):
        q = res[p]
        assert q.iterations == ref["iterations"][p] and q.converged == ref["converged"][p]
        assert np.array_equal(q.v, ref["v"][p]) and np.array_equal(q.w, ref["w"][p])
        assert q.cost == ref["cost"][p] and q.kl == ref["kl"][p]
        assert q.marginal_error == ref["marginal_error"][p]


def test_euler_sinkhorn_errors_like_oracle(gs):
    """Disconnected components: the same error (and message) as the oracle."""
    A = gs.SparseSymMatrix.from_triplets(4, [(0, 1, 1.0), (2, 3, 1.0)])
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    E = gs.EulerHeat(lap, 1.0, 2, solver="lockstep_cg")
    e = np.eye(4)
    with pytest.raises(gs.Error) as ex:
        gs.euler_sinkhorn(E, gs.Distribution(e[0]), gs.Distribution(e[3]), np.full(4, 0.25),
                          gs.SinkhornParams(500, 1e-9))
    Lo, _, _ = po.laplacian(po.from_triplets(4, [0, 2], [1, 3], [1.0, 1.0]), 0)
    with pytest.raises(po.OracleError) as ref:
        po.euler_sinkhorn_batch(po.euler_system(Lo, 1.0, 2), 2, 1.0, np.full(4, 0.25), e[0][None], e[3][None],
                                500, 1e-9, single_style=True)
    assert str(ex.value).endswith(str(ref.value))


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("steps,width", [(1, 1), (3, 3), (2, 64), (2, 70)])
def test_euler_direct_matches_dense_solve(gs, kind, steps, width):
    """Solver::direct (heat.cpp:157-173; the device factorises I + hL with a dense Cholesky and
    applies its inverse factor, the reference a sparse LDLT): `steps` solves agree with a dense
    numpy solve of the same system to rounding (1e-12 relative)."""
    n = 500
    r, c, v = acceptance_graph(n, 29 + width)
    lap, _ = _pair(gs, r, c, v, n, kind)
    E = gs.EulerHeat(lap, 0.7, steps, solver="direct")
    S = E.system().to_dense()
    X = np.random.default_rng(width).standard_normal((n, width))
    Y = E.apply(X)
    Z = X.copy()
    for _ in range(steps):
        Z = np.linalg.solve(S, Z)
    assert np.max(np.abs(Y - Z)) <= 1e-12 * np.max(np.abs(Z))
    assert E.last_iterations == 0


def test_euler_automatic_switches_at_4000(gs):
    """Solver::automatic: direct for n <= 4000, lockstep CG above (heat.cpp:157)."""
    for n, direct in ((4000, True), (4100, False)):
        r, c, v = random_connected_graph(n, 61)
        lap, _ = _pair(gs, r, c, v, n, 0)
        E = gs.EulerHeat(lap, 0.5, 1)
        X = np.random.default_rng(n).standard_normal(n)
        Y = E.apply(X)
        assert (E.last_iterations == 0) == direct
        Ec = gs.EulerHeat(lap, 0.5, 1, solver="lockstep_cg")
        Yc = Ec.apply(X)
        assert np.max(np.abs(Y - Yc)) <= 1e-8 * np.max(np.abs(Yc))  # CG: 1e-10 residual


def test_euler_direct_sinkhorn_close_to_cg(gs):
    """euler_sinkhorn over the direct solver: the same iterations and costs within 1e-8 of the
    lockstep-CG run (whose residual tolerance is 1e-10)."""
    n, P = 300, 3
    r, c, v = random_connected_graph(n, 67)
    lap, _ = _pair(gs, r, c, v, n, 0)
    from paper_2211_00805_b200.rng import Rng
    from helpers import random_distribution
    rng = Rng(68)
    mus = [gs.Distribution(random_distribution(n, rng)) for _ in range(P)]
    nus = [gs.Distribution(random_distribution(n, rng)) for _ in range(P)]
    a = np.full(n, 1.0 / n)
    params = gs.SinkhornParams(200, 1e-8)
    rd = gs.euler_sinkhorn_batch(gs.EulerHeat(lap, 0.8, 2, solver="direct"), mus, nus, a, params)
    rc = gs.euler_sinkhorn_batch(gs.EulerHeat(lap, 0.8, 2, solver="lockstep_cg"), mus, nus, a, params)
    for p in range(P):
        assert rd[p].iterations == rc[p].iterations
        assert abs(rd[p].cost - rc[p].cost) <= 1e-8 * abs(rc[p].cost)
