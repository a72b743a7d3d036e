"""Row-partitioned path (gs_part_*; SURVEY.md §8(e) row partitioning, config 3 shape) on one GPU.

* The partition plan (ranges, halo rows, send lists) against a numpy model of the same rules.
* One part == the unpartitioned engine, bit for bit (apply; Sinkhorn v, w).
* 2, 3 and 5 parts run as threads with an in-process comm (tests/part_comm.py): the stitched
  rows equal the unpartitioned engine bit for bit (every product row is the same fma chain);
  Sinkhorn scalars (cost, KL, marginal error) are sums re-associated across parts, held to
  1e-12 relative; iterations and convergence flags equal.
The unpartitioned engine is itself pinned to the CPU oracle by test_gpu_parity.py.
"""
import math

import numpy as np
import pytest

from helpers import partition_plan, rel
from part_comm import ThreadGroup

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


@pytest.fixture(scope="module")
def roll_filter(gs):
    from paper_2211_00805_b200 import workloads
    roll = workloads.swiss_roll(1500, 1)
    A, _ = gs.knn_gaussian_graph(roll.points, 10)
    lap = gs.laplacian(A, gs.LaplacianKind.combinatorial)
    f = gs.HeatFilter(lap, 1.0, 30)
    return roll, f


def _pairs(roll, P, seed):
    """P (mu, nu) bump pairs close enough to converge."""
    from paper_2211_00805_b200 import workloads
    rng = np.random.default_rng(seed)
    mus, nus = [], []
    for _ in range(P):
        c = rng.uniform(1.7 * math.pi, 4.0 * math.pi)
        mus.append(workloads.bump_in_s(roll, c, 0.5))
        nus.append(workloads.bump_in_s(roll, c + 0.4, 0.5))
    return mus, nus


def plan_model(f, nparts):
    L = f.scaled_laplacian()
    return partition_plan(L.row_offsets(), L.col_indices(), L.values(), f.vertex_order(), nparts)


@pytest.mark.parametrize("nparts", [1, 2, 3, 7])
def test_partition_plan_matches_model(gs, roll_filter, nparts):
    _, f = roll_filter
    model = plan_model(f, nparts)
    for p in range(nparts):
        part = gs.RowPartition(f, nparts, p)
        m = model[p]
        assert (part.row_begin, part.row_end) == (m["rb"], m["re"])
        assert np.array_equal(part.vertices, m["vertices"])
        assert part.n_halo == m["nh"]
        assert np.array_equal(part.recv_counts, m["recv"])
        assert np.array_equal(part.send_counts, m["send"])
        assert part.n_send == part.send_counts.sum()
        assert part.interior == m["interior"]
        if nparts > 1 and m["nh"] > 0:  # the overlap path has work on both sides of the exchange
            assert m["interior"][1] > m["interior"][0]
    # what q receives from p is what p sends to q
    for p in range(nparts):
        for q in range(nparts):
            assert model[q]["recv"][p] == model[p]["send"][q]


@pytest.mark.parametrize("width", [1, 5, 67])
def test_single_part_apply_bit_exact(gs, roll_filter, width):
    _, f = roll_filter
    n = f.size()
    X = np.random.default_rng(width).standard_normal((n, width))
    full = f.apply(X)
    part = gs.RowPartition(f, 1, 0)
    loc = part.apply(X[part.vertices])
    assert np.array_equal(loc, full[part.vertices])


def test_single_part_sinkhorn_bit_exact(gs, roll_filter):
    roll, f = roll_filter
    n = f.size()
    mus, nus = _pairs(roll, 3, 5)
    a = np.full(n, 1.0 / n)
    params = gs.SinkhornParams(200, 1e-9)
    full = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m) for m in mus],
                                      [gs.Distribution(v) for v in nus], a, params)
    part = gs.RowPartition(f, 1, 0)
    vid = part.vertices
    loc = part.sinkhorn([m[vid] for m in mus], [v[vid] for v in nus], a[vid], params)
    for r, q in zip(loc, full):
        assert np.array_equal(r.v, q.v[vid]) and np.array_equal(r.w, q.w[vid])
        assert r.iterations == q.iterations and r.converged == q.converged
        assert rel(np.array([r.cost, r.kl, r.marginal_error]),
                   np.array([q.cost, q.kl, q.marginal_error])) <= 1e-12


def _stitch(parts, vals, n, width=None):
    out = np.zeros((n,) if width is None else (n, width))
    for p, v in zip(parts, vals):
        out[p.vertices] = v
    return out


@pytest.mark.parametrize("nparts", [2, 3, 5])
@pytest.mark.parametrize("fp32", [False, True])
def test_threaded_parts_apply_bit_exact(gs, roll_filter, nparts, fp32):
    _, f = roll_filter
    n = f.size()
    X = np.random.default_rng(nparts).standard_normal((n, 3))
    full = f.apply(X, fp32=fp32)
    parts = [None] * nparts

    def body(r, comm):
        ctx = gs.Context(0)
        part = gs.RowPartition(f, nparts, r, ctx=ctx)
        parts[r] = part
        y = part.apply(X[part.vertices], comm=comm.comm, fp32=fp32)
        assert comm.error is None
        assert comm.a2a_calls == f.degree()  # one halo exchange per Chebyshev step
        return y

    ys = ThreadGroup(nparts).run(body)
    assert np.array_equal(_stitch(parts, ys, n, 3), full)


@pytest.mark.parametrize("nparts", [2, 3])
def test_threaded_parts_sinkhorn(gs, roll_filter, nparts):
    roll, f = roll_filter
    n = f.size()
    mus, nus = _pairs(roll, 3, 11)
    a = np.full(n, 1.0 / n)
    params = gs.SinkhornParams(200, 1e-9)
    full = gs.geodesic_sinkhorn_batch(f, [gs.Distribution(m) for m in mus],
                                      [gs.Distribution(v) for v in nus], a, params)
    parts = [None] * nparts

    def body(r, comm):
        ctx = gs.Context(0)
        part = gs.RowPartition(f, nparts, r, ctx=ctx)
        parts[r] = part
        vid = part.vertices
        return part.sinkhorn([m[vid] for m in mus], [v[vid] for v in nus], a[vid], params,
                             comm=comm.comm)

    res = ThreadGroup(nparts).run(body)
    for p in range(len(mus)):
        v = _stitch(parts, [res[r][p].v for r in range(nparts)], n)
        w = _stitch(parts, [res[r][p].w for r in range(nparts)], n)
        assert np.array_equal(v, full[p].v) and np.array_equal(w, full[p].w)
        for r in range(nparts):  # scalars are global: identical on every rank
            q = res[r][p]
            assert (q.cost, q.kl, q.iterations, q.converged, q.marginal_error) == \
                   (res[0][p].cost, res[0][p].kl, res[0][p].iterations, res[0][p].converged,
                    res[0][p].marginal_error)
        q = res[0][p]
        assert q.iterations == full[p].iterations and q.converged == full[p].converged
        assert rel(np.array([q.cost, q.kl, q.marginal_error]),
                   np.array([full[p].cost, full[p].kl, full[p].marginal_error])) <= 1e-12


def test_threaded_parts_disconnected_and_validation(gs, roll_filter):
    """Config 0's far pair stagnates (Disconnected at sweep 50) on every rank alike; an invalid
    distribution is rejected on every rank with the reference's errc."""
    roll, f = roll_filter
    from paper_2211_00805_b200 import workloads
    n = f.size()
    mu = workloads.bump_in_s(roll, 2 * math.pi, 0.5)
    nu = workloads.bump_in_s(roll, 4 * math.pi, 0.5)
    a = np.full(n, 1.0 / n)
    params = gs.SinkhornParams(100, 1e-6)
    try:
        gs.geodesic_sinkhorn_batch(f, [gs.Distribution(mu)], [gs.Distribution(nu)], a, params)
        full_code = None
    except gs.Error as e:
        full_code = e.code

    def body(r, comm):
        part = gs.RowPartition(f, 2, r, ctx=gs.Context(0))
        vid = part.vertices
        out = []
        try:
            part.sinkhorn([mu[vid]], [nu[vid]], a[vid], params, comm=comm.comm)
            out.append(None)
        except gs.Error as e:
            out.append(e.code)
        try:
            part.sinkhorn([2.0 * mu[vid]], [nu[vid]], a[vid], params, comm=comm.comm)
            out.append(None)
        except gs.Error as e:
            out.append(e.code)
        return out

    codes = ThreadGroup(2).run(body)
    assert codes[0] == codes[1]
    assert codes[0][0] == full_code
    assert codes[0][1] == gs.errc.invalid_argument


def test_multi_part_needs_hooks(gs, roll_filter):
    _, f = roll_filter
    part = gs.RowPartition(f, 2, 0)
    with pytest.raises(gs.Error) as e:
        part.apply(np.zeros(part.n_local))
    assert e.value.code == gs.errc.invalid_argument
