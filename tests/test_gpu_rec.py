"""k_cheb_rec (csrc/gs_step.cuh): the fp64 step kernel for rows shared by several lanes (3-32
columns: the barycenter layouts of configs 2 and 4) that stages each warp's CSR slice in shared
memory as 16-byte records. Against the oracle's HeatFilter::apply (heat.cpp:116-131 over
sparse.cpp:85-99) and against k_cheb_step (GS_REC=0): bit-identical. GS_RPC=4 / 1 cover both CTA
geometries; GS_WIN=0 keeps 32 columns (256-byte rows) off the windowed kernel."""
import numpy as np
import pytest

from helpers import engine_filter, oracle_filter, random_connected_graph, random_distribution

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


def _hub_graph(n, seed, hub=400):
    """ring + chords + one hub row of degree `hub` (a warp slice beyond the stage: folded from
    global memory) + medium rows"""
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i); cols.append((i + 1) % n); vals.append(rng.uniform(0.2, 1.0))
    for j in range(1, hub + 1):
        rows.append(7); cols.append((7 + 2 * j + 1) % n); vals.append(rng.uniform(0.1, 0.9))
    for i in range(5, n, 37):
        for d in (3, 11, 29, 47):
            if i != 7 and (i + d * 3) % n != 7:
                rows.append(i); cols.append((i + d * 3) % n); vals.append(rng.uniform(0.1, 0.5))
    return np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals)


@pytest.mark.parametrize("rpc", ["1", "4"])
@pytest.mark.parametrize("width", [3, 4, 7, 8, 12, 16, 24, 32])
@pytest.mark.parametrize("n", [29, 1300, 2049])
def test_apply_bit_exact(gs, monkeypatch, width, n, rpc):
    """fp64 applies equal the oracle bit for bit with the record kernel on and off"""
    monkeypatch.setenv("GS_RPC", rpc)
    monkeypatch.setenv("GS_WIN", "0")
    r, c, v = _hub_graph(n, 500 + n) if n > 1000 else random_connected_graph(n, 500 + n)
    f, _ = engine_filter(r, c, v, n, 0, 0.9, 30)
    fo = oracle_filter(r, c, v, n, 0, 0.9, 30)
    X = np.random.default_rng(width + n).standard_normal((n, width))
    ref = fo.apply(X)
    monkeypatch.setenv("GS_REC", "1")
    assert np.array_equal(f.apply(X), ref)
    monkeypatch.setenv("GS_REC", "0")
    assert np.array_equal(f.apply(X), ref)


def test_multiply_bit_exact(gs, monkeypatch):
    """plain SpMM (k = 0 launch, sparse.cpp:85-99) on the same widths"""
    import pyoracle as po
    n = 1500
    r, c, v = _hub_graph(n, 78)
    A = gs.SparseSymMatrix.from_arrays(n, r, c, v)
    Ao = po.from_triplets(n, r, c, v)
    for width in (4, 8, 16):
        X = np.random.default_rng(width).standard_normal((n, width))
        assert np.array_equal(A.multiply(X), po.spmm(Ao, X))


@pytest.mark.parametrize("rpc", ["1", "4"])
@pytest.mark.parametrize("P", [3, 8, 16])
def test_sinkhorn_epilogues_bit_identical(gs, monkeypatch, P, rpc):
    """Fused Sinkhorn epilogues (psi / phi, error partials per CTA tile) through the record
    kernel: v, w, costs, errors and iteration counts equal k_cheb_step's and the oracle's
    (transport.cpp:144-239)."""
    import pyoracle as po
    from paper_2211_00805_b200.rng import Rng
    monkeypatch.setenv("GS_RPC", rpc)
    n = 1100
    r, c, v = random_connected_graph(n, 95)
    f, _ = engine_filter(r, c, v, n, 0, 0.8, 30)
    fo = oracle_filter(r, c, v, n, 0, 0.8, 30)
    rng = Rng(96)
    mus = np.stack([random_distribution(n, rng) for _ in range(P)])
    nus = np.stack([random_distribution(n, rng) for _ in range(P)])
    a = np.full(n, 1.0 / n)
    prm = gs.SinkhornParams(40, 1e-11)
    dm = [gs.Distribution(m, validate=False) for m in mus]
    dn = [gs.Distribution(m, validate=False) for m in nus]
    monkeypatch.setenv("GS_REC", "1")
    on = gs.geodesic_sinkhorn_batch(f, dm, dn, a, prm)
    monkeypatch.setenv("GS_REC", "0")
    off = gs.geodesic_sinkhorn_batch(f, dm, dn, a, prm)
    ref = po.sinkhorn_batch(fo, a, mus, nus, 40, 1e-11)
    for p in range(P):
        assert np.array_equal(on[p].v, off[p].v) and np.array_equal(on[p].w, off[p].w)
        assert on[p].cost == off[p].cost
        assert on[p].marginal_error == off[p].marginal_error
        assert on[p].iterations == off[p].iterations == ref["iterations"][p]
        assert np.array_equal(on[p].v, ref["v"][p]) and np.array_equal(on[p].w, ref["w"][p])


@pytest.mark.parametrize("m", [3, 8, 16])
def test_barycenter_bit_identical(gs, monkeypatch, m):
    """Barycenter sweeps (BARY_PSI epilogue with the fused log-domain mean, barycenter.cpp:75-78)
    through the record kernel equal k_cheb_step's bit for bit."""
    from paper_2211_00805_b200.rng import Rng
    n = 950
    r, c, v = random_connected_graph(n, 97)
    f, _ = engine_filter(r, c, v, n, 1, 0.6, 30)
    rng = Rng(98)
    fam = gs.DistributionFamily([gs.Distribution(random_distribution(n, rng)) for _ in range(m)])
    a = np.full(n, 1.0 / n)
    monkeypatch.setenv("GS_REC", "1")
    on = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(50, 1e-12))
    monkeypatch.setenv("GS_REC", "0")
    off = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(50, 1e-12))
    assert on.iterations == off.iterations
    assert np.array_equal(on.barycenter.weights, off.barycenter.weights)
    for k in range(m):
        assert np.array_equal(on.scalings[k][0], off.scalings[k][0])
        assert np.array_equal(on.scalings[k][1], off.scalings[k][1])


@pytest.mark.parametrize("rpc", ["1", "4"])
@pytest.mark.parametrize("P", [4, 8, 16])
def test_heavy_first_launch_order_bit_identical(gs, monkeypatch, P, rpc):
    """The degree-sorted layout's launch order (the heavier half of every 256-row window first,
    gs_step.cuh tile_of; GS_HEAVY_FIRST=0: row order) only permutes which CTA runs which tile:
    v, w, costs, the per-tile error partials (marginal_error) and iteration counts are equal, and
    equal to the oracle's (transport.cpp:144-239). n = 1500: several windows and a partial one."""
    import pyoracle as po
    from paper_2211_00805_b200.rng import Rng
    monkeypatch.setenv("GS_RPC", rpc)
    n = 1500
    r, c, v = _hub_graph(n, 99, hub=300)
    f, _ = engine_filter(r, c, v, n, 0, 0.8, 30)
    fo = oracle_filter(r, c, v, n, 0, 0.8, 30)
    rng = Rng(100)
    mus = np.stack([random_distribution(n, rng) for _ in range(P)])
    nus = np.stack([random_distribution(n, rng) for _ in range(P)])
    a = np.full(n, 1.0 / n)
    prm = gs.SinkhornParams(30, 1e-11)
    dm = [gs.Distribution(m, validate=False) for m in mus]
    dn = [gs.Distribution(m, validate=False) for m in nus]
    monkeypatch.setenv("GS_HEAVY_FIRST", "1")
    on = gs.geodesic_sinkhorn_batch(f, dm, dn, a, prm)
    monkeypatch.setenv("GS_HEAVY_FIRST", "0")
    off = gs.geodesic_sinkhorn_batch(f, dm, dn, a, prm)
    ref = po.sinkhorn_batch(fo, a, mus, nus, 30, 1e-11)
    for p in range(P):
        assert np.array_equal(on[p].v, off[p].v) and np.array_equal(on[p].w, off[p].w)
        assert on[p].cost == off[p].cost and on[p].marginal_error == off[p].marginal_error
        assert on[p].iterations == off[p].iterations == ref["iterations"][p]
        assert np.array_equal(on[p].v, ref["v"][p]) and np.array_equal(on[p].w, ref["w"][p])
