"""Sliced step kernels k_cheb_sell / k_cheb_sellw (csrc/gs_sell.cuh, jagged SELL-C store of
gs_sell.cu; opt-in with GS_SELL=1, one row per lane also needs GS_SELL_C32=1) against the oracle's
HeatFilter::apply (heat.cpp:116-131 over sparse.cpp:85-99) and against the default register-gather
kernel k_cheb_step (GS_SELL=0) on the layouts with several rows per warp: one row per lane
(1/2 fp64 columns, 1-4 32-bit columns: C = 32), narrow rows (4/8 fp64 columns: C = 8 / 4) and
128-byte rows (16 fp64 columns: C = 4)."""
import numpy as np
import pytest

from helpers import (acceptance_graph, engine_filter, oracle_filter, random_connected_graph,
                     random_distribution)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


def _hub_graph(n, seed):
    """ring + one hub of degree 150 + medium rows: row lengths from 3 to 150 inside one slice"""
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i); cols.append((i + 1) % n); vals.append(rng.uniform(0.2, 1.0))
    for j in range(1, 151):
        rows.append(7); cols.append((7 + 2 * j + 1) % n); vals.append(rng.uniform(0.1, 0.9))
    for i in range(5, n, 37):
        for d in (3, 11, 29, 47):
            if i != 7 and (i + d * 3) % n != 7:
                rows.append(i); cols.append((i + d * 3) % n); vals.append(rng.uniform(0.1, 0.5))
    return np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals)


@pytest.mark.parametrize("sell", ["1", "0"])
@pytest.mark.parametrize("width", [1, 2, 3, 4, 7, 8, 12, 16])
@pytest.mark.parametrize("n", [29, 401, 1300])
def test_apply_bit_exact_both_kernels(gs, monkeypatch, sell, width, n):
    """fp64 applies equal the oracle bit for bit with the sliced kernel on and off; the 32-bit
    mode stays within 1e-4. n = 29 is a single partial slice, 1300 several CTAs."""
    monkeypatch.setenv("GS_SELL", sell)
    monkeypatch.setenv("GS_SELL_C32", "1")
    r, c, v = _hub_graph(n, 300 + n) if n > 200 else acceptance_graph(n, 300 + n)
    f, _ = engine_filter(r, c, v, n, 0, 0.9, 30)
    fo = oracle_filter(r, c, v, n, 0, 0.9, 30)
    X = np.random.default_rng(width + n).standard_normal((n, width))
    if width == 1:
        X = X[:, 0]
    assert np.array_equal(f.apply(X), fo.apply(X))
    X32 = np.asarray(X, np.float32).astype(np.float64)
    ref = fo.apply(X32)
    assert np.max(np.abs(f.apply(X32, fp32=True) - ref)) <= 1e-4 * np.max(np.abs(ref))


@pytest.mark.parametrize("width", [1, 4, 8, 16, 32])
def test_32bit_mode_identical_to_register_kernel(gs, monkeypatch, width):
    """32-bit mode: the sliced and the register-gather kernels store the same words and run the
    same fp64 chains, so their applies are bit-identical (C = 32, 8, 4, 4 rows per warp)."""
    monkeypatch.setenv("GS_SELL_C32", "1")
    n = 900
    r, c, v = _hub_graph(n, 41)
    f, _ = engine_filter(r, c, v, n, 1, 0.6, 30)
    X = np.abs(np.random.default_rng(width).standard_normal((n, width))) + 0.05
    if width == 1:
        X = X[:, 0]
    monkeypatch.setenv("GS_SELL", "1")
    y1 = f.apply(X, fp32=True)
    monkeypatch.setenv("GS_SELL", "0")
    y0 = f.apply(X, fp32=True)
    assert np.array_equal(y0, y1)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_sinkhorn_epilogues_bit_identical(gs, monkeypatch, P):
    """Fused Sinkhorn epilogues (psi / phi, marginal error partials per tile) through the sliced
    kernel: v, w, costs, errors and iteration counts equal the register-gather kernel's and the
    oracle's (transport.cpp:144-239). P pairs = 2 P... columns per apply = P."""
    import pyoracle as po
    from paper_2211_00805_b200.rng import Rng
    n = 1100
    r, c, v = random_connected_graph(n, 57)
    f, _ = engine_filter(r, c, v, n, 0, 0.8, 30)
    fo = oracle_filter(r, c, v, n, 0, 0.8, 30)
    rng = Rng(58)
    mus = np.stack([random_distribution(n, rng) for _ in range(P)])
    nus = np.stack([random_distribution(n, rng) for _ in range(P)])
    a = np.full(n, 1.0 / n)
    prm = gs.SinkhornParams(40, 1e-11)
    dm = [gs.Distribution(m, validate=False) for m in mus]
    dn = [gs.Distribution(m, validate=False) for m in nus]
    monkeypatch.setenv("GS_SELL", "1")
    on = gs.geodesic_sinkhorn_batch(f, dm, dn, a, prm)
    ref = po.sinkhorn_batch(fo, a, mus, nus, 40, 1e-11)
    monkeypatch.setenv("GS_SELL", "0")
    off = gs.geodesic_sinkhorn_batch(f, dm, dn, a, prm)
    for p in range(P):
        assert np.array_equal(on[p].v, off[p].v) and np.array_equal(on[p].w, off[p].w)
        assert on[p].cost == off[p].cost
        assert abs(on[p].marginal_error - off[p].marginal_error) <= 1e-12 * max(1e-300, off[p].marginal_error)
        assert on[p].iterations == off[p].iterations == ref["iterations"][p]
        assert np.array_equal(on[p].v, ref["v"][p]) and np.array_equal(on[p].w, ref["w"][p])


@pytest.mark.parametrize("m", [2, 8, 16])
def test_barycenter_bit_identical(gs, monkeypatch, m):
    """Barycenter sweeps (BARY_PSI epilogue with the fused log-domain mean, barycenter.cpp:75-78)
    through the sliced kernel equal the register-gather kernel's bit for bit."""
    from paper_2211_00805_b200.rng import Rng
    n = 950
    r, c, v = random_connected_graph(n, 61)
    f, _ = engine_filter(r, c, v, n, 1, 0.6, 30)
    rng = Rng(62)
    fam = gs.DistributionFamily([gs.Distribution(random_distribution(n, rng)) for _ in range(m)])
    a = np.full(n, 1.0 / n)
    monkeypatch.setenv("GS_SELL", "1")
    on = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(50, 1e-12))
    monkeypatch.setenv("GS_SELL", "0")
    off = gs.sinkhorn_barycenter(f, fam, a, gs.SinkhornParams(50, 1e-12))
    assert on.iterations == off.iterations
    assert np.array_equal(on.barycenter.weights, off.barycenter.weights)
    for k in range(m):
        assert np.array_equal(on.scalings[k][0], off.scalings[k][0])
        assert np.array_equal(on.scalings[k][1], off.scalings[k][1])
