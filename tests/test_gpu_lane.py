"""k_cheb_lane (csrc/gs_step.cuh): the one-row-per-lane step kernel that stages each 256-row
block's CSR slice in shared memory with bulk copies (1-2 fp64 columns, 1-4 columns of the 32-bit
mode; config 3's layout). Against the oracle's HeatFilter::apply (heat.cpp:116-131 over
sparse.cpp:85-99) and against k_cheb_step on the same CTA geometry (GS_LANE=0): bit-identical.
GS_RPC=4 forces the multi-block CTA geometry the kernel runs on at sizes the oracle finishes in
seconds (the automatic choice needs n > 3e5)."""
import numpy as np
import pytest

from helpers import engine_filter, oracle_filter, random_connected_graph, random_distribution

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


def _graph(n, seed, hub=0):
    """ring + chords of mixed lengths; `hub` > 0 adds one row of that degree (a block whose
    slice exceeds a shared-memory stage, folded from global memory instead)"""
    from paper_2211_00805_b200.rng import Rng
    rng = Rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i); cols.append((i + 1) % n); vals.append(rng.uniform(0.2, 1.0))
    for i in range(0, n, 3):
        for d in (5, 17, 101)[: 1 + i % 3]:
            rows.append(i); cols.append((i + d) % n); vals.append(rng.uniform(0.1, 0.6))
    seen = set(zip(rows, cols)) | set(zip(cols, rows))
    h = n // 2 + 3
    for j in range(hub):
        c = (h + 2 + j) % n
        if (h, c) not in seen and c != h:
            rows.append(h); cols.append(c); vals.append(rng.uniform(0.01, 0.05))
    return np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals)


@pytest.mark.parametrize("width", [1, 2, 3, 4])
@pytest.mark.parametrize("n,hub", [(700, 0), (2049, 0), (6100, 5200)])
def test_apply_bit_exact(gs, monkeypatch, width, n, hub):
    """fp64 (1-2 columns take the kernel; 3-4 are the narrow layout) equals the oracle bit for
    bit; the 32-bit mode (1-4 columns) is bit-identical with the kernel on and off and within
    1e-4 of the fp64 oracle. n = 700: one partial CTA; 2049: a one-row last block; 6100 with a
    hub of degree 5200: an oversize slice between staged ones."""
    monkeypatch.setenv("GS_RPC", "4")
    monkeypatch.setenv("GS_W1_MAX", "0")
    r, c, v = _graph(n, 400 + n, hub)
    f, _ = engine_filter(r, c, v, n, 0, 0.9, 30)
    fo = oracle_filter(r, c, v, n, 0, 0.9, 30)
    X = np.abs(np.random.default_rng(width + n).standard_normal((n, width))) + 0.01
    if width == 1:
        X = X[:, 0]
    ref = fo.apply(X)
    monkeypatch.setenv("GS_LANE", "1")
    assert np.array_equal(f.apply(X), ref)
    y1 = f.apply(X, fp32=True)
    monkeypatch.setenv("GS_LANE", "0")
    assert np.array_equal(f.apply(X), ref)
    y0 = f.apply(X, fp32=True)
    assert np.array_equal(y0, y1)
    assert np.max(np.abs(y1 - ref)) <= 1e-4 * np.max(np.abs(ref))


def test_multiply_bit_exact(gs, monkeypatch):
    """plain SpMV / SpMM (k = 0 launch, sparse.cpp:85-99) through the staged kernel"""
    monkeypatch.setenv("GS_RPC", "4")
    monkeypatch.setenv("GS_W1_MAX", "0")
    monkeypatch.setenv("GS_LANE", "1")
    import pyoracle as po
    n = 3000
    r, c, v = _graph(n, 77)
    A = gs.SparseSymMatrix.from_arrays(n, r, c, v)
    Ao = po.from_triplets(n, r, c, v)
    for width in (1, 2):
        X = np.random.default_rng(width).standard_normal((n, width))
        if width == 1:
            X = X[:, 0]
        assert np.array_equal(A.multiply(X), po.spmm(Ao, X))


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("P", [1, 2, 4])
def test_sinkhorn_epilogues_bit_identical(gs, monkeypatch, P, fp32):
    """Fused Sinkhorn epilogues (psi / phi, error partials per CTA tile) through the staged
    kernel: v, w, costs, errors and iteration counts equal k_cheb_step's, and in fp64 the
    oracle's (transport.cpp:144-239). fp64 takes the kernel for P <= 2, the 32-bit mode for all."""
    import pyoracle as po
    from paper_2211_00805_b200.rng import Rng
    monkeypatch.setenv("GS_RPC", "4")
    monkeypatch.setenv("GS_PERSIST", "0")
    monkeypatch.setenv("GS_W1_MAX", "0")
    n = 2500
    r, c, v = random_connected_graph(n, 91)
    f, _ = engine_filter(r, c, v, n, 0, 0.8, 30)
    rng = Rng(92)
    mus = np.stack([random_distribution(n, rng) for _ in range(P)])
    nus = np.stack([random_distribution(n, rng) for _ in range(P)])
    a = np.full(n, 1.0 / n)
    prm = gs.SinkhornParams(40, 1e-11)
    dm = [gs.Distribution(m, validate=False) for m in mus]
    dn = [gs.Distribution(m, validate=False) for m in nus]
    monkeypatch.setenv("GS_LANE", "1")
    on = gs.geodesic_sinkhorn_batch(f, dm, dn, a, prm, fp32=fp32)
    monkeypatch.setenv("GS_LANE", "0")
    off = gs.geodesic_sinkhorn_batch(f, dm, dn, a, prm, fp32=fp32)
    for p in range(P):
        assert np.array_equal(on[p].v, off[p].v) and np.array_equal(on[p].w, off[p].w)
        assert on[p].cost == off[p].cost
        assert on[p].marginal_error == off[p].marginal_error
        assert on[p].iterations == off[p].iterations
    if not fp32:
        fo = oracle_filter(r, c, v, n, 0, 0.8, 30)
        ref = po.sinkhorn_batch(fo, a, mus, nus, 40, 1e-11)
        for p in range(P):
            assert on[p].iterations == ref["iterations"][p]
            assert np.array_equal(on[p].v, ref["v"][p]) and np.array_equal(on[p].w, ref["w"][p])


@pytest.mark.parametrize("fp32", [False, True])
def test_barycenter_bit_identical(gs, monkeypatch, fp32):
    """Two-member barycenter (BARY_PSI epilogue with the fused log-domain mean,
    barycenter.cpp:75-78) through the staged kernel equals k_cheb_step's bit for bit."""
    from paper_2211_00805_b200.rng import Rng
    monkeypatch.setenv("GS_RPC", "4")
    n = 1900
    r, c, v = random_connected_graph(n, 93)
    f, _ = engine_filter(r, c, v, n, 1, 0.6, 30)
    rng = Rng(94)
    fam = gs.DistributionFamily([gs.Distribution(random_distribution(n, rng)) for _ in range(2)])
    a = np.full(n, 1.0 / n)
    prm = gs.SinkhornParams(50, 1e-12)
    monkeypatch.setenv("GS_LANE", "1")
    on = gs.sinkhorn_barycenter(f, fam, a, prm, fp32=fp32)
    monkeypatch.setenv("GS_LANE", "0")
    off = gs.sinkhorn_barycenter(f, fam, a, prm, fp32=fp32)
    assert on.iterations == off.iterations
    assert np.array_equal(on.barycenter.weights, off.barycenter.weights)
    for k in range(2):
        assert np.array_equal(on.scalings[k][0], off.scalings[k][0])
        assert np.array_equal(on.scalings[k][1], off.scalings[k][1])
