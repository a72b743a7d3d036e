"""Grid kNN (gs_graph.cu k_knn_grid, d <= 3) against the tiled brute force on the same device:
identical neighbour lists (the (d2, index) order of select_knn, graph.cpp:30-71, ties to the
lower index) and identical eps_k, bit for bit. The brute force is itself pinned to the CPU
oracle by test_gpu_parity.py."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gs(ctx):
    import paper_2211_00805_b200 as gs
    return gs


def _both(gs, pts, k):
    out = {}
    for mode in ("brute", "grid"):
        os.environ["GS_KNN"] = mode
        try:
            out[mode] = gs.select_knn(pts, k)
        finally:
            del os.environ["GS_KNN"]
    return out["brute"], out["grid"]


def _clouds():
    rng = np.random.default_rng(7)
    yield "uniform3d", rng.uniform(-3, 5, size=(40000, 3)), 10
    from paper_2211_00805_b200 import workloads
    yield "swiss_roll", workloads.swiss_roll(30000, 2).points, 10
    g = np.stack(np.meshgrid(np.arange(60), np.arange(50), np.arange(3), indexing="ij"), -1)
    yield "lattice_ties", g.reshape(-1, 3).astype(np.float64), 12  # exact distance ties
    yield "plane2d", rng.standard_normal((20000, 2)) * [10.0, 0.1], 7
    yield "line1d", np.sort(rng.uniform(0, 1, size=(5000, 1)), axis=0), 5
    yield "k32", rng.uniform(0, 1, size=(8000, 3)), 32


@pytest.mark.parametrize("name,pts,k", list(_clouds()), ids=lambda v: v if isinstance(v, str) else "")
def test_grid_knn_equals_brute_force(gs, name, pts, k):
    (nb_b, eps_b), (nb_g, eps_g) = _both(gs, pts, k)
    assert np.array_equal(nb_b, nb_g), name
    assert np.array_equal(eps_b, eps_g), name


def test_grid_graph_equals_brute_force(gs):
    from paper_2211_00805_b200 import workloads
    pts = workloads.swiss_roll(20000, 3).points
    mats = {}
    for mode in ("brute", "grid"):
        os.environ["GS_KNN"] = mode
        try:
            A, sigma = gs.knn_gaussian_graph(pts, 10)
        finally:
            del os.environ["GS_KNN"]
        mats[mode] = (A.row_offsets(), A.col_indices(), A.values(), sigma)
    for a, b in zip(mats["brute"], mats["grid"]):
        assert np.array_equal(a, b)
