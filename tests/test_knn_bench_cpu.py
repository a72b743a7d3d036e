"""Host logic of the kNN benchmark driver (paper_2211_00805_b200/knn_bench.py; bench.cpp:44-214):
sample construction, ground truth, rank metrics."""
import math

import numpy as np

from paper_2211_00805_b200 import knn_bench as kb


def test_average_ranks_ties_and_metrics():
    r = kb._average_ranks(np.array([3.0, 1.0, 3.0, 2.0]))
    assert np.array_equal(r, [3.5, 1.0, 3.5, 2.0])  # 1-based, ties share the mean rank
    x = np.array([1.0, 2.0, 3.0, 4.0])
    assert abs(kb._pearson(x, 2 * x + 1) - 1.0) < 1e-15
    m = 6
    rng = np.random.default_rng(0)
    pts = rng.standard_normal((m, 2))
    truth = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    rep = kb.rank_metrics(truth, truth)
    assert rep["p_at_5"] == 1.0 and abs(rep["spearman"] - 1.0) < 1e-15
    rep2 = kb.rank_metrics(truth.max() - truth + np.eye(m) * 0, truth)
    assert rep2["spearman"] < 0


def test_swiss_roll_sample_and_truth():
    s1 = kb.make_swiss_roll(4, 10, 0.5, 6, seed=3)
    s2 = kb.make_swiss_roll(4, 10, 0.5, 6, seed=3)
    assert np.array_equal(s1.ambient, s2.ambient)
    assert s1.ambient.shape == (40, 6) and np.array_equal(np.bincount(s1.labels), [10] * 4)
    # the rotation is orthogonal: intrinsic geometry (norms) is preserved
    s, h = s1.intrinsic[:, 0], s1.intrinsic[:, 1]
    flat = np.stack([s * np.cos(s), h, s * np.sin(s)], 1)
    assert np.allclose(np.linalg.norm(s1.ambient, axis=1), np.linalg.norm(flat, axis=1), rtol=1e-12)
    d = kb.ground_truth_distances(s1)
    assert d.shape == (4, 4) and np.allclose(d, d.T) and np.all(np.diag(d) == 0)
    c = s1.centers
    exp = math.hypot(kb.spiral_arclength(c[0, 0]) - kb.spiral_arclength(c[1, 0]), c[0, 1] - c[1, 1])
    assert abs(d[0, 1] - exp) <= 1e-12 * exp
