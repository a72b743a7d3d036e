"""The kNN benchmark driver (knn_bench.py, bench.cpp:246-371) on the device against the same
pipeline on the CPU oracle: the same outcome -- pairwise distances within 1e-9 relative, or the
same Disconnected pair (the stagnation rule, transport.cpp:202-205)."""
import numpy as np
import pytest

import pyoracle as po

pytestmark = pytest.mark.gpu


def _oracle(kb, cfg, seed):
    m = cfg.n_distributions
    sample = kb.make_swiss_roll(m, cfg.samples_per_dist, cfg.noise_sigma, cfg.ambient_dim, seed)
    A = po.knn_graph(sample.ambient, cfg.k, 0, cfg.alpha)[0]
    L, lam, _ = po.laplacian(A, int(cfg.kind))
    fo = po.Filter(L, int(cfg.kind), lam, cfg.t, cfg.degree)
    n = sample.ambient.shape[0]
    mus, nus = [], []
    for i in range(m):
        for j in range(i + 1, m):
            mu = (sample.labels == i).astype(float)
            nu = (sample.labels == j).astype(float)
            mus.append(mu / mu.sum())
            nus.append(nu / nu.sum())
    try:
        return po.sinkhorn_batch(fo, np.full(n, 1.0 / n), np.array(mus), np.array(nus),
                                 cfg.sinkhorn.max_iter, cfg.sinkhorn.tol), None
    except po.OracleError as e:
        return None, str(e)


@pytest.mark.parametrize("m,per,noise,t,seed", [(5, 120, 1.0, 5.0, 2), (4, 200, 3.0, 20.0, 1)])
def test_knn_benchmark_matches_oracle(ctx, m, per, noise, t, seed):
    import paper_2211_00805_b200 as gs
    from paper_2211_00805_b200 import knn_bench as kb
    cfg = kb.KnnBenchConfig(n_distributions=m, samples_per_dist=per, noise_sigma=noise, seeds=[seed],
                            degree=60, t=t)
    ref, ref_err = _oracle(kb, cfg, seed)
    try:
        res = kb.knn_benchmark(cfg)
        err = None
    except gs.Error as e:
        res, err = None, str(e)
    if ref_err is not None or err is not None:
        assert err == ref_err  # same errc, message and failing pair
        return
    d = res["per_seed"][0]["distances"]
    q = 0
    for i in range(m):
        for j in range(i + 1, m):
            assert abs(d[i, j] - ref["cost"][q]) <= 1e-9 * abs(ref["cost"][q])
            q += 1
    rep = res["mean_report"]["geodesic_sinkhorn"]
    assert -1.0 <= rep["spearman"] <= 1.0 and 0.0 <= rep["p_at_5"] <= 1.0
