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
                            degree=60, t=t, methods=["geodesic_sinkhorn"])
    ref, ref_err = _oracle(kb, cfg, seed)
    try:
        res = kb.knn_benchmark(cfg)
        err = None
    except gs.Error as e:
        res, err = None, str(e)
    if ref_err is not None or err is not None:
        assert err == ref_err  # same errc, message and failing pair
        return
    d = res["per_seed"][0]["distances"]["geodesic_sinkhorn"]
    q = 0
    for i in range(m):
        for j in range(i + 1, m):
            assert abs(d[i, j] - ref["cost"][q]) <= 1e-9 * abs(ref["cost"][q])
            q += 1
    rep = res["mean_report"]["geodesic_sinkhorn"]
    assert -1.0 <= rep["spearman"] <= 1.0 and 0.0 <= rep["p_at_5"] <= 1.0


def test_ebe_experiment_matches_oracle(ctx):
    """bench.cpp:483-540 on the device: the barycenters (and so tau) within 1e-9 of the oracle's;
    the heat-kernel effect is robust to the outlier member where the TV baseline is not."""
    from paper_2211_00805_b200 import knn_bench as kb
    cfg = kb.EbeConfig(samples_per_member=60)
    res = kb.ebe_experiment(cfg)
    pts = res["points"]
    n, per = pts.shape[0], cfg.samples_per_member
    A = po.knn_graph(pts, cfg.k, 0, cfg.alpha)[0]
    L, lam, _ = po.laplacian(A, int(cfg.kind))
    fo = po.Filter(L, int(cfg.kind), lam, cfg.t, cfg.degree)

    def fam(lo, hi):
        out = []
        for c in range(lo, hi):
            w = np.zeros(n)
            w[c * per:(c + 1) * per] = 1.0
            out.append(w / w.sum())
        return np.array(out)

    a = np.full(n, 1.0 / n)
    bt = po.barycenter(fo, a, fam(10, 20), None, cfg.sinkhorn.max_iter, cfg.sinkhorn.tol)["barycenter"]
    bc = po.barycenter(fo, a, fam(0, 10), None, cfg.sinkhorn.max_iter, cfg.sinkhorn.tol)["barycenter"]
    tau_ref = pts.T @ (bt - bc)
    assert abs(res["tau"][0] - tau_ref[0]) <= 1e-9 * abs(tau_ref[0])
    assert abs(res["tau"][0] - cfg.treatment_shift) < abs(res["tau_tv"][0] - cfg.treatment_shift)
