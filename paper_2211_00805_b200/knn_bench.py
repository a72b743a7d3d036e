"""kNN-graph benchmark driver (proj/src/bench.cpp:44-371): the paper's
distance-ranking experiment on the device path.

m clusters on a rotated swiss roll (make_swiss_roll, bench.cpp:59-100) -> alpha-decay kNN graph
-> Laplacian -> heat filter -> geodesic Sinkhorn distances between all m(m-1)/2 pairs of cluster
indicator distributions in ONE batched call -> Pearson / Spearman / precision@5 against the
unrolled-spiral ground truth (bench.cpp:107-214). Methods (bench.hpp:70): `geodesic_sinkhorn`,
the `euler_sinkhorn` competitor (EulerHeat + the same Sinkhorn control) and the dense baselines
`dense_sinkhorn_w1` / `dense_sinkhorn_w2` (bench.cpp:311-331: entropic Sinkhorn between the two
clusters' ambient points with the distance / squared-distance cost, all pairs in one device call,
gs_dense_sinkhorn_groups).

Draws follow geosink::Rng (rng.hpp:13-68) in the reference order; the random rotation is the
Householder QR of a Gaussian matrix with R's diagonal made positive (numpy's LAPACK QR instead of
Eigen's: the same Q up to rounding).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Dict, List

import numpy as np

from . import geosink as gs
from .rng import Rng


@dataclass
class KnnBenchConfig:  # bench.hpp:75-93
    n_distributions: int = 15
    samples_per_dist: int = 1000
    noise_sigma: float = 3.0
    ambient_dim: int = 10
    seeds: List[int] = field(default_factory=lambda: [1])
    k: int = 5
    alpha: float = 40.0
    kind: gs.LaplacianKind = gs.LaplacianKind.normalized
    t: float = 20.0
    degree: int = 100
    sinkhorn: gs.SinkhornParams = field(default_factory=lambda: gs.SinkhornParams(500, 1e-6))
    euler_steps: int = 30  # backward-Euler substeps
    methods: List[str] = field(default_factory=lambda: ["geodesic_sinkhorn", "dense_sinkhorn_w1",
                                                        "dense_sinkhorn_w2"])
    lambda_w1: float = 2.0   # dense baseline regularisation, distance cost
    lambda_w2: float = 20.0  # dense baseline regularisation, squared cost
    # bench-only deviation (as bench.py): run every pair to max_iter instead of raising
    # Disconnected when a pair's marginal error stays above 0.5 for 50 sweeps
    no_stagnation_abort: bool = False


@dataclass
class SwissRollSample:  # bench.hpp SwissRollSample
    ambient: np.ndarray
    intrinsic: np.ndarray
    labels: np.ndarray
    centers: np.ndarray


def random_rotation(dim: int, rng: Rng) -> np.ndarray:
    """bench.cpp:46-57."""
    g = np.array([[rng.normal() for _ in range(dim)] for _ in range(dim)])
    q, r = np.linalg.qr(g)
    return q * np.where(np.diag(r) < 0.0, -1.0, 1.0)[None, :]


def make_swiss_roll(m: int, per: int, noise: float, ambient_dim: int, seed: int) -> SwissRollSample:
    """bench.cpp:59-100."""
    if m < 1 or per < 1:
        raise gs.Error(gs.errc.invalid_argument, "InvalidArgument: need at least one distribution and one sample")
    if ambient_dim < 3:
        raise gs.Error(gs.errc.invalid_argument, "InvalidArgument: ambient dimension must be >= 3")
    if noise < 0.0:
        raise gs.Error(gs.errc.invalid_argument, "InvalidArgument: noise sigma must be >= 0")
    rng = Rng(seed)
    centers = np.empty((m, 2))
    for c in range(m):
        centers[c, 0] = rng.uniform(1.5 * math.pi, 4.5 * math.pi)
        centers[c, 1] = rng.uniform(0.0, 20.0)
    n = m * per
    intrinsic = np.empty((n, 2))
    labels = np.repeat(np.arange(m), per).astype(np.int32)
    flat = np.empty((n, 3))
    for row in range(n):
        c = labels[row]
        s = centers[c, 0] + noise * rng.normal()
        h = centers[c, 1] + noise * rng.normal()
        intrinsic[row] = (s, h)
        flat[row] = (s * math.cos(s), h, s * math.sin(s))
    padded = np.zeros((n, ambient_dim))
    padded[:, :3] = flat
    rot = random_rotation(ambient_dim, rng)
    return SwissRollSample(padded @ rot.T, intrinsic, labels, centers)


def spiral_arclength(s: float) -> float:
    """bench.cpp:102."""
    return 0.5 * (s * math.sqrt(1.0 + s * s) + math.asinh(s))


def ground_truth_distances(sample: SwissRollSample) -> np.ndarray:
    """bench.cpp:104-122: distances between cluster centres on the unrolled spiral."""
    un = np.array([[spiral_arclength(c[0]), c[1]] for c in sample.centers])
    return np.sqrt(((un[:, None, :] - un[None, :, :]) ** 2).sum(-1))


def _average_ranks(v: np.ndarray) -> np.ndarray:  # bench.cpp:128-146
    order = sorted(range(v.size), key=lambda a: (v[a], a))
    ranks = np.empty(v.size)
    i = 0
    while i < v.size:
        j = i
        while j + 1 < v.size and v[order[j + 1]] == v[order[i]]:
            j += 1
        for q in range(i, j + 1):
            ranks[order[q]] = 0.5 * (i + j) + 1.0
        i = j + 1
    return ranks


def _pearson(x: np.ndarray, y: np.ndarray) -> float:  # bench.cpp:148-155
    xc, yc = x - x.mean(), y - y.mean()
    den = np.linalg.norm(xc) * np.linalg.norm(yc)
    if not den > 0.0:
        raise gs.Error(gs.errc.degenerate_input, "DegenerateInput: constant input has no correlation")
    return float(xc @ yc / den)


def rank_metrics(pred: np.ndarray, truth: np.ndarray) -> Dict[str, float]:
    """bench.cpp:161-214: Pearson and Spearman over the upper triangle, row-wise precision@5."""
    m = pred.shape[0]
    iu = np.triu_indices(m, 1)
    up, ut = pred[iu], truth[iu]
    k = min(5, m - 1)

    def row_knn(mat, i):
        idx = [j for j in range(m) if j != i]
        return sorted(idx, key=lambda a: (mat[i, a], a))[:k]

    hits = sum(len(set(row_knn(pred, i)) & set(row_knn(truth, i))) for i in range(m))
    return {"pearson": _pearson(up, ut), "spearman": _pearson(_average_ranks(up), _average_ranks(ut)),
            "p_at_5": hits / (m * k)}


def knn_benchmark(config: KnnBenchConfig = KnnBenchConfig(), ctx=None) -> dict:
    """bench.cpp:246-371 for the geodesic_sinkhorn method; wall times per phase as the reference
    reports them (graph, prepare, distance)."""
    if config.n_distributions < 3:
        raise gs.Error(gs.errc.invalid_argument, "InvalidArgument: need at least three distributions")
    m = config.n_distributions
    keys = ("pearson", "spearman", "p_at_5", "graph", "prepare", "distance")
    per_seed, means = [], {mth: dict.fromkeys(keys, 0.0) for mth in config.methods}
    for seed in config.seeds:
        sample = make_swiss_roll(m, config.samples_per_dist, config.noise_sigma, config.ambient_dim, seed)
        truth = ground_truth_distances(sample)
        n = sample.ambient.shape[0]
        t0 = time.perf_counter()
        needs_graph = any(mth in ("geodesic_sinkhorn", "euler_sinkhorn") for mth in config.methods)
        lap = None
        if needs_graph:  # bench.cpp:264-275
            A = gs.knn_alpha_decay_graph(sample.ambient, config.k, config.alpha, ctx=ctx)
            lap = gs.laplacian(A, config.kind)
        t_graph = time.perf_counter() - t0 if needs_graph else 0.0
        groups = [np.flatnonzero(sample.labels == c) for c in range(m)]
        mus, nus = [], []
        for i in range(m):
            for j in range(i + 1, m):
                mus.append(gs.Distribution.indicator(n, groups[i]))
                nus.append(gs.Distribution.indicator(n, groups[j]))
        a = np.full(n, 1.0 / n)
        seed_out = {"seed": seed, "truth": truth, "distances": {}, "reports": {}, "iterations": {}}
        pair_list = [(i, j) for i in range(m) for j in range(i + 1, m)]
        for method in config.methods:
            t1 = time.perf_counter()
            if method in ("dense_sinkhorn_w1", "dense_sinkhorn_w2"):  # bench.cpp:311-331
                squared = method == "dense_sinkhorn_w2"
                lam = config.lambda_w2 if squared else config.lambda_w1
                runs = gs.dense_sinkhorn_groups(sample.ambient, groups, pair_list, squared, lam,
                                                config.sinkhorn, ctx=ctx)
                t_dist = time.perf_counter() - t1
                costs = [math.sqrt(max(0.0, r.cost)) if squared else r.cost for r in runs]
                d = np.zeros((m, m))
                for (i, j), cst in zip(pair_list, costs):
                    d[i, j] = d[j, i] = cst
                rep = rank_metrics(d, truth)
                rep.update(graph=0.0, prepare=0.0, distance=t_dist)
                seed_out["distances"][method] = d
                seed_out["reports"][method] = rep
                seed_out["iterations"][method] = [r.iterations for r in runs]
                for key in keys:
                    means[method][key] += rep[key] / len(config.seeds)
                continue
            if method == "geodesic_sinkhorn":
                op = gs.HeatFilter(lap, config.t, config.degree)
                solve = gs.geodesic_sinkhorn_batch
            elif method == "euler_sinkhorn":
                op = gs.EulerHeat(lap, config.t, config.euler_steps)
                solve = gs.euler_sinkhorn_batch
            else:
                raise gs.Error(gs.errc.invalid_argument, f"InvalidArgument: unknown benchmark method '{method}'")
            t_prep = time.perf_counter() - t1
            t2 = time.perf_counter()
            runs = solve(op, mus, nus, a, config.sinkhorn, no_stagnation_abort=config.no_stagnation_abort)
            t_dist = time.perf_counter() - t2
            d = np.zeros((m, m))
            q = 0
            for i in range(m):
                for j in range(i + 1, m):
                    d[i, j] = d[j, i] = runs[q].cost
                    q += 1
            rep = rank_metrics(d, truth)
            rep.update(graph=t_graph, prepare=t_prep, distance=t_dist)
            seed_out["distances"][method] = d
            seed_out["reports"][method] = rep
            seed_out["iterations"][method] = [r.iterations for r in runs]
            for key in keys:
                means[method][key] += rep[key] / len(config.seeds)
        per_seed.append(seed_out)
    for mth in means:
        means[mth]["total"] = means[mth]["graph"] + means[mth]["prepare"] + means[mth]["distance"]
    return {"per_seed": per_seed, "mean_report": means}


# ---------------------------------------------------------------------------------------------
# Expected-barycenter-effect experiment (bench.cpp:483-540; PAPER.md "Barycentric distance")
# ---------------------------------------------------------------------------------------------
@dataclass
class EbeConfig:  # bench.hpp:152-167
    has_outlier: bool = True
    outlier_mean: float = -60.0
    treatment_shift: float = 5.0
    control_members: int = 10
    treated_members: int = 10  # the outlier replaces one clean member
    samples_per_member: int = 500
    dim: int = 1
    seed: int = 1
    k: int = 5
    alpha: float = 40.0
    kind: gs.LaplacianKind = gs.LaplacianKind.normalized
    t: float = 3.0
    degree: int = 36
    sinkhorn: gs.SinkhornParams = field(default_factory=lambda: gs.SinkhornParams(60, 1e-6))


def make_ebe_points(config: EbeConfig) -> np.ndarray:
    """bench.cpp:493-509: member blocks of N(shift e_0, I) samples, control first."""
    rng = Rng(config.seed)
    per, members = config.samples_per_member, config.control_members + config.treated_members
    pts = np.empty((members * per, config.dim))
    shifts = [0.0] * config.control_members
    clean = config.treated_members - (1 if config.has_outlier else 0)
    shifts += [config.treatment_shift] * clean
    if config.has_outlier:
        shifts.append(config.outlier_mean)
    for mbr, shift in enumerate(shifts):
        for q in range(per):
            for d in range(config.dim):
                pts[mbr * per + q, d] = (shift if d == 0 else 0.0) + rng.normal()
    return pts


def ebe_experiment(config: EbeConfig = EbeConfig(), ctx=None) -> dict:
    """bench.cpp:483-540: heat-kernel barycenter effect tau and the TV baseline tau_tv."""
    if not (config.control_members >= 1 and config.treated_members >= 1):
        raise gs.Error(gs.errc.invalid_argument, "InvalidArgument: need at least one member per family")
    if config.samples_per_member < 2:
        raise gs.Error(gs.errc.invalid_argument, "InvalidArgument: need at least two samples")
    if config.dim < 1:
        raise gs.Error(gs.errc.invalid_argument, "InvalidArgument: dimension must be >= 1")
    if config.has_outlier and config.treated_members < 2:
        raise gs.Error(gs.errc.invalid_argument, "InvalidArgument: outlier needs at least two treated members")
    pts = make_ebe_points(config)
    n, per = pts.shape[0], config.samples_per_member
    lap = gs.laplacian(gs.knn_alpha_decay_graph(pts, config.k, config.alpha, ctx=ctx), config.kind)
    filt = gs.HeatFilter(lap, config.t, config.degree)
    a = np.full(n, 1.0 / n)

    def member(idx):
        return gs.Distribution.indicator(n, range(idx * per, (idx + 1) * per))

    members_total = config.control_members + config.treated_members
    control = gs.DistributionFamily([member(c) for c in range(config.control_members)], label="control")
    treated = gs.DistributionFamily([member(c) for c in range(config.control_members, members_total)],
                                    label="treated")
    bt = gs.sinkhorn_barycenter(filt, treated, a, config.sinkhorn)
    bc = gs.sinkhorn_barycenter(filt, control, a, config.sinkhorn)
    return {"tau": pts.T @ (bt.barycenter.weights - bc.barycenter.weights),
            "tau_tv": gs.tv_baseline_effect(treated, control, pts), "graph_size": n,
            "converged_treated": bt.converged, "converged_control": bc.converged,
            "barycenters": (bt.barycenter.weights, bc.barycenter.weights), "points": pts}
