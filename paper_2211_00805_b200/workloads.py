"""Seeded synthetic inputs for the BASELINE.json configs (host-side input generation).

All draws go through geosink::Rng semantics (rng.hpp:13-68) so a config is reproducible from
its seed on any host. Decisions recorded in DESIGN.md ("Workloads"):
  * swiss roll: per point draw s ~ U(1.5pi, 4.5pi), h ~ U(0, 20), then three N(0, 0.1^2)
    noise terms, in that order; x = (s cos s + nx, h + ny, s sin s + nz);
  * graph: symmetrised k-NN, Gaussian weights exp(-d^2/sigma^2), sigma = median eps_k;
  * bump "width" = Gaussian standard deviation; mixtures are equal-weight sums of bumps;
  * Gaussian mixtures in R^d: means ~ N(0, 5^2 I), isotropic sigma = 1, balanced components
    (point i belongs to component i mod C);
  * cluster-subset members: uniform over a random `frac` subset of the points of the chosen
    clusters.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

TWO_PI = 2.0 * math.pi


_RNG_CLASS = None


def set_rng_class(cls) -> None:
    """Draw inputs from another geosink::Rng implementation with the same interface (the
    reference arm of bench.py uses the oracle's, oracle/pyoracle.py Rng, so it never loads the
    product library). None restores the engine's host RNG (paper_2211_00805_b200/rng.py)."""
    global _RNG_CLASS
    _RNG_CLASS = cls


def Rng(seed: int):
    if _RNG_CLASS is not None:
        return _RNG_CLASS(seed)
    from .rng import Rng as EngineRng
    return EngineRng(seed)


def _normalise(w: np.ndarray) -> np.ndarray:
    w = np.array(w, np.float64)
    w /= w.sum()
    w /= w.sum()
    return w


@dataclass
class SwissRoll:
    points: np.ndarray  # n x 3
    s: np.ndarray
    h: np.ndarray


def swiss_roll(n: int, seed: int, noise: float = 0.1) -> SwissRoll:
    raw = Rng(seed).pattern(5 * n, [("u", 1.5 * math.pi, 4.5 * math.pi), ("u", 0.0, 20.0),
                                    ("n", 0.0, noise), ("n", 0.0, noise), ("n", 0.0, noise)])
    raw = raw.reshape(n, 5)
    s, h = raw[:, 0].copy(), raw[:, 1].copy()
    pts = np.empty((n, 3))
    pts[:, 0] = s * np.cos(s) + raw[:, 2]
    pts[:, 1] = h + raw[:, 3]
    pts[:, 2] = s * np.sin(s) + raw[:, 4]
    return SwissRoll(pts, s, h)


def bump_in_s(roll: SwissRoll, centre: float, width: float) -> np.ndarray:
    """Config 0/3: normalised Gaussian bump in the roll parameter s."""
    return _normalise(np.exp(-((roll.s - centre) ** 2) / (2.0 * width * width)))


def bump_mixture_pairs(roll: SwissRoll, pairs: int, seed: int, bumps: int = 3,
                       wmin: float = 0.3, wmax: float = 1.0):
    """Config 1: `pairs` (source, target) distributions, each a normalised equal-weight mixture of
    `bumps` Gaussian bumps in (s, h) with centres s ~ U(1.5pi, 4.5pi), h ~ U(0, 20) and widths
    ~ U(wmin, wmax). Returns (mus, nus) shaped (pairs, n)."""
    rng = Rng(seed)
    out = np.empty((2 * pairs, roll.s.size))
    for q in range(2 * pairs):
        dens = np.zeros(roll.s.size)
        for _ in range(bumps):
            sc = rng.uniform(1.5 * math.pi, 4.5 * math.pi)
            hc = rng.uniform(0.0, 20.0)
            w = rng.uniform(wmin, wmax)
            dens += np.exp(-((roll.s - sc) ** 2 + (roll.h - hc) ** 2) / (2.0 * w * w))
        out[q] = _normalise(dens)
    return out[0::2].copy(), out[1::2].copy()


def bump_mixture_companions(roll: SwissRoll, pairs: int, seed: int, bumps: int = 3,
                            wmin: float = 0.3, wmax: float = 1.0, shift: float = 0.5):
    """Well-posed companion of config 1 (SURVEY §7 hard part 1): each source is a config-1-style
    mixture (`bumps` equal-weight Gaussian bumps in (s, h), widths ~ U(wmin, wmax), centres kept
    one width-unit inside the roll's s/h range so no bump is cut by the boundary); its target
    moves every bump centre by a geodesic offset drawn uniformly in [-shift, shift]^2 (an s
    offset of d / sqrt(1 + s^2): the roll's arc-length element) and keeps the width, so each target bump carries its source bump's mass and lies within the K-hop reach
    of it: the reference converges instead of raising Disconnected. Returns (mus, nus)."""
    rng = Rng(seed)
    n = roll.s.size
    mus = np.empty((pairs, n))
    nus = np.empty((pairs, n))
    for q in range(pairs):
        src = np.zeros(n)
        dst = np.zeros(n)
        for _ in range(bumps):
            sc = rng.uniform(1.5 * math.pi + 2.0, 4.5 * math.pi - 2.0)
            hc = rng.uniform(3.0, 17.0)
            w = rng.uniform(wmin, wmax)
            ds = rng.uniform(-shift, shift)
            dh = rng.uniform(-shift, shift)
            ds = ds / math.sqrt(1.0 + sc * sc)
            src += np.exp(-((roll.s - sc) ** 2 + (roll.h - hc) ** 2) / (2.0 * w * w))
            dst += np.exp(-((roll.s - sc - ds) ** 2 + (roll.h - hc - dh) ** 2) / (2.0 * w * w))
        mus[q] = _normalise(src)
        nus[q] = _normalise(dst)
    return mus, nus


@dataclass
class Mixture:
    points: np.ndarray  # n x d
    labels: np.ndarray  # n


def gaussian_mixture(n: int, d: int, components: int, seed: int, mean_scale: float = 5.0,
                     sigma: float = 1.0) -> Mixture:
    rng = Rng(seed)
    means = rng.pattern(components * d, [("n", 0.0, mean_scale)]).reshape(components, d)
    labels = (np.arange(n) % components).astype(np.int32)
    noise = rng.pattern(n * d, [("n", 0.0, sigma)]).reshape(n, d)
    return Mixture(means[labels] + noise, labels)


def cluster_subset_members(mix: Mixture, members: int, clusters_each: int, frac: float, seed: int,
                           cluster_pool=None) -> np.ndarray:
    """Configs 2/4: each member uniform over a random `frac` subset of the points of
    `clusters_each` random clusters drawn from `cluster_pool` (default: all)."""
    rng = Rng(seed)
    pool = np.arange(mix.labels.max() + 1) if cluster_pool is None else np.asarray(cluster_pool)
    n = mix.labels.size
    out = np.zeros((members, n))
    for m in range(members):
        chosen = []
        avail = list(pool)
        for _ in range(min(clusters_each, len(avail))):
            chosen.append(avail.pop(rng.below(len(avail))))
        idx = np.flatnonzero(np.isin(mix.labels, chosen))
        keep = rng.pattern(idx.size, [("u", 0.0, 1.0)]) < frac
        sel = idx[keep] if keep.any() else idx[:1]
        out[m, sel] = 1.0
        out[m] = _normalise(out[m])
    return out


@dataclass
class Config1:
    roll: SwissRoll
    mus: np.ndarray
    nus: np.ndarray
    k: int = 10
    t: float = 1.0
    degree: int = 30
    sweeps: int = 200


def config1(n: int = 200_000, pairs: int = 64, seed: int = 1, pair_seed: int = 2) -> Config1:
    roll = swiss_roll(n, seed)
    mus, nus = bump_mixture_pairs(roll, pairs, pair_seed)
    return Config1(roll, mus, nus)


@dataclass
class Config2:
    mix: Mixture
    members: np.ndarray  # m x n
    k: int = 15
    t: float = 0.5
    degree: int = 30
    sweeps: int = 200


def config2(n: int = 1_000_000, m: int = 8, d: int = 30, components: int = 20, seed: int = 3,
            member_seed: int = 4) -> Config2:
    """Config 2: 20-component Gaussian mixture in R^30 (means ~ N(0, 5^2 I), sigma = 1); m members,
    each uniform over a random 60% subset of the points of 4 random clusters."""
    mix = gaussian_mixture(n, d, components, seed)
    members = cluster_subset_members(mix, m, 4, 0.6, member_seed)
    return Config2(mix, members)


def _cluster_choice(rng: Rng, pool, count):
    avail = list(pool)
    return [avail.pop(rng.below(len(avail))) for _ in range(min(count, len(avail)))]


@dataclass
class Config4:
    mix: Mixture
    group_a: np.ndarray  # m x n
    group_b: np.ndarray  # m x n
    k: int = 15
    t: float = 0.5
    degree: int = 30
    sweeps: int = 200


def config4_from_mixture(mix: Mixture, m: int = 16, member_seed: int = 6) -> Config4:
    """Config 4's two groups on a given 40-component mixture (config4's member draws)."""
    rng = Rng(member_seed)
    lab = mix.labels
    n = lab.size

    def uniform_over(clusters):
        w = np.isin(lab, clusters).astype(np.float64)
        return w / w.sum()

    ga = np.empty((m, n))
    gb = np.empty((m, n))
    for q in range(m):
        ga[q] = _normalise(uniform_over(_cluster_choice(rng, range(0, 20), 10)))
    for q in range(m):
        base = uniform_over(_cluster_choice(rng, range(0, 20), 10))
        shift = uniform_over(_cluster_choice(rng, range(20, 40), 10))
        gb[q] = _normalise(0.8 * base + 0.2 * shift)
    return Config4(mix, ga, gb)


def config4(n: int = 4_000_000, m: int = 16, d: int = 30, components: int = 40, seed: int = 5,
            member_seed: int = 6) -> Config4:
    """Config 4: 40-component Gaussian mixture in R^30 (means ~ N(0, 5^2 I), sigma = 1). Decisions
    (DESIGN.md "Workloads"): a group-A member is uniform over the points of a random half (10) of
    clusters 0-19; a group-B member is the same construction with 20% of its mass moved onto the
    points of a random half of clusters 20-39 (a seeded mixture weight)."""
    mix = gaussian_mixture(n, d, components, seed)
    rng = Rng(member_seed)
    lab = mix.labels

    def uniform_over(clusters):
        w = np.isin(lab, clusters).astype(np.float64)
        return w / w.sum()

    ga = np.empty((m, n))
    gb = np.empty((m, n))
    for q in range(m):
        ga[q] = _normalise(uniform_over(_cluster_choice(rng, range(0, 20), 10)))
    for q in range(m):
        base = uniform_over(_cluster_choice(rng, range(0, 20), 10))
        shift = uniform_over(_cluster_choice(rng, range(20, 40), 10))
        gb[q] = _normalise(0.8 * base + 0.2 * shift)
    return Config4(mix, ga, gb)
