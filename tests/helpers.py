"""Test fixtures restated from the reference test utilities (tests/test_util.hpp:13-57,
tests/acceptance/acceptance.cpp:47-68), seeded through geosink::Rng semantics."""
from __future__ import annotations

import numpy as np

import pyoracle as po
from paper_2211_00805_b200.rng import Rng


def random_connected_graph(n, seed, chord_fraction=1.0):
    """test_util.hpp:20-39 -> (rows, cols, vals) triplets."""
    rng = Rng(seed)
    edges = set()
    rows, cols, vals = [], [], []
    for i in range(n):
        j = (i + 1) % n
        e = (min(i, j), max(i, j))
        edges.add(e)
        rows.append(e[0]); cols.append(e[1]); vals.append(rng.uniform(0.3, 1.0))
    for _ in range(int(chord_fraction * n)):
        i = rng.below(n)
        j = rng.below(n)
        w = rng.uniform(0.2, 0.8)
        e = (min(i, j), max(i, j))
        if i == j or e in edges:
            continue
        edges.add(e)
        rows.append(e[0]); cols.append(e[1]); vals.append(w)
    return np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals)


def acceptance_graph(n, seed):
    """acceptance.cpp:47-62."""
    rng = Rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i); cols.append((i + 1) % n); vals.append(rng.uniform(0.3, 1.0))
    seen = set()
    for _ in range(n):
        i = rng.below(n)
        j = rng.below(n)
        w = rng.uniform(0.2, 0.8)
        lo, hi = min(i, j), max(i, j)
        if i == j or abs(i - j) == 1 or (lo == 0 and hi == n - 1):
            continue
        if (lo, hi) in seen:
            continue
        seen.add((lo, hi))
        rows.append(lo); cols.append(hi); vals.append(w)
    return np.array(rows, np.int32), np.array(cols, np.int32), np.array(vals)


def path_graph(n, weight=1.0):
    r = np.arange(n - 1, dtype=np.int32)
    return r, r + 1, np.full(n - 1, weight)


def random_signal(n, rng: Rng):
    return np.array([rng.normal() for _ in range(n)])


def from_weights(w):
    w = np.array(w, np.float64)
    w /= w.sum()
    w /= w.sum()
    return w


def random_distribution(n, rng: Rng):
    return from_weights([rng.uniform() + 1e-3 for _ in range(n)])


def oracle_filter(rows, cols, vals, n, kind, t, K):
    A = po.from_triplets(n, rows, cols, vals)
    L, lam, _ = po.laplacian(A, kind)
    return po.Filter(L, kind, lam, t, K)


def engine_filter(rows, cols, vals, n, kind, t, K, ctx=None):
    import paper_2211_00805_b200 as gs
    A = gs.SparseSymMatrix.from_arrays(n, rows, cols, vals, ctx) if ctx is not None else \
        gs.SparseSymMatrix.from_arrays(n, rows, cols, vals)
    lap = gs.laplacian(A, gs.LaplacianKind(kind))
    return gs.HeatFilter(lap, t, K), lap


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def partition_plan(offs, cols, vals, order, nparts):
    """numpy restatement of the row-partition rules of gs_part.cu: vertices renumbered by
    `order` (order[new] = old), nnz-balanced contiguous ranges, halo rows sorted by position
    (hence by owner), send rows per destination ascending, local CSR with entries kept in the
    original order and columns renumbered to [0, nl) local / nl + halo index."""
    offs, cols, vals = np.asarray(offs), np.asarray(cols), np.asarray(vals)
    order = np.asarray(order)
    n = order.size
    newpos = np.empty(n, np.int64)
    newpos[order] = np.arange(n)
    poffs = np.concatenate([[0], np.cumsum(np.diff(offs)[order])])
    nnz = int(poffs[-1])
    bounds = [0] + [int(np.searchsorted(poffs, nnz * p // nparts, side="left"))
                    for p in range(1, nparts)] + [n]
    owner = np.searchsorted(np.array(bounds), np.arange(n), side="right") - 1
    parts = []
    for p in range(nparts):
        rb, re = bounds[p], bounds[p + 1]
        halo, sends = set(), [set() for _ in range(nparts)]
        for r in range(rb, re):
            o = order[r]
            for c in newpos[cols[offs[o]:offs[o + 1]]]:
                if not rb <= c < re:
                    halo.add(int(c))
                    sends[owner[c]].add(r - rb)
        halo = np.array(sorted(halo), np.int64)
        hidx = {int(c): i for i, c in enumerate(halo)}
        lo_offs, lo_cols, lo_vals = [0], [], []
        for r in range(rb, re):
            o = order[r]
            for c, v in zip(newpos[cols[offs[o]:offs[o + 1]]], vals[offs[o]:offs[o + 1]]):
                lo_cols.append(c - rb if rb <= c < re else (re - rb) + hidx[int(c)])
                lo_vals.append(v)
            lo_offs.append(len(lo_cols))
        recv = np.bincount(owner[halo], minlength=nparts) if halo.size else np.zeros(nparts, int)
        nl = re - rb
        bnd = [i for i in range(nl) if (np.array(lo_cols[lo_offs[i]:lo_offs[i + 1]]) >= nl).any()]
        lo_b = [i for i in bnd if i < nl // 2]
        hi_b = [i for i in bnd if i >= nl // 2]
        ilo = (max(lo_b) + 1) if lo_b else 0
        ihi = max(min(hi_b) if hi_b else nl, ilo)
        parts.append(dict(rb=rb, re=re, vertices=order[rb:re], nh=int(halo.size), halo=halo,
                          interior=(ilo, ihi),
                          recv=recv, send_rows=[np.array(sorted(s), np.int64) for s in sends],
                          send=np.array([len(s) for s in sends]),
                          offs=np.array(lo_offs), cols=np.array(lo_cols, np.int64),
                          vals=np.array(lo_vals)))
    return parts
