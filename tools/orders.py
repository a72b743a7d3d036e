"""Host-side locality orders for experiments (gs_filter_set_order): graph-only recursive BFS
bisection and a 3-D Morton order of the point coordinates. Not on the product path."""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import breadth_first_order, connected_components


def morton3(X: np.ndarray, bits: int = 20) -> np.ndarray:
    X = (X - X.min(0)) / max((X.max(0) - X.min(0)).max(), 1e-300)
    q = (X * ((1 << bits) - 1)).astype(np.uint64)

    def spread(v):
        v = v & np.uint64(0x1fffff)
        v = (v | (v << np.uint64(32))) & np.uint64(0x1f00000000ffff)
        v = (v | (v << np.uint64(16))) & np.uint64(0x1f0000ff0000ff)
        v = (v | (v << np.uint64(8))) & np.uint64(0x100f00f00f00f00f)
        v = (v | (v << np.uint64(4))) & np.uint64(0x10c30c30c30c30c3)
        v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
        return v

    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
    return np.argsort(code, kind="stable").astype(np.int32)


def bisect_order(offs, cols, n: int, leaf: int = 64) -> np.ndarray:
    """Recursive bisection: BFS each part from a pseudo-peripheral vertex, split at the median
    BFS position, recurse; leaves concatenated in order."""
    A = sp.csr_matrix((np.ones(len(cols)), np.asarray(cols), np.asarray(offs)), shape=(n, n))

    def bfs_sub(vs):
        sub = A[vs][:, vs]
        ncomp, lab = connected_components(sub, directed=False)
        seqs = []
        for c in range(ncomp):
            mem = np.where(lab == c)[0]
            s0 = mem[0]
            for _ in range(2):
                s0 = breadth_first_order(sub, s0, directed=False, return_predecessors=False)[-1]
            seqs.append(breadth_first_order(sub, s0, directed=False, return_predecessors=False))
        return vs[np.concatenate(seqs)]

    work = [np.arange(n)]
    final = []
    while work:
        vs = work.pop()
        if vs.size <= leaf:
            final.append(vs)
            continue
        o = bfs_sub(vs)
        h = o.size // 2
        work.append(o[h:])
        work.append(o[:h])
    return np.concatenate(final).astype(np.int32)
