"""Why the 32-bit mode stores fp64's upper word instead of IEEE binary32 (DESIGN.md §4 "Precision";
profiles/r02_fp32_range.md). CPU only: the oracle (fp64, the reference's restated algorithm) against
numpy restatements of the same recurrence and Sinkhorn control in three storage formats, on config 1
as specified at n = 6000 (pairs 1 and 3 of workloads.config1(6000, 16)):
  emu   : fp32 significand (24-bit rounding after every operation), unlimited exponent range;
  f32/s : IEEE binary32 with a per-column power-of-two scale putting the column max at 2^s
          (s = 0, 60, 100 -> 100 / 160 / 220 binary orders of range below the max) and a division
          floor at the bottom of that range.
Prints the L1 marginal error per sweep. usage: python tools/fp32_range_probe.py
"""
import os
import sys
import warnings

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import pyoracle as po  # noqa: E402
from paper_2211_00805_b200 import workloads  # noqa: E402

workloads.set_rng_class(po.Rng)
warnings.simplefilter("ignore")
n = 6000
cfg = workloads.config1(n, 16, seed=1, pair_seed=2)
sel = [1, 3]
mus, nus = cfg.mus[sel], cfg.nus[sel]
A, _ = po.knn_graph(cfg.roll.points, 10, 1, 0.0)
L, lam, _ = po.laplacian(A, 0)
fo = po.Filter(L, 0, lam, 1.0, 30)
S = fo.scaled
b = fo.coeffs


def r24(x):
    m, e = np.frexp(x)
    return np.ldexp(np.round(m * 2.0 ** 24) / 2.0 ** 24, e)


L64 = sp.csr_matrix((S.vals, S.cols, S.offs), shape=(n, n))
L32 = sp.csr_matrix((S.vals.astype(np.float32), S.cols, S.offs), shape=(n, n))
LR = sp.csr_matrix((r24(S.vals), S.cols, S.offs), shape=(n, n))


def cheb(X, mode, shift):
    if mode == "f64":
        T0 = X
        T1 = L64 @ T0 - T0
        acc = b[0] / 2 * T0 + b[1] * T1
        Tm2, Tm1 = T0, T1
        for k in range(2, len(b)):
            Tk = 2 * (L64 @ Tm1 - Tm1) - Tm2
            acc = acc + b[k] * Tk
            Tm2, Tm1 = Tm1, Tk
        return acc
    if mode == "emu":
        R, bb = r24, r24(b)
        T0 = R(X)
        T1 = R(R(LR @ T0) - T0)
        acc = R(R(bb[0] / 2 * T0) + R(bb[1] * T1))
        Tm2, Tm1 = T0, T1
        for k in range(2, len(b)):
            Tk = R(R(2 * R(R(LR @ Tm1) - Tm1)) - Tm2)
            acc = R(acc + R(bb[k] * Tk))
            Tm2, Tm1 = Tm1, Tk
        return acc
    mx = np.max(np.abs(X), axis=0)
    e = np.floor(np.log2(np.where(mx > 0, mx, 1.0)))
    sc = np.ldexp(1.0, (e - shift).astype(int))
    T0 = (X / sc).astype(np.float32)
    T1 = L32 @ T0 - T0
    acc = np.float32(b[0] / 2) * T0 + np.float32(b[1]) * T1
    Tm2, Tm1 = T0, T1
    for k in range(2, len(b)):
        Tk = np.float32(2) * (L32 @ Tm1 - Tm1) - Tm2
        acc = acc + np.float32(b[k]) * Tk
        Tm2, Tm1 = Tm1, Tk
    return acc.astype(np.float64) * sc


def run(mode, shift=0, iters=60):
    M, N = mus.T.copy(), nus.T.copy()
    a = np.full(n, 1.0 / n)[:, None]

    def floor(X):
        if mode != "f32":
            return 1e-300
        return np.maximum(1e-300, 2.0 ** (-100 - shift) * np.max(np.abs(X), 0))

    X = a * np.ones_like(M)
    phi = cheb(X, mode, shift)
    f = floor(X)
    errs = []
    for _ in range(iters):
        V = M / np.maximum(phi, f)
        X = a * V
        psi = cheb(X, mode, shift)
        f = floor(X)
        W = N / np.maximum(psi, f)
        X = a * W
        phi = cheb(X, mode, shift)
        f = floor(X)
        errs.append(np.abs(V * phi - M).sum(0))
    return np.array(errs)


runs = {"fp64 (oracle arithmetic)": run("f64"), "fp32 significand, fp64 range": run("emu")}
for s in (0, 60, 100):
    runs[f"binary32, column max at 2^{s}"] = run("f32", s)
print("sweep | " + " | ".join(runs))
for s in (1, 6, 20, 40, 50, 60):
    print(f"{s} | " + " | ".join(np.array2string(v[s - 1], precision=6) for v in runs.values()))
