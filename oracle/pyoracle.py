"""ctypes front end for the CPU oracle (oracle/liboracle.so) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this module; the
product package (paper_2211_00805_b200) never does. Every wrapper mirrors one entry point of
oracle/geosink_oracle.h, which in turn cites the reference routine it restates.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

ERRC_NAMES = [
    "DimensionMismatch", "DuplicatePoints", "NegativeWeight", "NonPositiveTime",
    "LengthMismatch", "TooLarge", "IndexOutOfRange", "SizeMismatch", "DegenerateInput",
    "InvalidArgument", "KernelNotPositive", "Disconnected", "SolveFailure",
    "NumericalUnderflow", "DegeneratePlan", "IoError",
]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status
        self.code = ERRC_NAMES[status - 1] if 1 <= status <= len(ERRC_NAMES) else "Unknown"


class go_csr(C.Structure):
    _fields_ = [("n", C.c_int), ("nnz", C.c_int64), ("row_offsets", C.POINTER(C.c_int)),
                ("col_indices", C.POINTER(C.c_int)), ("values", C.POINTER(C.c_double))]


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def lib(native: bool = False):
    """Load (building if needed) the oracle. native=True builds -march=native for timing."""
    global _LIB
    name = "liboracle_native.so" if native else "liboracle.so"
    path = os.path.join(_HERE, name)
    if native or _LIB is None:
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", _HERE, "native" if native else "all"], check=True)
        L = C.CDLL(path)
        _declare(L)
        if native:
            return L
        _LIB = L
    return _LIB


def _declare(L):
    L.go_last_error.restype = C.c_char_p
    for nm, ptr in (("go_rng_bits", _up), ("go_rng_uniform", _dp), ("go_rng_normal", _dp)):
        getattr(L, nm).argtypes = [C.c_uint64, C.c_int64, ptr]
    L.go_rng_below.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _up]
    L.go_rng_seed_mix.argtypes = [C.c_uint64, C.c_uint64]
    L.go_rng_seed_mix.restype = C.c_uint64
    L.go_rng_new.restype = C.c_void_p
    L.go_rng_new.argtypes = [C.c_uint64]
    L.go_rng_free.argtypes = [C.c_void_p]
    L.go_rng_next_bits.restype = C.c_uint64
    L.go_rng_next_bits.argtypes = [C.c_void_p]
    L.go_rng_next_uniform.restype = C.c_double
    L.go_rng_next_uniform.argtypes = [C.c_void_p]
    L.go_rng_next_normal.restype = C.c_double
    L.go_rng_next_normal.argtypes = [C.c_void_p]
    L.go_rng_next_below.restype = C.c_uint64
    L.go_rng_next_below.argtypes = [C.c_void_p, C.c_uint64]
    L.go_rng_fill_pattern.argtypes = [C.c_void_p, _dp, C.c_int64, _ip, _dp, _dp, C.c_int]
    L.go_csr_from_triplets.argtypes = [C.c_int, C.c_int64, _ip, _ip, _dp, C.POINTER(go_csr)]
    L.go_csr_from_arrays.argtypes = [C.c_int, C.c_int64, _ip, _ip, _dp, C.POINTER(go_csr)]
    L.go_csr_free.argtypes = [C.POINTER(go_csr)]
    L.go_spmm.argtypes = [C.POINTER(go_csr), _dp, _dp, C.c_int]
    L.go_gershgorin.argtypes = [C.POINTER(go_csr)]
    L.go_gershgorin.restype = C.c_double
    L.go_detdot.argtypes = [_dp, _dp, C.c_int64]
    L.go_detdot.restype = C.c_double
    L.go_knn.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _ip, _dp]
    L.go_knn_rows.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _ip, C.c_int, _ip, _dp]
    L.go_knn_graph.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                               C.POINTER(go_csr), C.POINTER(C.c_double)]
    L.go_laplacian.argtypes = [C.POINTER(go_csr), C.c_int, C.POINTER(go_csr),
                               C.POINTER(C.c_double), C.POINTER(C.c_int)]
    L.go_lambda_max.argtypes = [C.POINTER(go_csr), C.POINTER(C.c_double), C.POINTER(C.c_int)]
    L.go_heat_coefficients.argtypes = [C.c_double, C.c_int, _dp]
    L.go_filter_prepare.argtypes = [C.POINTER(go_csr), C.c_int, C.c_double, C.c_double, C.c_int,
                                    C.POINTER(go_csr), _dp, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
    L.go_filter_apply.argtypes = [C.POINTER(go_csr), _dp, C.c_int, _dp, _dp, C.c_int]
    L.go_euler_system.argtypes = [C.POINTER(go_csr), C.c_double, C.c_int, C.POINTER(go_csr)]
    L.go_euler_apply.argtypes = [C.POINTER(go_csr), C.c_int, _dp, _dp, C.c_int, C.POINTER(C.c_int)]
    L.go_euler_sinkhorn_batch.argtypes = [C.POINTER(go_csr), C.c_int, C.c_double, _dp, _dp, _dp,
                                          C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _dp,
                                          _dp, _dp, _dp, _ip, _ip, _dp, _ip]
    L.go_sinkhorn_batch.argtypes = [C.POINTER(go_csr), _dp, C.c_int, C.c_double, _dp, _dp, _dp,
                                    C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, _dp, _dp,
                                    _dp, _dp, _ip, _ip, _dp, _ip]
    L.go_barycenter.argtypes = [C.POINTER(go_csr), _dp, C.c_int, _dp, _dp, C.c_int,
                                C.c_void_p, C.c_int, C.c_double, _dp, _dp, _dp, _ip, _ip, _dp]
    L.go_squared_distances.argtypes = [_dp, C.c_int, _dp, C.c_int, C.c_int, _dp]
    L.go_dense_sinkhorn.argtypes = [_dp, C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_int,
                                    C.c_double, _dp, _dp, _dp, _dp, _ip, _ip, _dp]


def _check(rc: int, L=None):
    if rc != 0:
        L = L or lib()
        raise OracleError(rc, L.go_last_error().decode())


# --------------------------------------------------------------------------- RNG (rng.hpp)
def rng_normal(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    lib().go_rng_normal(seed, count, out)
    return out


def rng_uniform(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    lib().go_rng_uniform(seed, count, out)
    return out


def rng_bits(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    lib().go_rng_bits(seed, count, out)
    return out


def rng_below(seed: int, bound: int, count: int) -> np.ndarray:
    out = np.empty(count, np.uint64)
    lib().go_rng_below(seed, bound, count, out)
    return out


class Rng:
    """Stateful geosink::Rng (rng.hpp:13-68) on the oracle: the same interface as the engine's
    paper_2211_00805_b200.rng.Rng, so input generators can run without the product library
    (the reference arm of bench.py)."""

    def __init__(self, seed: int):
        self._L = lib()
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self._h = self._L.go_rng_new(self.seed)

    def fork(self, stream: int) -> "Rng":
        return Rng(self.seed_mix(self.seed, stream))

    def bits(self) -> int:
        return int(self._L.go_rng_next_bits(self._h))

    def uniform(self, lo=None, hi=None) -> float:
        u = float(self._L.go_rng_next_uniform(self._h))
        return u if lo is None else lo + (hi - lo) * u

    def normal(self) -> float:
        return float(self._L.go_rng_next_normal(self._h))

    def below(self, n: int) -> int:
        return int(self._L.go_rng_next_below(self._h, n))

    @staticmethod
    def seed_mix(a: int, b: int) -> int:
        return int(lib().go_rng_seed_mix(a & 0xFFFFFFFFFFFFFFFF, b & 0xFFFFFFFFFFFFFFFF))

    def pattern(self, count: int, spec) -> np.ndarray:
        kinds = np.array([{"u": 0, "n": 1, "b": 2}[k] for k, _, _ in spec], np.int32)
        lo = np.array([float(l) for _, l, _ in spec], np.float64)
        hi = np.array([float(h) for _, _, h in spec], np.float64)
        out = np.empty(count, np.float64)
        self._L.go_rng_fill_pattern(self._h, out, count, kinds, lo, hi, len(spec))
        return out

    def normals(self, count: int) -> np.ndarray:
        return self.pattern(count, [("n", 0.0, 1.0)])

    def __del__(self):
        try:
            self._L.go_rng_free(self._h)
        except Exception:
            pass


def ref_rng():
    """The reference's own rng.hpp compiled into oracle/_ref (None when it was not built)."""
    global _REF
    path = os.path.join(_HERE, "_ref", "librefrng.so")
    if _REF is None and os.path.exists(path):
        R = C.CDLL(path)
        for nm, ptr in (("ref_rng_bits", _up), ("ref_rng_uniform", _dp), ("ref_rng_normal", _dp)):
            getattr(R, nm).argtypes = [C.c_uint64, C.c_int64, ptr]
        R.ref_rng_below.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _up]
        R.ref_rng_seed_mix.argtypes = [C.c_uint64, C.c_uint64]
        R.ref_rng_seed_mix.restype = C.c_uint64
        _REF = R
    return _REF


# --------------------------------------------------------------------------- CSR
class CSR:
    """Host CSR owned by numpy (both triangles, rows sorted by column; sparse.hpp:23-61)."""

    def __init__(self, n, offs, cols, vals):
        self.n = int(n)
        self.offs = np.ascontiguousarray(offs, np.int32)
        self.cols = np.ascontiguousarray(cols, np.int32)
        self.vals = np.ascontiguousarray(vals, np.float64)

    @property
    def nnz(self):
        return int(self.cols.size)

    def _struct(self):
        s = go_csr()
        s.n = self.n
        s.nnz = self.nnz
        s.row_offsets = self.offs.ctypes.data_as(C.POINTER(C.c_int))
        s.col_indices = self.cols.ctypes.data_as(C.POINTER(C.c_int))
        s.values = self.vals.ctypes.data_as(C.POINTER(C.c_double))
        return s

    def to_dense(self):
        d = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.offs))
        d[rows, self.cols] = self.vals
        return d

    def coeff(self, i, j):
        lo, hi = self.offs[i], self.offs[i + 1]
        k = np.searchsorted(self.cols[lo:hi], j)
        return float(self.vals[lo + k]) if k < hi - lo and self.cols[lo + k] == j else 0.0


def _adopt(s: go_csr) -> CSR:
    n, nnz = s.n, s.nnz
    offs = np.ctypeslib.as_array(s.row_offsets, shape=(n + 1,)).copy()
    cols = np.ctypeslib.as_array(s.col_indices, shape=(max(nnz, 1),))[:nnz].copy()
    vals = np.ctypeslib.as_array(s.values, shape=(max(nnz, 1),))[:nnz].copy()
    lib().go_csr_free(C.byref(s))
    return CSR(n, offs, cols, vals)


def from_triplets(n, rows, cols, vals) -> CSR:
    rows = np.ascontiguousarray(rows, np.int32)
    cols = np.ascontiguousarray(cols, np.int32)
    vals = np.ascontiguousarray(vals, np.float64)
    s = go_csr()
    _check(lib().go_csr_from_triplets(n, rows.size, rows, cols, vals, C.byref(s)))
    return _adopt(s)


def spmm(m: CSR, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    width = 1 if x.ndim == 1 else x.shape[1]
    y = np.empty_like(x)
    s = m._struct()
    _check(lib().go_spmm(C.byref(s), x, y, width))
    return y


def gershgorin(m: CSR) -> float:
    s = m._struct()
    return lib().go_gershgorin(C.byref(s))


def detdot(x, y) -> float:
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return lib().go_detdot(x, y, x.size)


# --------------------------------------------------------------------------- graph
def knn(points, k):
    pts = np.ascontiguousarray(points, np.float64)
    n, d = pts.shape
    nb = np.empty((n, k), np.int32)
    eps = np.empty(n, np.float64)
    _check(lib().go_knn(pts, n, d, k, nb, eps))
    return nb, eps


def knn_rows(points, k, rows):
    pts = np.ascontiguousarray(points, np.float64)
    n, d = pts.shape
    rows = np.ascontiguousarray(rows, np.int32)
    nb = np.empty((rows.size, k), np.int32)
    eps = np.empty(rows.size, np.float64)
    _check(lib().go_knn_rows(pts, n, d, k, rows, rows.size, nb, eps))
    return nb, eps


def knn_graph(points, k, kernel=0, param=40.0):
    pts = np.ascontiguousarray(points, np.float64)
    n, d = pts.shape
    s = go_csr()
    sigma = C.c_double(0.0)
    _check(lib().go_knn_graph(pts, n, d, k, kernel, param, C.byref(s), C.byref(sigma)))
    return _adopt(s), sigma.value


def laplacian(A: CSR, kind: int):
    s = A._struct()
    out = go_csr()
    lam = C.c_double(0.0)
    rounds = C.c_int(0)
    _check(lib().go_laplacian(C.byref(s), kind, C.byref(out), C.byref(lam), C.byref(rounds)))
    return _adopt(out), lam.value, rounds.value


def lambda_max(L: CSR):
    s = L._struct()
    lam = C.c_double(0.0)
    rounds = C.c_int(0)
    _check(lib().go_lambda_max(C.byref(s), C.byref(lam), C.byref(rounds)))
    return lam.value, rounds.value


# --------------------------------------------------------------------------- heat
def heat_coefficients(t, degree):
    b = np.empty(degree + 1, np.float64)
    _check(lib().go_heat_coefficients(t, degree, b))
    return b


class Filter:
    """heat.cpp:72-131 restated: scaled Laplacian + coefficients + the batched recurrence."""

    def __init__(self, L: CSR, kind: int, lambda_bound: float, t: float, degree: int):
        s = L._struct()
        out = go_csr()
        self.coeffs = np.empty(degree + 1, np.float64)
        scale = C.c_double(0.0)
        teff = C.c_double(0.0)
        _check(lib().go_filter_prepare(C.byref(s), kind, lambda_bound, t, degree, C.byref(out),
                                       self.coeffs, C.byref(scale), C.byref(teff)))
        self.scaled = _adopt(out)
        self.scale, self.t_eff, self.t, self.degree, self.kind = scale.value, teff.value, t, degree, kind
        self.n = L.n

    def apply(self, X: np.ndarray) -> np.ndarray:
        X = np.ascontiguousarray(X, np.float64)
        width = 1 if X.ndim == 1 else X.shape[1]
        Y = np.empty_like(X)
        s = self.scaled._struct()
        _check(lib().go_filter_apply(C.byref(s), self.coeffs, self.degree, X, Y, width))
        return Y


def euler_system(L: CSR, t: float, steps: int) -> CSR:
    """heat.cpp:133-162: I + (t/steps) L."""
    s = L._struct()
    out = go_csr()
    _check(lib().go_euler_system(C.byref(s), float(t), int(steps), C.byref(out)))
    return _adopt(out)


def euler_apply(system: CSR, steps: int, X: np.ndarray):
    """heat.cpp:166-219 (lockstep CG); X (n,) or row-major (n, B). Returns (Y, iterations of the
    last solve)."""
    X = np.ascontiguousarray(X, np.float64)
    width = 1 if X.ndim == 1 else X.shape[1]
    Y = np.empty_like(X)
    it = C.c_int(0)
    s = system._struct()
    _check(lib().go_euler_apply(C.byref(s), int(steps), X, Y, width, C.byref(it)))
    return Y, it.value


def euler_sinkhorn_batch(system: CSR, steps: int, t: float, a, mus, nus, max_iter=500, tol=1e-6,
                         flags=0, single_style=False, L=None):
    """transport.cpp:257-269: sinkhorn_many over EulerHeat (system from euler_system)."""
    L = L or lib()
    mus = np.ascontiguousarray(np.atleast_2d(mus), np.float64)
    nus = np.ascontiguousarray(np.atleast_2d(nus), np.float64)
    a = np.ascontiguousarray(a, np.float64)
    P, n = mus.shape
    v, w = np.zeros((P, n)), np.zeros((P, n))
    cost, kl, err = np.zeros(P), np.zeros(P), np.zeros(P)
    iters, conv = np.zeros(P, np.int32), np.zeros(P, np.int32)
    fail_info = np.zeros(2, np.int32)
    s = system._struct()
    rc = L.go_euler_sinkhorn_batch(C.byref(s), int(steps), float(t), a, mus, nus, P, max_iter, tol,
                                   flags, int(single_style), v, w, cost, kl, iters, conv, err,
                                   fail_info)
    _check(rc, L)
    return dict(v=v, w=w, cost=cost, kl=kl, iterations=iters, converged=conv.astype(bool),
                marginal_error=err)


def sinkhorn_batch(f: Filter, a, mus, nus, max_iter=500, tol=1e-6, flags=0, single_style=False,
                   L=None):
    """transport.cpp:144-239; mus/nus shaped (P, n). Returns a dict of per-pair results."""
    L = L or lib()
    mus = np.ascontiguousarray(np.atleast_2d(mus), np.float64)
    nus = np.ascontiguousarray(np.atleast_2d(nus), np.float64)
    a = np.ascontiguousarray(a, np.float64)
    P, n = mus.shape
    v = np.zeros((P, n))
    w = np.zeros((P, n))
    cost = np.zeros(P)
    kl = np.zeros(P)
    iters = np.zeros(P, np.int32)
    conv = np.zeros(P, np.int32)
    err = np.zeros(P)
    fail_info = np.zeros(2, np.int32)
    s = f.scaled._struct()
    rc = L.go_sinkhorn_batch(C.byref(s), f.coeffs, f.degree, f.t, a, mus, nus, P, max_iter, tol,
                             flags, int(single_style), v, w, cost, kl, iters, conv, err, fail_info)
    _check(rc, L)
    return dict(v=v, w=w, cost=cost, kl=kl, iterations=iters, converged=conv.astype(bool),
                marginal_error=err)


def barycenter(f: Filter, a, members, alphas=None, max_iter=500, tol=1e-6, L=None):
    """barycenter.cpp:45-99; members shaped (m, n)."""
    L = L or lib()
    members = np.ascontiguousarray(np.atleast_2d(members), np.float64)
    a = np.ascontiguousarray(a, np.float64)
    m, n = members.shape
    al = None if alphas is None else np.ascontiguousarray(alphas, np.float64)
    bary = np.zeros(n)
    V = np.zeros((m, n))
    W = np.zeros((m, n))
    it = np.zeros(1, np.int32)
    conv = np.zeros(1, np.int32)
    err = np.zeros(1)
    s = f.scaled._struct()
    rc = L.go_barycenter(C.byref(s), f.coeffs, f.degree, a, members, m,
                         None if al is None else al.ctypes.data, max_iter, tol, bary, V, W, it,
                         conv, err)
    _check(rc, L)
    return dict(barycenter=bary, V=V, W=W, iterations=int(it[0]), converged=bool(conv[0]),
                marginal_error=float(err[0]))


def squared_distances(X, Y, L=None):
    """bench.cpp:32-39 (go_squared_distances)."""
    L = L or lib()
    X = np.ascontiguousarray(X, np.float64)
    Y = np.ascontiguousarray(Y, np.float64)
    out = np.empty((X.shape[0], Y.shape[0]))
    _check(L.go_squared_distances(X, X.shape[0], Y, Y.shape[0], X.shape[1], out), L)
    return out


def dense_sinkhorn(cost, mu, nu, lam, max_iter=500, tol=1e-6, L=None):
    """transport.cpp:271-311 (go_dense_sinkhorn)."""
    L = L or lib()
    cost = np.ascontiguousarray(cost, np.float64)
    r, c = cost.shape
    mu = np.ascontiguousarray(mu, np.float64)
    nu = np.ascontiguousarray(nu, np.float64)
    v, w = np.empty(r), np.empty(c)
    cs, kl, err = np.empty(1), np.empty(1), np.empty(1)
    it, cv = np.empty(1, np.int32), np.empty(1, np.int32)
    _check(L.go_dense_sinkhorn(cost, r, c, mu, nu, float(lam), int(max_iter), float(tol), v, w, cs,
                               kl, it, cv, err), L)
    return {"v": v, "w": w, "cost": float(cs[0]), "kl": float(kl[0]), "iterations": int(it[0]),
            "converged": bool(cv[0]), "marginal_error": float(err[0])}
