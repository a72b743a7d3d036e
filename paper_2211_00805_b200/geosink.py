"""Python mirror of the reference `geosink` public API over the B200 engine's C ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/geosink/*.hpp:
  SparseSymMatrix            sparse.hpp:23-61        (device-resident CSR handle)
  knn_alpha_decay_graph      graph.hpp:26-33
  laplacian / GraphLaplacian graph.hpp:10-37
  estimate_lambda_max        graph.hpp:39-42
  heat_chebyshev_coefficients heat.hpp:12-19
  HeatFilter                 heat.hpp:21-54
  Distribution, SinkhornParams, TransportResult   transport.hpp:14-49
  geodesic_sinkhorn[_batch]  transport.hpp:51-69
  DistributionFamily, BarycenterResult, sinkhorn_barycenter, barycentric_distance
                             barycenter.hpp:11-42
Errors surface as `Error` carrying the reference `errc` name (errors.hpp:10-85). Every compute
call runs on the GPU through libgeosink_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _capi

# ---------------------------------------------------------------------------------- errors
ERRC = [
    "dimension_mismatch", "duplicate_points", "negative_weight", "non_positive_time",
    "length_mismatch", "too_large", "index_out_of_range", "size_mismatch", "degenerate_input",
    "invalid_argument", "kernel_not_positive", "disconnected", "solve_failure",
    "numerical_underflow", "degenerate_plan", "io_error",
]
errc = enum.IntEnum("errc", {name: i for i, name in enumerate(ERRC)})
_NUMERICAL = {errc.kernel_not_positive, errc.disconnected, errc.solve_failure,
              errc.numerical_underflow, errc.degenerate_plan, errc.io_error}


class Error(RuntimeError):
    """geosink::Error (errors.hpp:54-79): message is "<ErrcName>: <what>"."""

    def __init__(self, code, what: str):
        super().__init__(what)
        self.code = code

    def is_validation(self) -> bool:
        return self.code not in _NUMERICAL if isinstance(self.code, errc) else False

    def is_io(self) -> bool:
        return self.code == errc.io_error


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside the engine."""


def _raise(rc: int, ctx) -> None:
    if rc == 0:
        return
    msg = _capi.load().gs_last_error(ctx).decode() if ctx else ""
    if 1 <= rc <= len(ERRC):
        raise Error(errc(rc - 1), msg)
    raise DeviceError(f"engine status {rc}: {msg}")


# ---------------------------------------------------------------------------------- context
class Context:
    """One device + one CUDA stream (gs_ctx). A process-wide default exists per device."""

    _defaults = {}
    _lock = threading.Lock()

    def __init__(self, device: int = 0):
        lib = _capi.load()
        h = C.c_void_p()
        rc = lib.gs_ctx_create(device, C.byref(h))
        if rc != 0:
            raise _capi.EngineUnavailable(
                f"gs_ctx_create(device={device}) failed with status {rc}: no usable CUDA device")
        self.handle = h
        self.device = device
        self.lib = lib

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        with cls._lock:
            ctx = cls._defaults.get(device)
            if ctx is None:
                ctx = cls._defaults[device] = Context(device)
            return ctx

    def check(self, rc: int):
        _raise(rc, self.handle)

    def synchronize(self):
        self.check(self.lib.gs_ctx_synchronize(self.handle))

    def set_stream(self, stream_ptr: int | None):
        self.check(self.lib.gs_ctx_set_stream(self.handle, stream_ptr))

    def set_timing(self, on, period: int = 1):
        """Event-time engine launches per class; `period` > 1 samples every Nth launch."""
        self.check(self.lib.gs_ctx_set_timing(self.handle, (period if period > 1 else 1) if on else 0))

    def timing(self, cls: int):
        n = C.c_int64()
        ms = C.c_double()
        self.check(self.lib.gs_ctx_timing(self.handle, cls, C.byref(n), C.byref(ms)))
        return n.value, ms.value

    def launch_count(self) -> int:
        return int(self.lib.gs_ctx_launch_count(self.handle))

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.gs_ctx_destroy(self.handle)
        except Exception:
            pass


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx or Context.default()


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------------- sparse
@dataclass
class Triplet:
    row: int
    col: int
    value: float


class SparseSymMatrix:
    """Device-resident symmetric CSR (sparse.hpp:23-61). Host accessors download on demand."""

    def __init__(self, handle, ctx: Context):
        self._h = handle
        self._ctx = ctx
        n = C.c_int()
        nnz = C.c_int64()
        ctx.lib.gs_graph_info(handle, C.byref(n), C.byref(nnz))
        self._n, self._nnz = n.value, nnz.value
        self._host = None
        self._owned = True

    @classmethod
    def _borrow(cls, handle, ctx, owner):
        m = cls(handle, ctx)
        m._owned = False
        m._owner = owner
        return m

    @staticmethod
    def from_triplets(n: int, entries, ctx: Optional[Context] = None) -> "SparseSymMatrix":
        """sparse.cpp:15-53. `entries`: iterable of (row, col, value) or Triplet."""
        ctx = _ctx(ctx)
        ent = list(entries)
        rows = np.array([e.row if isinstance(e, Triplet) else e[0] for e in ent], np.int32)
        cols = np.array([e.col if isinstance(e, Triplet) else e[1] for e in ent], np.int32)
        vals = np.array([e.value if isinstance(e, Triplet) else e[2] for e in ent], np.float64)
        return SparseSymMatrix.from_arrays(n, rows, cols, vals, ctx)

    @staticmethod
    def from_arrays(n, rows, cols, vals, ctx: Optional[Context] = None) -> "SparseSymMatrix":
        ctx = _ctx(ctx)
        rows = np.ascontiguousarray(rows, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        vals = _f64(vals)
        h = C.c_void_p()
        ctx.check(ctx.lib.gs_graph_from_triplets(ctx.handle, int(n), rows.size, _ptr(rows),
                                                 _ptr(cols), _ptr(vals), _capi.GS_MEM_HOST,
                                                 C.byref(h)))
        return SparseSymMatrix(h, ctx)

    @staticmethod
    def from_csr(n, offs, cols, vals, ctx: Optional[Context] = None) -> "SparseSymMatrix":
        ctx = _ctx(ctx)
        offs = np.ascontiguousarray(offs, np.int32)
        cols = np.ascontiguousarray(cols, np.int32)
        vals = _f64(vals)
        h = C.c_void_p()
        ctx.check(ctx.lib.gs_graph_from_csr(ctx.handle, int(n), cols.size, _ptr(offs), _ptr(cols),
                                            _ptr(vals), _capi.GS_MEM_HOST, C.byref(h)))
        return SparseSymMatrix(h, ctx)

    def size(self) -> int:
        return self._n

    def stored_entries(self) -> int:
        return self._nnz

    def _download(self):
        if self._host is None:
            offs = np.empty(self._n + 1, np.int32)
            cols = np.empty(max(self._nnz, 1), np.int32)
            vals = np.empty(max(self._nnz, 1), np.float64)
            self._ctx.check(self._ctx.lib.gs_graph_download(self._ctx.handle, self._h, _ptr(offs),
                                                            _ptr(cols), _ptr(vals),
                                                            _capi.GS_MEM_HOST))
            self._host = (offs, cols[: self._nnz], vals[: self._nnz])
        return self._host

    def row_offsets(self):
        return self._download()[0]

    def col_indices(self):
        return self._download()[1]

    def values(self):
        return self._download()[2]

    def coeff(self, i: int, j: int) -> float:
        if not (0 <= i < self._n and 0 <= j < self._n):
            raise Error(errc.index_out_of_range, "IndexOutOfRange: coeff index")
        offs, cols, vals = self._download()
        lo, hi = offs[i], offs[i + 1]
        k = np.searchsorted(cols[lo:hi], j)
        return float(vals[lo + k]) if k < hi - lo and cols[lo + k] == j else 0.0

    def to_dense(self) -> np.ndarray:
        offs, cols, vals = self._download()
        d = np.zeros((self._n, self._n))
        d[np.repeat(np.arange(self._n), np.diff(offs)), cols] = vals
        return d

    def multiply(self, x) -> np.ndarray:
        """y = A x (sparse.cpp:70-99); x is (n,) or row-major (n, B) as RowMajorXd."""
        x = _f64(x)
        if x.shape[0] != self._n:
            raise Error(errc.length_mismatch, "LengthMismatch: matvec size")
        cols = _f64(x.reshape(self._n, -1).T)  # B contiguous n-vectors
        out = np.empty_like(cols)
        self._ctx.check(self._ctx.lib.gs_graph_multiply(self._ctx.handle, self._h, _ptr(cols),
                                                        _ptr(out), cols.shape[0],
                                                        _capi.GS_MEM_HOST))
        return out.T.reshape(x.shape).copy()

    def gershgorin_bound(self) -> float:
        out = C.c_double()
        self._ctx.check(self._ctx.lib.gs_graph_gershgorin(self._ctx.handle, self._h, C.byref(out)))
        return out.value

    def max_abs(self) -> float:
        v = self.values()
        return float(np.abs(v).max()) if v.size else 0.0

    def __del__(self):
        try:
            if self._owned and self._h:
                self._ctx.lib.gs_graph_destroy(self._h)
        except Exception:
            pass


# ---------------------------------------------------------------------------------- graph
class LaplacianKind(enum.IntEnum):
    combinatorial = 0
    normalized = 1


def laplacian_kind_from_string(s: str) -> LaplacianKind:
    if s == "combinatorial":
        return LaplacianKind.combinatorial
    if s == "normalized":
        return LaplacianKind.normalized
    raise Error(errc.invalid_argument, f"InvalidArgument: unknown laplacian kind '{s}'")


@dataclass
class GraphLaplacian:
    matrix: SparseSymMatrix
    kind: LaplacianKind = LaplacianKind.combinatorial
    lambda_max_bound: float = 0.0
    power_rounds: int = 0  # engine diagnostic: power-iteration rounds, -1 = Gershgorin fallback

    def size(self) -> int:
        return self.matrix.size()


def _points(points) -> np.ndarray:
    pts = _f64(points)
    if pts.ndim == 1:
        pts = pts.reshape(-1, 1)
    return pts


def select_knn(points, k: int, ctx: Optional[Context] = None):
    """graph.cpp:30-71: (neighbours n x k ascending by (d^2, index), eps_k)."""
    ctx = _ctx(ctx)
    pts = _points(points)
    n, d = pts.shape
    nb = np.empty((n, k), np.int32)
    eps = np.empty(n, np.float64)
    ctx.check(ctx.lib.gs_knn(ctx.handle, _ptr(pts), n, d, k, _capi.GS_MEM_HOST, _ptr(nb), _ptr(eps)))
    return nb, eps


def knn_alpha_decay_graph(points, k: int, alpha: float,
                          ctx: Optional[Context] = None) -> SparseSymMatrix:
    """graph.cpp:75-108."""
    ctx = _ctx(ctx)
    pts = _points(points)
    n, d = pts.shape
    h = C.c_void_p()
    ctx.check(ctx.lib.gs_knn_graph(ctx.handle, _ptr(pts), n, d, int(k), 0, float(alpha),
                                   _capi.GS_MEM_HOST, C.byref(h), None))
    return SparseSymMatrix(h, ctx)


def knn_gaussian_graph(points, k: int, ctx: Optional[Context] = None):
    """BASELINE extension: w = exp(-d^2 / sigma^2), sigma = median k-NN bandwidth.
    Returns (SparseSymMatrix, sigma)."""
    ctx = _ctx(ctx)
    pts = _points(points)
    n, d = pts.shape
    h = C.c_void_p()
    sigma = C.c_double()
    ctx.check(ctx.lib.gs_knn_graph(ctx.handle, _ptr(pts), n, d, int(k), 1, 0.0, _capi.GS_MEM_HOST,
                                   C.byref(h), C.byref(sigma)))
    return SparseSymMatrix(h, ctx), sigma.value


def laplacian(A: SparseSymMatrix, kind: LaplacianKind) -> GraphLaplacian:
    """graph.cpp:110-165."""
    ctx = A._ctx
    h = C.c_void_p()
    lam = C.c_double()
    rounds = C.c_int()
    ctx.check(ctx.lib.gs_laplacian(ctx.handle, A._h, int(kind), C.byref(h), C.byref(lam),
                                   C.byref(rounds)))
    return GraphLaplacian(SparseSymMatrix(h, ctx), LaplacianKind(int(kind)), lam.value, rounds.value)


def estimate_lambda_max(L: SparseSymMatrix) -> float:
    """graph.cpp:167-194."""
    ctx = L._ctx
    lam = C.c_double()
    rounds = C.c_int()
    ctx.check(ctx.lib.gs_lambda_max(ctx.handle, L._h, C.byref(lam), C.byref(rounds)))
    return lam.value


# ---------------------------------------------------------------------------------- heat
def heat_chebyshev_coefficients(t: float, degree: int, ctx: Optional[Context] = None) -> np.ndarray:
    """heat.cpp:34-70, computed on the device."""
    ctx = _ctx(ctx)
    if degree < 1:
        raise Error(errc.invalid_argument, "InvalidArgument: Chebyshev degree must be >= 1")
    out = np.empty(degree + 1, np.float64)
    ctx.check(ctx.lib.gs_heat_coefficients(ctx.handle, float(t), int(degree), _ptr(out)))
    return out


class HeatFilter:
    """heat.hpp:25-54: p_K(L_s) with L_s = scale * L on the device."""

    def __init__(self, laplacian: GraphLaplacian, t: float, degree: int):
        ctx = laplacian.matrix._ctx
        self._ctx = ctx
        h = C.c_void_p()
        ctx.check(ctx.lib.gs_filter_create(ctx.handle, laplacian.matrix._h, int(laplacian.kind),
                                           float(laplacian.lambda_max_bound), float(t),
                                           int(degree), C.byref(h)))
        self._h = h
        n = C.c_int()
        tt, te, sc = C.c_double(), C.c_double(), C.c_double()
        dg, kd = C.c_int(), C.c_int()
        ctx.lib.gs_filter_info(h, C.byref(n), C.byref(tt), C.byref(te), C.byref(sc), C.byref(dg),
                               C.byref(kd))
        self._n, self._t, self._teff, self._scale = n.value, tt.value, te.value, sc.value
        self._degree, self._kind = dg.value, LaplacianKind(kd.value)
        self._coeff = np.empty(self._degree + 1, np.float64)
        ctx.lib.gs_filter_coefficients(h, _ptr(self._coeff))

    def size(self) -> int:
        return self._n

    def time(self) -> float:
        return self._t

    def effective_time(self) -> float:
        return self._teff

    def scale(self) -> float:
        return self._scale

    def degree(self) -> int:
        return self._degree

    def kind(self) -> LaplacianKind:
        return self._kind

    def coefficients(self) -> np.ndarray:
        return self._coeff.copy()

    def scaled_laplacian(self) -> SparseSymMatrix:
        return SparseSymMatrix._borrow(self._ctx.lib.gs_filter_scaled(self._h), self._ctx, self)

    def vertex_order(self) -> np.ndarray:
        """Engine diagnostic: internal locality order (order[new] = old)."""
        out = np.empty(self._n, np.int32)
        self._ctx.check(self._ctx.lib.gs_filter_order(self._ctx.handle, self._h, _ptr(out),
                                                      _capi.GS_MEM_HOST))
        return out

    def set_vertex_order(self, order, layout: int = 0) -> None:
        """Engine tuning: replace the locality order of a layout (0: wide column groups, 1: narrow
        ones) with order[new] = old. Results are unchanged; only gather locality moves."""
        o = np.ascontiguousarray(order, np.int32)
        if o.shape != (self._n,):
            raise Error(errc.invalid_argument, "order must have n entries")
        self._ctx.check(self._ctx.lib.gs_filter_set_order(self._ctx.handle, self._h, int(layout),
                                                          _ptr(o), _capi.GS_MEM_HOST))

    def apply(self, f, fp32: bool = False) -> np.ndarray:
        """heat.cpp:98-131: (n,) vector or row-major (n, B) signals. fp32=True runs the optional
        fp32 mode (vectors and L_s in fp32; results returned as float64)."""
        x = _f64(f)
        if x.shape[0] != self._n:
            raise Error(errc.length_mismatch, "LengthMismatch: signal length")
        cols = _f64(x.reshape(self._n, -1).T)
        out = np.empty_like(cols)
        self._ctx.check(self._ctx.lib.gs_filter_apply_ex(self._ctx.handle, self._h, _ptr(cols),
                                                         _ptr(out), cols.shape[0],
                                                         _capi.GS_MEM_HOST,
                                                         _capi.GS_FLAG_FP32 if fp32 else 0))
        return out.T.reshape(x.shape).copy()

    def __del__(self):
        try:
            if self._h:
                self._ctx.lib.gs_filter_destroy(self._h)
        except Exception:
            pass


class EulerHeat:
    """heat.hpp:60-82: implicit Euler, `steps` solves of (I + (t/steps) L) x = b. Solver
    "automatic" (the reference's default) factorises directly below n = 4000 (the reference: sparse
    LDLT; the device: dense Cholesky and its inverse factor, the same solution up to rounding) and
    runs the reference's lockstep conjugate gradient above; "direct" / "lockstep_cg" force one."""

    _SOLVERS = {"automatic": 0, "direct": 1, "lockstep_cg": 2}

    def __init__(self, laplacian: GraphLaplacian, t: float, steps: int, solver: str = "automatic"):
        if solver not in self._SOLVERS:
            raise Error(errc.invalid_argument, "InvalidArgument: unknown solver")
        self._ctx = laplacian.matrix._ctx
        self._n = laplacian.size()
        h = C.c_void_p()
        self._ctx.check(self._ctx.lib.gs_euler_create_ex(self._ctx.handle, laplacian.matrix._h,
                                                         float(t), int(steps), self._SOLVERS[solver],
                                                         C.byref(h)))
        self._h = h
        self._t, self._steps = float(t), int(steps)
        self.last_iterations = 0  # engine diagnostic: CG iterations of the last solve

    def size(self) -> int:
        return self._n

    def steps(self) -> int:
        return self._steps

    def time(self) -> float:
        return self._t

    def system(self) -> SparseSymMatrix:
        """I + (t/steps) L (heat.hpp:80)."""
        return SparseSymMatrix._borrow(self._ctx.lib.gs_euler_system(self._h), self._ctx, self)

    def apply(self, f) -> np.ndarray:
        """heat.cpp:203-214: (n,) vector or row-major (n, B) signals."""
        x = _f64(f)
        if x.shape[0] != self._n:
            raise Error(errc.length_mismatch, "LengthMismatch: signal length")
        cols = _f64(x.reshape(self._n, -1).T)
        out = np.empty_like(cols)
        it = C.c_int()
        self._ctx.check(self._ctx.lib.gs_euler_apply(self._ctx.handle, self._h, _ptr(cols),
                                                     _ptr(out), cols.shape[0], _capi.GS_MEM_HOST,
                                                     C.byref(it)))
        self.last_iterations = it.value
        return out.T.reshape(x.shape).copy()

    def __del__(self):
        try:
            if self._h:
                self._ctx.lib.gs_euler_destroy(self._h)
        except Exception:
            pass


def apply_euler(laplacian: GraphLaplacian, t: float, steps: int, f) -> np.ndarray:
    """heat.cpp:216-219 (one-shot wrapper)."""
    return EulerHeat(laplacian, t, steps).apply(f)


# ---------------------------------------------------------------------------------- transport
class Distribution:
    """transport.hpp:15-27."""

    def __init__(self, weights=None, validate: bool = True):
        self.weights = _f64(weights) if weights is not None else np.zeros(0)
        if weights is not None and validate:
            self.validate()

    @staticmethod
    def uniform(n: int) -> "Distribution":
        if n < 1:
            raise Error(errc.invalid_argument, "InvalidArgument: empty support")
        return Distribution(np.full(n, 1.0 / n))

    @staticmethod
    def indicator(n: int, vertices: Sequence[int]) -> "Distribution":
        if len(vertices) == 0:
            raise Error(errc.invalid_argument, "InvalidArgument: empty indicator set")
        w = np.zeros(n)
        for v in vertices:
            if not 0 <= v < n:
                raise Error(errc.index_out_of_range, "IndexOutOfRange: indicator vertex out of range")
            w[v] += 1.0
        return Distribution(w / w.sum())

    @staticmethod
    def from_weights(w) -> "Distribution":
        w = _f64(w).copy()
        if w.size < 1:
            raise Error(errc.invalid_argument, "InvalidArgument: empty weight vector")
        if not (w >= 0.0).all():
            raise Error(errc.invalid_argument, "InvalidArgument: weights must be non-negative")
        total = w.sum()
        if not (total > 0.0 and math.isfinite(total)):
            raise Error(errc.invalid_argument, "InvalidArgument: weights must have positive mass")
        w /= total
        w /= w.sum()
        return Distribution(w)

    def size(self) -> int:
        return int(self.weights.size)

    def validate(self) -> None:
        w = self.weights
        if w.size < 1:
            raise Error(errc.length_mismatch, "LengthMismatch: empty distribution")
        if not np.isfinite(w).all():
            raise Error(errc.invalid_argument, "InvalidArgument: non-finite weights")
        if not (w >= 0.0).all():
            raise Error(errc.invalid_argument, "InvalidArgument: negative weights")
        if not abs(w.sum() - 1.0) <= 1e-12:
            raise Error(errc.invalid_argument, "InvalidArgument: distribution must sum to 1")


@dataclass
class SinkhornParams:
    max_iter: int = 500
    tol: float = 1e-6


@dataclass
class TransportResult:
    v: np.ndarray = field(default_factory=lambda: np.zeros(0))
    w: np.ndarray = field(default_factory=lambda: np.zeros(0))
    cost: float = 0.0
    kl: float = 0.0
    lambda_: float = 0.0
    iterations: int = 0
    converged: bool = False
    marginal_error: float = math.inf

    def kl_form_cost(self) -> float:
        return math.sqrt(self.lambda_ * max(0.0, 1.0 + self.kl))

    def normalized_cost(self) -> float:
        return 2.0 * self.kl_form_cost()

    def dual_cost(self) -> float:
        return self.lambda_ * (1.0 + self.kl)


def _stack(dists, n) -> np.ndarray:
    arr = np.empty((len(dists), n), np.float64)
    for p, d in enumerate(dists):
        w = d.weights if isinstance(d, Distribution) else _f64(d)
        if w.size != n:
            raise Error(errc.length_mismatch,
                        "LengthMismatch: distributions must live on the filter's graph")
        arr[p] = w
    return arr


def _sinkhorn(filter: HeatFilter, mus, nus, a, params: SinkhornParams, flags: int):
    ctx = filter._ctx
    n = filter.size()
    if len(mus) != len(nus):
        raise Error(errc.size_mismatch, "SizeMismatch: pair lists differ in length")
    P = len(mus)
    if P == 0:
        return []
    M = _stack(mus, n)
    N = _stack(nus, n)
    a = _f64(a)
    if a.size != n:
        raise Error(errc.length_mismatch,
                    "LengthMismatch: vertex weights must live on the filter's graph")
    v = np.empty((P, n))
    w = np.empty((P, n))
    cost = np.empty(P)
    kl = np.empty(P)
    it = np.empty(P, np.int32)
    conv = np.empty(P, np.int32)
    err = np.empty(P)
    fp, fs = C.c_int(), C.c_int()
    ctx.check(ctx.lib.gs_sinkhorn(ctx.handle, filter._h, _ptr(a), _ptr(M), _ptr(N), P,
                                  int(params.max_iter), float(params.tol), flags,
                                  _capi.GS_MEM_HOST, _ptr(v), _ptr(w), _ptr(cost), _ptr(kl),
                                  _ptr(it), _ptr(conv), _ptr(err), C.byref(fp), C.byref(fs)))
    lam = 4.0 * filter.time()
    return [TransportResult(v[p].copy(), w[p].copy(), float(cost[p]), float(kl[p]), lam, int(it[p]),
                            bool(conv[p]), float(err[p])) for p in range(P)]


def geodesic_sinkhorn(filter: HeatFilter, mu: Distribution, nu: Distribution, a,
                      params: SinkhornParams = SinkhornParams(), fp32: bool = False) -> TransportResult:
    """transport.cpp:243-247 (sinkhorn_single semantics and messages)."""
    flags = _capi.GS_FLAG_SINGLE | (_capi.GS_FLAG_FP32 if fp32 else 0)
    return _sinkhorn(filter, [mu], [nu], a, params, flags)[0]


def geodesic_sinkhorn_batch(filter: HeatFilter, mus: List[Distribution], nus: List[Distribution],
                            a, params: SinkhornParams = SinkhornParams(),
                            no_stagnation_abort: bool = False,
                            fp32: bool = False) -> List[TransportResult]:
    """transport.cpp:249-255. `no_stagnation_abort` is the bench-only deviation;
    `fp32` the optional fp32 mode."""
    flags = _capi.GS_FLAG_NO_STAGNATION_ABORT if no_stagnation_abort else 0
    if fp32:
        flags |= _capi.GS_FLAG_FP32
    return _sinkhorn(filter, mus, nus, a, params, flags)


def _euler_sinkhorn(euler: "EulerHeat", mus, nus, a, params: SinkhornParams, flags: int):
    ctx = euler._ctx
    n = euler.size()
    if len(mus) != len(nus):
        raise Error(errc.size_mismatch, "SizeMismatch: pair lists differ in length")
    P = len(mus)
    if P == 0:
        return []
    M, N, a = _stack(mus, n), _stack(nus, n), _f64(a)
    if a.size != n:
        raise Error(errc.length_mismatch, "LengthMismatch: vertex weights must live on the filter's graph")
    v, w = np.empty((P, n)), np.empty((P, n))
    cost, kl, err = np.empty(P), np.empty(P), np.empty(P)
    it, conv = np.empty(P, np.int32), np.empty(P, np.int32)
    fp, fs = C.c_int(), C.c_int()
    ctx.check(ctx.lib.gs_euler_sinkhorn(ctx.handle, euler._h, _ptr(a), _ptr(M), _ptr(N), P,
                                        int(params.max_iter), float(params.tol), flags,
                                        _capi.GS_MEM_HOST, _ptr(v), _ptr(w), _ptr(cost), _ptr(kl),
                                        _ptr(it), _ptr(conv), _ptr(err), C.byref(fp), C.byref(fs)))
    lam = 4.0 * euler.time()
    return [TransportResult(v[p].copy(), w[p].copy(), float(cost[p]), float(kl[p]), lam, int(it[p]),
                            bool(conv[p]), float(err[p])) for p in range(P)]


def dense_sinkhorn(cost_matrix, mu: Distribution, nu: Distribution, lam: float,
                   params: SinkhornParams = SinkhornParams(), ctx: Optional[Context] = None) -> TransportResult:
    """transport.cpp:271-311: entropic Sinkhorn with the dense kernel exp(-C / lam), on the device
    (gs_dense_sinkhorn)."""
    ctx = _ctx(ctx)
    Cm = np.ascontiguousarray(cost_matrix, np.float64)
    if Cm.ndim != 2:
        raise Error(errc.invalid_argument, "InvalidArgument: cost matrix must be two-dimensional")
    m = mu.weights if isinstance(mu, Distribution) else _f64(mu)
    x = nu.weights if isinstance(nu, Distribution) else _f64(nu)
    r, c = Cm.shape
    if m.size != r or x.size != c:
        Distribution(m).validate()
        Distribution(x).validate()
        raise Error(errc.length_mismatch, "LengthMismatch: cost matrix shape does not match the marginals")
    v, w = np.empty(r), np.empty(c)
    cost, kl, err = np.empty(1), np.empty(1), np.empty(1)
    it, conv = np.empty(1, np.int32), np.empty(1, np.int32)
    ctx.check(ctx.lib.gs_dense_sinkhorn(ctx.handle, _ptr(Cm), r, c, _ptr(m), _ptr(x), float(lam),
                                        int(params.max_iter), float(params.tol), _capi.GS_MEM_HOST,
                                        _ptr(v), _ptr(w), _ptr(cost), _ptr(kl), _ptr(it), _ptr(conv),
                                        _ptr(err)))
    return TransportResult(v, w, float(cost[0]), float(kl[0]), float(lam), int(it[0]), bool(conv[0]),
                           float(err[0]))


def dense_sinkhorn_groups(points, groups: Sequence[Sequence[int]], pairs: Sequence[Tuple[int, int]],
                          squared: bool, lam: float, params: SinkhornParams = SinkhornParams(),
                          ctx: Optional[Context] = None) -> List[TransportResult]:
    """The kNN benchmark's dense baselines (bench.cpp:311-331) for many pairs at once: pair (a, b)
    transports the uniform distribution on points[groups[a]] onto the one on points[groups[b]]
    with cost squared_distances (bench.cpp:32-39) or its square root (squared=False). Results
    carry cost, kl, iterations, converged and marginal_error (v and w are not returned)."""
    ctx = _ctx(ctx)
    X = np.ascontiguousarray(points, np.float64)
    if X.ndim != 2:
        raise Error(errc.invalid_argument, "InvalidArgument: points must be n x d")
    gidx = np.ascontiguousarray(np.concatenate([np.asarray(g, np.int32) for g in groups]), np.int32)
    goff = np.zeros(len(groups) + 1, np.int32)
    goff[1:] = np.cumsum([len(g) for g in groups])
    pa = np.ascontiguousarray([p[0] for p in pairs], np.int32)
    pb = np.ascontiguousarray([p[1] for p in pairs], np.int32)
    P = len(pairs)
    cost, kl, err = np.empty(P), np.empty(P), np.empty(P)
    it, conv = np.empty(P, np.int32), np.empty(P, np.int32)
    fp = C.c_int()
    ctx.check(ctx.lib.gs_dense_sinkhorn_groups(ctx.handle, _ptr(X), X.shape[0], X.shape[1], _ptr(gidx),
                                               _ptr(goff), len(groups), _ptr(pa), _ptr(pb), P,
                                               1 if squared else 0, float(lam), int(params.max_iter),
                                               float(params.tol), _ptr(cost), _ptr(kl), _ptr(it),
                                               _ptr(conv), _ptr(err), C.byref(fp)))
    return [TransportResult(np.zeros(0), np.zeros(0), float(cost[p]), float(kl[p]), float(lam), int(it[p]),
                            bool(conv[p]), float(err[p])) for p in range(P)]


def euler_sinkhorn(euler: "EulerHeat", mu: Distribution, nu: Distribution, a,
                   params: SinkhornParams = SinkhornParams()) -> TransportResult:
    """transport.cpp:257-261 (sinkhorn_single semantics over EulerHeat)."""
    return _euler_sinkhorn(euler, [mu], [nu], a, params, _capi.GS_FLAG_SINGLE)[0]


def euler_sinkhorn_batch(euler: "EulerHeat", mus, nus, a, params: SinkhornParams = SinkhornParams(),
                         no_stagnation_abort: bool = False) -> List[TransportResult]:
    """transport.cpp:263-269 (sinkhorn_many over EulerHeat)."""
    return _euler_sinkhorn(euler, mus, nus, a, params,
                           _capi.GS_FLAG_NO_STAGNATION_ABORT if no_stagnation_abort else 0)


# ------------------------------------------------------------------------------ row partitions
class RowPartition:
    """One rank's rows of a filter for row-partitioned multi-GPU runs (gs_part_*; SURVEY.md
    §8(e)). The reference is single-process; this splits HeatFilter::apply (heat.cpp:116-131) and
    sinkhorn_many (transport.cpp:144-239) by rows. Local vectors are indexed like `vertices`
    (original vertex ids of this part's rows); `comm` is a gs_comm (distributed.TorchComm.comm)
    and may be None only for a single part."""

    def __init__(self, filter: HeatFilter, nparts: int, part: int, ctx: Optional[Context] = None):
        self.filter = filter
        self._ctx = ctx if ctx is not None else filter._ctx
        self.nparts, self.part = int(nparts), int(part)
        h = C.c_void_p()
        self._ctx.check(self._ctx.lib.gs_part_create(self._ctx.handle, filter._h, self.nparts,
                                                     self.part, C.byref(h)))
        self._h = h
        rb, re_, nh, ns = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        nnz = C.c_int64()
        self._ctx.check(self._ctx.lib.gs_part_info(h, C.byref(rb), C.byref(re_), C.byref(nh),
                                                   C.byref(nnz), C.byref(ns)))
        self.row_begin, self.row_end = rb.value, re_.value
        self.n_local = self.row_end - self.row_begin
        self.n_halo, self.n_send, self.nnz_local = nh.value, ns.value, nnz.value
        self.send_counts = np.zeros(self.nparts, np.int64)
        self.recv_counts = np.zeros(self.nparts, np.int64)
        self._ctx.check(self._ctx.lib.gs_part_counts(h, _ptr(self.send_counts),
                                                     _ptr(self.recv_counts)))
        lo, hi = C.c_int(), C.c_int()
        self._ctx.check(self._ctx.lib.gs_part_interior(h, C.byref(lo), C.byref(hi)))
        self.interior = (lo.value, hi.value)  # rows computed while the halo is in flight
        self.vertices = np.empty(self.n_local, np.int32)
        self._ctx.check(self._ctx.lib.gs_part_vertices(self._ctx.handle, h, _ptr(self.vertices),
                                                       _capi.GS_MEM_HOST))

    def _comm(self, comm):
        if comm is None:
            return None
        if isinstance(comm, C.c_void_p):  # a gs_comm* (the engine's NCCL communicator)
            return comm
        return C.byref(comm)

    def apply(self, f_local, comm=None, fp32: bool = False) -> np.ndarray:
        """H f on this part's rows: (n_local,) or (n_local, B) local signals."""
        x = _f64(f_local)
        if x.shape[0] != self.n_local:
            raise Error(errc.length_mismatch, "LengthMismatch: signal length")
        cols = _f64(x.reshape(self.n_local, -1).T)
        out = np.empty_like(cols)
        self._ctx.check(self._ctx.lib.gs_part_filter_apply(
            self._ctx.handle, self._h, self._comm(comm), _ptr(cols), _ptr(out), cols.shape[0],
            _capi.GS_FLAG_FP32 if fp32 else 0, _capi.GS_MEM_HOST))
        return out.T.reshape(x.shape).copy()

    def sinkhorn(self, mus_local, nus_local, a_local, params: SinkhornParams = SinkhornParams(),
                 comm=None, no_stagnation_abort: bool = False, fp32: bool = False,
                 single: bool = False) -> List[TransportResult]:
        """geodesic_sinkhorn_batch on local rows; v, w of each result are local rows, the scalars
        (cost, kl, iterations, converged, marginal_error) are global and equal on every rank."""
        nl = self.n_local
        if len(mus_local) != len(nus_local):
            raise Error(errc.size_mismatch, "SizeMismatch: pair lists differ in length")
        P = len(mus_local)
        if P == 0:
            return []
        M = _stack(mus_local, nl)
        N = _stack(nus_local, nl)
        a = _f64(a_local)
        if a.size != nl:
            raise Error(errc.length_mismatch,
                        "LengthMismatch: vertex weights must live on the filter's graph")
        flags = (_capi.GS_FLAG_NO_STAGNATION_ABORT if no_stagnation_abort else 0) | \
                (_capi.GS_FLAG_FP32 if fp32 else 0) | (_capi.GS_FLAG_SINGLE if single else 0)
        v = np.empty((P, nl))
        w = np.empty((P, nl))
        cost = np.empty(P)
        kl = np.empty(P)
        it = np.empty(P, np.int32)
        conv = np.empty(P, np.int32)
        err = np.empty(P)
        fp, fs = C.c_int(), C.c_int()
        self._ctx.check(self._ctx.lib.gs_part_sinkhorn(
            self._ctx.handle, self._h, self._comm(comm), _ptr(a), _ptr(M), _ptr(N), P,
            int(params.max_iter), float(params.tol), flags, _capi.GS_MEM_HOST, _ptr(v), _ptr(w),
            _ptr(cost), _ptr(kl), _ptr(it), _ptr(conv), _ptr(err), C.byref(fp), C.byref(fs)))
        lam = 4.0 * self.filter.time()
        return [TransportResult(v[p].copy(), w[p].copy(), float(cost[p]), float(kl[p]), lam,
                                int(it[p]), bool(conv[p]), float(err[p])) for p in range(P)]

    def __del__(self):
        try:
            if self._h:
                self._ctx.lib.gs_part_destroy(self._h)
        except Exception:
            pass


# ---------------------------------------------------------------------------------- barycenter
@dataclass
class DistributionFamily:
    members: List[Distribution] = field(default_factory=list)
    alphas: Optional[np.ndarray] = None  # None / empty means uniform
    label: str = ""

    def resolved_alphas(self) -> np.ndarray:
        if self.alphas is None or len(self.alphas) == 0:
            return np.full(len(self.members), 1.0 / len(self.members))
        return _f64(self.alphas)

    def validate(self, n: int) -> None:
        if not self.members:
            raise Error(errc.invalid_argument, "InvalidArgument: family must be non-empty")
        for m in self.members:
            m.validate()
            if m.size() != n:
                raise Error(errc.length_mismatch,
                            "LengthMismatch: family members must share the graph")
        al = self.resolved_alphas()
        if al.size != len(self.members):
            raise Error(errc.length_mismatch, "LengthMismatch: one alpha per member required")
        if not (al >= 0.0).all():
            raise Error(errc.invalid_argument, "InvalidArgument: alphas must be non-negative")
        if not abs(al.sum() - 1.0) <= 1e-9:
            raise Error(errc.invalid_argument, "InvalidArgument: alphas must sum to 1")


@dataclass
class BarycenterResult:
    barycenter: Distribution
    scalings: list
    iterations: int = 0
    converged: bool = False
    marginal_error: float = math.inf


def sinkhorn_barycenter(filter: HeatFilter, family: DistributionFamily, a,
                        params: SinkhornParams = SinkhornParams(),
                        fp32: bool = False) -> BarycenterResult:
    """barycenter.cpp:45-99."""
    ctx = filter._ctx
    n = filter.size()
    family.validate(n)
    a = _f64(a)
    if a.size != n:
        raise Error(errc.length_mismatch,
                    "LengthMismatch: vertex weights must live on the filter's graph")
    members = _stack(family.members, n)
    m = members.shape[0]
    al = family.resolved_alphas()
    bary = np.empty(n)
    V = np.empty((m, n))
    W = np.empty((m, n))
    it = np.zeros(1, np.int32)
    conv = np.zeros(1, np.int32)
    err = np.zeros(1)
    ctx.check(ctx.lib.gs_barycenter_ex(ctx.handle, filter._h, _ptr(a), _ptr(members), m, _ptr(al),
                                       int(params.max_iter), float(params.tol), _capi.GS_MEM_HOST,
                                       None, _capi.GS_FLAG_FP32 if fp32 else 0, _ptr(bary), _ptr(V),
                                       _ptr(W), _ptr(it), _ptr(conv), _ptr(err)))
    return BarycenterResult(Distribution(bary, validate=False),
                            [(V[c].copy(), W[c].copy()) for c in range(m)], int(it[0]),
                            bool(conv[0]), float(err[0]))


def barycentric_distance(filter: HeatFilter, family_t: DistributionFamily,
                         family_c: DistributionFamily, a,
                         params: SinkhornParams = SinkhornParams()) -> float:
    """barycenter.cpp:101-107."""
    bt = sinkhorn_barycenter(filter, family_t, a, params)
    bc = sinkhorn_barycenter(filter, family_c, a, params)
    return geodesic_sinkhorn(filter, bt.barycenter, bc.barycenter, a, params).cost


def expected_barycenter_effect(filter: HeatFilter, family_t: DistributionFamily,
                               family_c: DistributionFamily, features, a,
                               params: SinkhornParams = SinkhornParams()) -> np.ndarray:
    """barycenter.cpp:108-119: features^T (barycenter_t - barycenter_c); features n x d."""
    F = _f64(features).reshape(filter.size(), -1)
    bt = sinkhorn_barycenter(filter, family_t, a, params)
    bc = sinkhorn_barycenter(filter, family_c, a, params)
    return F.T @ (bt.barycenter.weights - bc.barycenter.weights)


def tv_baseline_effect(family_t: DistributionFamily, family_c: DistributionFamily,
                       features) -> np.ndarray:
    """barycenter.cpp:121-135: features^T (mixture_t - mixture_c), mixtures alpha-weighted."""
    F = _f64(features)
    n = F.shape[0]
    F = F.reshape(n, -1)
    family_t.validate(n)
    family_c.validate(n)

    def mixture(fam):
        mix = np.zeros(n)
        for al, mem in zip(fam.resolved_alphas(), fam.members):
            mix = mix + al * mem.weights
        return mix

    return F.T @ (mixture(family_t) - mixture(family_c))


# ---------------------------------------------------------------------------------- next (§8(f))
def plan_rows(result: TransportResult, filter: HeatFilter, a, rows) -> np.ndarray:
    """plan_row (transport.cpp:314-324) for several rows at once: (len(rows), n) array."""
    ctx = filter._ctx
    n = filter.size()
    if result.v.size != n or result.w.size != n:
        raise Error(errc.length_mismatch, "LengthMismatch: result does not match the filter's graph")
    rows = np.ascontiguousarray(np.atleast_1d(rows), np.int32)
    out = np.empty((rows.size, n))
    a = _f64(a)
    ctx.check(ctx.lib.gs_plan_rows(ctx.handle, filter._h, _ptr(a), _ptr(_f64(result.v)),
                                   _ptr(_f64(result.w)), _ptr(rows), rows.size, _capi.GS_MEM_HOST,
                                   _ptr(out)))
    return out


def plan_row(result: TransportResult, filter: HeatFilter, a, i: int) -> np.ndarray:
    """transport.cpp:314-324."""
    return plan_rows(result, filter, a, [i])[0]


def _validate_points(x, what: str) -> np.ndarray:
    """PointCloud::validate (pointcloud.hpp:20-24)."""
    x = np.asarray(x, np.float64)
    if x.ndim != 2 or x.shape[0] < 1 or x.shape[1] < 1:
        raise Error(errc.dimension_mismatch, "DimensionMismatch: point cloud must be non-empty")
    if not np.isfinite(x).all():
        raise Error(errc.dimension_mismatch, "DimensionMismatch: point cloud has non-finite entries")
    return x


def mccann_interpolate(source, target, plan_row_fn, s: float, num_samples: int,
                       rng_seed: int) -> np.ndarray:
    """transport.cpp:326-376: McCann interpolation at time s by sampling the transport plan --
    sources drawn by their plan-row mass, then a target within the sampled row, each emitting
    (1 - s) x_i + s y_j. `plan_row_fn(i)` returns plan row i over the target points (the device
    computes them: `geodesic_plan_rows` below). Row masses, their total and the cumulative sums
    are sequential sums in index order (Eigen's sum() order is unpinned); draws follow
    geosink::Rng (rng.hpp) in the reference order."""
    from .rng import Rng
    src = _validate_points(source, "source")
    tgt = _validate_points(target, "target")
    if src.shape[1] != tgt.shape[1]:
        raise Error(errc.size_mismatch, "SizeMismatch: source and target dimensions differ")
    if not (0.0 <= s <= 1.0):
        raise Error(errc.invalid_argument, "InvalidArgument: interpolation time must be in [0, 1]")
    if num_samples < 1:
        raise Error(errc.invalid_argument, "InvalidArgument: need at least one sample")
    m_src, m_tgt = src.shape[0], tgt.shape[0]
    row_mass = np.empty(m_src)
    for i in range(m_src):
        row = np.asarray(plan_row_fn(i), np.float64)
        if row.size != m_tgt:
            raise Error(errc.length_mismatch, "LengthMismatch: plan row has wrong length")
        row_mass[i] = np.cumsum(np.maximum(row, 0.0))[-1]
    cum = np.cumsum(row_mass)  # std::partial_sum
    total = float(cum[-1])
    if not (total >= 1.0 - 1e-6):
        raise Error(errc.degenerate_plan,
                    "DegeneratePlan: plan mass below 1; transport result unusable for interpolation")
    rng = Rng(rng_seed)
    counts = np.zeros(m_src, np.int64)
    for _ in range(num_samples):
        u = rng.uniform() * total
        i = int(np.searchsorted(cum, u, side="left"))  # std::lower_bound
        counts[min(i, m_src - 1)] += 1
    out = np.empty((num_samples, src.shape[1]))
    written = 0
    for i in range(m_src):
        c = int(counts[i])
        if c == 0:
            continue
        row_cum = np.cumsum(np.maximum(np.asarray(plan_row_fn(i), np.float64), 0.0))
        row_total = float(row_cum[-1])
        if not (row_total > 0.0):
            raise Error(errc.degenerate_plan, "DegeneratePlan: sampled an empty plan row")
        for _ in range(c):
            u = rng.uniform() * row_total
            j = int(np.searchsorted(row_cum, u, side="left"))
            out[written] = (1.0 - s) * src[i] + s * tgt[min(j, m_tgt - 1)]
            written += 1
    return out


def geodesic_plan_rows(result: TransportResult, filter: HeatFilter, a, source_vertices,
                       target_vertices) -> np.ndarray:
    """The source x target block of the geodesic plan (transport.cpp:314-324 row by row; the
    interpolation benchmark's batched form, bench.cpp:439-448): all source rows in one device
    call, restricted to the target vertices. Returns (len(source_vertices), len(target_vertices))."""
    rows = plan_rows(result, filter, a, np.asarray(source_vertices, np.int32))
    return np.ascontiguousarray(rows[:, np.asarray(target_vertices, np.int64)])


def save_graph(m: SparseSymMatrix, path: str) -> None:
    """sparse.cpp:137-157."""
    rc = m._ctx.lib.gs_graph_save(m._ctx.handle, m._h, path.encode())
    if rc:
        raise Error(errc.io_error, f"IoError: cannot write '{path}'")


def load_graph(path: str, ctx: Optional[Context] = None) -> SparseSymMatrix:
    """sparse.cpp:159-174."""
    ctx = _ctx(ctx)
    h = C.c_void_p()
    rc = ctx.lib.gs_graph_load(ctx.handle, path.encode(), C.byref(h))
    if rc == 16:
        raise Error(errc.io_error, f"IoError: cannot read graph file '{path}'")
    ctx.check(rc)
    return SparseSymMatrix(h, ctx)
