// gs_cheb.cu -- host drivers of the hot path: HeatFilter (heat.cpp:72-131), geodesic Sinkhorn
// (transport.cpp:108-255) and the barycenter (barycenter.cpp:45-107) on the device, for both the
// fp64 (reference-exact) and the optional fp32 precision. The fused Chebyshev step kernel lives
// in gs_step.cuh; this file holds the per-column finalise/control kernels, the layout kernels and
// the sweep loops.
//
// The Sinkhorn loop runs on the device: per sweep two K-step applies whose last step computes the
// next scaling vector in its epilogue, one finalise per apply (positivity check, thresholds,
// deterministic L1 error) and one control kernel (convergence / stagnation in pair order). The
// host polls a pinned status word with a two-sweep lag so the GPU queue never drains.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "gs_internal.cuh"
#include "gs_step.cuh"
#include "gs_win.cuh"
#include "gs_sell.cuh"
#include "gs_persist.cuh"

using namespace gsk;

namespace {

// ---- per-column finalise after an apply (transport.cpp:30-38 / barycenter.cpp:14-21) ----------
struct FinArgs {
  ColState cs;
  int B, tiles, Bpad;
  int check, has_next, has_err;
  gs_status* status;
  int knp_code;
  double slack;
};

__global__ void __launch_bounds__(kThreads) k_finalize(const FinArgs F) {
  const int col = blockIdx.x;
  if (col >= F.B) return;
  __shared__ double sh[kThreads];
  double acc = 0.0;
  if (F.has_err) {
    for (int t = threadIdx.x; t < F.tiles; t += kThreads) acc = acc + F.cs.part_err[(size_t)t * F.Bpad + col];
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const bool act = !F.cs.active || F.cs.active[col];
  if (F.check && act && F.status->error == 0) {
    const double mn = dunkey(F.cs.cmin[col]);
    if (!(mn >= -F.cs.thr[col])) atomicCAS(&F.status->error, 0, F.knp_code);
  }
  if (F.has_next) F.cs.thr[col] = F.slack * dunkey(F.cs.cmax[col]);
  if (F.has_err) F.cs.errcol[col] = sh[0];
  F.cs.cmin[col] = KEY_POS_INF;
  F.cs.cmax[col] = KEY_ZERO;
}

// ---- Sinkhorn control (transport.cpp:184-226), one thread, columns in pair order ------------
struct CtlArgs {
  int* active;
  int* gactive;
  int GW;
  const double* errcol;
  int* iters;
  int* conv;
  int* stag;
  int* final_sweep;
  double* err_out;
  gs_status* status;
  int* sweep_ctr;  // device sweep counter (so a captured sweep can be replayed)
  int P, max_iter, no_abort;
  int fp32;  // a non-finite marginal error is numerical_underflow (the fp32 range was left)
  double tol;
};

__global__ void k_sk_control(const CtlArgs C) {
  gs_status* st = C.status;
  const int s = ++(*C.sweep_ctr);
  if (st->error || s > C.max_iter) return;
  int na = 0;
  for (int c = 0; c < C.P; ++c) {
    if (!C.active[c]) continue;
    const double err = C.errcol[c];
    C.iters[c] = s;
    C.err_out[c] = err;
    if (C.fp32 && !isfinite(err)) {
      st->error = ERRC_NUMERICAL_UNDERFLOW + 1;
      st->fail_pair = c;
      st->fail_sweep = s;
      return;
    }
    const bool done = err <= C.tol;
    if (done) C.conv[c] = 1;
    if (done || s == C.max_iter) C.final_sweep[c] = s;
    if (!done) {
      C.stag[c] = err > 0.5 ? C.stag[c] + 1 : 0;
      if (!C.no_abort && !(C.stag[c] < 50)) {
        st->error = ERRC_DISCONNECTED + 1;
        st->fail_pair = c;
        st->fail_sweep = s;
        return;
      }
      ++na;
    } else {
      C.active[c] = 0;
      C.gactive[c / C.GW] -= 1;
    }
  }
  if (s == C.max_iter) {
    for (int c = 0; c < C.P; ++c) {
      if (C.active[c]) C.gactive[c / C.GW] -= 1;
      C.active[c] = 0;
    }
    na = 0;
  }
  st->n_active = na;
}

// ---- layout conversion: column-major fp64 (API) <-> grouped row-major S (engine) ------------
template <typename S>
__global__ void k_pack(const double* __restrict__ src, S* __restrict__ dst, int n, int width,
                       int GW, int G, const int* __restrict__ order, int64_t ld) {
  const int64_t total = (int64_t)G * n * GW;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % GW);
    const int64_t r = e / GW;
    const int i = (int)(r % n);
    const int g = (int)(r / n);
    const int col = g * GW + c;
    const int o = order ? order[i] : i;
    dst[((size_t)g * ld + i) * GW + c] = Prec<S>::enc(col < width ? src[(size_t)col * n + o] : 0.0);
  }
}

template <typename S>
__global__ void k_unpack(const S* __restrict__ src, double* __restrict__ dst, int n, int width,
                         int GW, const S* __restrict__ alt, const int* __restrict__ sel,
                         const int* __restrict__ newpos, int64_t ld) {
  const int64_t total = (int64_t)width * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(e / n);
    const int i0 = (int)(e % n);
    const int i = newpos ? newpos[i0] : i0;
    const int g = col / GW, c = col % GW;
    const size_t idx = ((size_t)g * ld + i) * GW + c;
    const S* s = (alt && sel && (sel[col] & 1)) ? alt : src;
    dst[e] = Prec<S>::dec(s[idx]);
  }
}

// permuted copy of an n-vector into the engine precision
template <typename S>
__global__ void k_gather_to(const double* __restrict__ src, const int* __restrict__ order, int n,
                            S* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = S(src[order ? order[i] : i]);
}

__global__ void k_gather(const double* __restrict__ src, const int* __restrict__ order, int n,
                         double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[order[i]];
}

// T_0 = a * 1 for the initial phi apply (transport.cpp:171-176 with W = 1), colmax |T_0|
template <typename S>
__global__ void k_sk_init(const double* __restrict__ a, S* __restrict__ T0, int n, int GW, int G, int B,
                          unsigned long long* cmax, int64_t ld) {
  const int64_t total = (int64_t)G * n * GW;
  double local = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % GW);
    const int i = (int)((e / GW) % n);
    const int g = (int)((e / GW) / n);
    const int col = g * GW + c;
    const double v = col < B ? a[i] * 1.0 : 0.0;
    T0[((size_t)g * ld + i) * GW + c] = Prec<S>::enc(v);
    if (col < B) local = fmax(local, (double)fabs(v));
  }
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = local;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < B; ++c) atomicMax(cmax + c, dkey(sh[0]));
}

// ---- validation (transport.cpp:56-66, 96-102; barycenter.cpp:32-43) ----------------------------
__global__ void k_validate_cols(const double* __restrict__ X, int n, double* sums, int* nonfinite,
                                int* negative) {
  const int col = blockIdx.y;
  const double* x = X + (size_t)col * n;
  __shared__ double sh[kThreads];
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  double total = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) {
    double acc = 0.0;
    int bad_f = 0, bad_n = 0;
    for (int j = 0; j < DET_J; ++j) {
      const int64_t i = c * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
      if (i < n) {
        const double v = x[i];
        if (!isfinite(v)) bad_f = 1;
        if (v < 0.0) bad_n = 1;
        acc = acc + v;
      }
    }
    if (bad_f) atomicExch(nonfinite + col, 1);
    if (bad_n) atomicExch(negative + col, 1);
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kThreads / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) total = total + sh[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[col] = total;
}

__global__ void k_validate_weights(const double* __restrict__ a, int n, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !(a[i] > 0.0)) atomicExch(bad, 1);
}

// ---- final cost / KL (transport.cpp:137-140, 229-237), accumulated in double ------------------
template <typename S>
__global__ void k_sk_cost_partial(const S* __restrict__ a, const S* __restrict__ M,
                                  const S* __restrict__ N, const S* __restrict__ V0,
                                  const S* __restrict__ V1, const S* __restrict__ W,
                                  const int* __restrict__ final_sweep, int n, int GW,
                                  double* part /* [chunks][P][4] */, int P, int64_t ld) {
  const int col = blockIdx.y;
  const int64_t c = blockIdx.x;
  const int g = col / GW, cc = col % GW;
  const S* V = (final_sweep[col] & 1) ? V1 : V0;
  double s[4] = {0, 0, 0, 0};
  for (int j = 0; j < DET_J; ++j) {
    const int64_t i = c * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
    if (i >= n) break;
    const size_t idx = ((size_t)g * ld + i) * GW + cc;
    const double mu = M[idx], nu = N[idx], ai = a[i];
    if (mu > 0.0) {
      const double lv = log((double)V[idx]);
      s[0] = s[0] + ai * mu * lv;
      s[2] = s[2] + mu * lv;
    }
    if (nu > 0.0) {
      const double w = W[idx];
      s[1] = s[1] + ai * nu * log(w);
      s[3] = s[3] + nu * log(fmax(ai * w, GS_FLOOR));
    }
  }
  __shared__ double sh[4][kThreads];
#pragma unroll
  for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = s[q];
  __syncthreads();
  for (int st = kThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st)
#pragma unroll
      for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = sh[q][threadIdx.x] + sh[q][threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x < 4) part[((size_t)c * P + col) * 4 + threadIdx.x] = sh[threadIdx.x][0];
}

__global__ void k_sk_cost_final(const double* part, int64_t nchunks, int P, double lambda,
                                double* cost, double* kl) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= P) return;
  double s[4] = {0, 0, 0, 0};
  for (int64_t c = 0; c < nchunks; ++c)
    for (int q = 0; q < 4; ++q) s[q] = s[q] + part[((size_t)c * P + col) * 4 + q];
  cost[col] = lambda * (s[0] + s[1]);
  kl[col] = s[2] + s[3] - 1.0;
}

// ---- barycenter row kernels (barycenter.cpp:75-84), computed in double ----------------------
__global__ void k_bary_lb(const double* __restrict__ psi, const double* __restrict__ alphas, int n, int m,
                          int GW, double* __restrict__ lb, const gs_status* st) {
  if (st->error || st->done) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int c = 0; c < m; ++c) {
    const double v = psi[((size_t)(c / GW) * n + i) * GW + (c % GW)];
    const double ps = fmin(fmax(v, GS_FLOOR), GS_CEIL);
    acc = fma(alphas[c], log(ps), acc);
  }
  lb[i] = acc;
}

__global__ void k_max_key(const double* __restrict__ x, int n, unsigned long long* key) {
  double local = -INFINITY;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    local = fmax(local, x[i]);
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = local;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(key, dkey(sh[0]));
}

// bary_i = exp(lb_i - max) with DET-chunk partial sums of the mass
__global__ void k_bary_exp(const double* __restrict__ lb, const unsigned long long* maxkey, int n,
                           double* __restrict__ bary, double* part, const gs_status* st) {
  if (st->error || st->done) return;
  const double mx = dunkey(*maxkey);
  double acc = 0.0;
  for (int j = 0; j < DET_J; ++j) {
    const int64_t i = (int64_t)blockIdx.x * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
    if (i < n) {
      const double b = exp(lb[i] - mx);
      bary[i] = b;
      acc = acc + b;
    }
  }
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// DET-chunk partial sums of an n-vector (one chunk of 4096 per CTA)
__global__ void k_chunk_sum(const double* __restrict__ x, int n, double* part) {
  double acc = 0.0;
  for (int j = 0; j < DET_J; ++j) {
    const int64_t i = (int64_t)blockIdx.x * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
    if (i < n) acc = acc + x[i];
  }
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// deterministic fold of chunk partials (lane t folds t, t+256, ... then the tree)
__global__ void k_fold(const double* part, int64_t nparts, double* out) {
  __shared__ double sh[kThreads];
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < nparts; q += kThreads) acc = acc + part[q];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void k_bary_mass_check(const double* mass, gs_status* st) {
  if (st->error || st->done) return;
  if (!(*mass > 0.0)) st->error = 1000 + ERRC_KERNEL_NOT_POSITIVE + 1;  // "collapsed" variant
}

constexpr int kBaryColChunk = 2048;  // columns per shared-memory max pass of k_bary_w

// bary /= mass; W_c = bary / max(psi_c, floor); T_0 = a * W_c; colmax |T_0| (order-free max:
// warp shuffle, one shared-memory atomic per warp, one global atomic per CTA and column)
template <typename S>
__global__ void k_bary_w(double* __restrict__ bary, const double* __restrict__ mass,
                         const double* __restrict__ psi, const double* __restrict__ a, int n, int m,
                         int GW, double* __restrict__ W, S* __restrict__ T0, unsigned long long* cmax,
                         const gs_status* st) {
  __shared__ unsigned long long s_max[kBaryColChunk];
  if (st->error || st->done) return;  // the same status word for the whole grid
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = i < n;
  const double ms = *mass;
  double b = 0.0, ai = 0.0;
  if (ok) {
    b = bary[i] / ms;
    bary[i] = b;
    ai = a[i];
  }
  for (int c0 = 0; c0 < m; c0 += kBaryColChunk) {
    const int cn = min(kBaryColChunk, m - c0);
    for (int c = threadIdx.x; c < cn; c += blockDim.x) s_max[c] = KEY_ZERO;
    __syncthreads();
    for (int c = c0; c < c0 + cn; ++c) {
      double v = 0.0;
      if (ok) {
        const size_t idx = ((size_t)(c / GW) * n + i) * GW + (c % GW);
        const double w = b / fmax(psi[idx], GS_FLOOR);
        W[idx] = w;
        const double t0 = ai * w;
        T0[idx] = Prec<S>::enc(t0);
        v = fabs(t0);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      if ((threadIdx.x & 31) == 0) atomicMax(&s_max[c - c0], dkey(v));
    }
    __syncthreads();
    for (int c = threadIdx.x; c < cn; c += blockDim.x) atomicMax(cmax + c0 + c, s_max[c]);
    __syncthreads();
  }
}

// errbuf[0] = this rank's marginal error (max over its members, barycenter.cpp:86), errbuf[1] =
// its status error code: both are max-allreduced across member shards before k_bary_control, so
// a failure on one rank (positivity check, collapsed mass) stops every rank at the same sweep
// with the same errc and every rank issues the same collectives.
__global__ void k_bary_errlocal(const double* errcol, int m, double* errbuf, const gs_status* st) {
  double e = 0.0;
  for (int c = 0; c < m; ++c) e = fmax(e, errcol[c]);
  errbuf[0] = e;
  errbuf[1] = (double)st->error;
}

__global__ void k_bary_control(const double* errbuf, gs_status* st, int* sweep_ctr, double tol,
                               int* iters, int* conv, double* err_out, int max_iter, int fp32) {
  const int sweep = ++(*sweep_ctr);  // device counter: a captured sweep can be replayed
  if (!st->done && errbuf[1] != 0.0) st->error = (int)errbuf[1];  // the agreed (max) error code
  if (st->error || st->done) return;
  const double err = *errbuf;
  *err_out = err;
  *iters = sweep;
  if (fp32 && !isfinite(err)) {  // the fp32 recurrence's range was left
    st->error = ERRC_NUMERICAL_UNDERFLOW + 1;
    st->fail_sweep = sweep;
    return;
  }
  if (err <= tol) {
    *conv = 1;
    st->done = 1;
  } else if (sweep == max_iter) {
    st->done = 2;
  }
}

__global__ void k_scale_div(double* x, const double* s, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] / *s;
}

__global__ void k_fill(double* x, int64_t n, double v) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    x[e] = v;
}

__global__ void k_fill_key(unsigned long long* x, int n, unsigned long long v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

__global__ void k_scale_vals(double* v, int64_t nnz, double scale) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) v[e] = v[e] * scale;
}

// entries whose column lies within 256 rows of their row (layout order)
__global__ void k_near_count(const int* __restrict__ offs, const int* __restrict__ cols, int n,
                             unsigned long long* __restrict__ cnt) {
  unsigned long long c = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    for (int p = offs[r]; p < offs[r + 1]; ++p) c += (unsigned)abs(cols[p] - r) <= 256u;
  atomicAdd(cnt, c);
}

__global__ void k_to_float(const double* __restrict__ v, int64_t nnz, float* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) out[e] = (float)v[e];
}

inline unsigned grid_for(int64_t work, int threads = kThreads) {
  int64_t b = (work + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

// Columns per group: the next power of two >= B, at most 64 (one warp per 512-byte fp64 row).
int choose_gw(int width) {
  static const int cap = [] {  // GS_MAX_GW: narrower groups (experiments; results unchanged)
    const char* e = getenv("GS_MAX_GW");
    const int v = e ? atoi(e) : 64;
    return v >= 1 && v <= 64 && (v & (v - 1)) == 0 ? v : 64;
  }();
  int g = 1;
  while (g < width && g < cap) g <<= 1;
  return g;
}

// GS_SEQ_GROUPS=1: an apply runs its K steps group after group (each group's T_{k-1} written by
// the previous step is then L2-resident for its gathers) instead of all groups in every launch
inline bool seq_groups() {
  static const bool v = [] {
    const char* e = getenv("GS_SEQ_GROUPS");
    return e && atoi(e) != 0;
  }();
  return v;
}

template <typename S>
int rows_per_block(int gw) {  // rows covered by one CTA pass (8 warps)
  switch (gw) {
    case 64: return Lay<64, S>::ROWS;
    case 32: return Lay<32, S>::ROWS;
    case 16: return Lay<16, S>::ROWS;
    case 8: return Lay<8, S>::ROWS;
    case 4: return Lay<4, S>::ROWS;
    case 2: return Lay<2, S>::ROWS;
    default: return Lay<1, S>::ROWS;
  }
}

// Latency-bound one-column fp64 problems up to this many rows take one warp per row (GS_W1_MAX)
inline int w1_max_rows() {
  const char* e = getenv("GS_W1_MAX");  // read per call
  return e ? atoi(e) : 32768;
}

// lanes per row of a group width's layout
template <typename S>
int rpc_lpr(int gw) {
  switch (gw) {
    case 64: return Lay<64, S>::LPR;
    case 32: return Lay<32, S>::LPR;
    case 16: return Lay<16, S>::LPR;
    case 8: return Lay<8, S>::LPR;
    case 4: return Lay<4, S>::LPR;
    case 2: return Lay<2, S>::LPR;
    default: return Lay<1, S>::LPR;
  }
}

// One-row-per-lane layouts with the CSR stream staged through shared memory (k_cheb_lane):
// GS_LANE=0 keeps them on k_cheb_step, GS_LANE_PAD=0 stages the plain CSR arrays instead of the
// odd-stride copy (both read per call).
inline bool lane_enabled() {
  const char* e = getenv("GS_LANE");
  return !(e && atoi(e) == 0);
}
// fp64 rows shared by several lanes through the record kernel (k_cheb_rec): bit-identical to
// k_cheb_step. GS_REC=1 / 0 forces it on / off (read per call, so tests can compare the two);
// unset, it runs the 128-byte rows (B = 9..16) of graphs without index locality -- config 4:
// 1325 -> 1276 us per step on the 2048-row degree-sorted layout -- and nothing else: config 2's
// 64-byte rows measure 411 vs 280 us, and on the 256-row layout the two kernels tie
// (profiles/r02_summary.md "Record kernel").
inline int rec_mode() {
  const char* e = getenv("GS_REC");
  return e ? (atoi(e) != 0 ? 1 : 0) : -1;
}
template <typename S>
bool rec_wanted(int gw, const gs_filter* f) {
  const int m = rec_mode();
  if (m >= 0) return m == 1;
  return gw * (int)sizeof(S) == 128 && f && f->sigma >= 1024;
}
inline size_t l2_bytes() {  // L2 capacity of the current device
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
  return v > 0 ? (size_t)v : (size_t)64 << 20;
}
// GS_HEAVY_FIRST=0: tiles of the degree-sorted layout launch in row order (read per call)
inline bool heavy_first_enabled() {
  const char* e = getenv("GS_HEAVY_FIRST");
  return !(e && atoi(e) == 0);
}
inline bool lane_pad_enabled() {
  const char* e = getenv("GS_LANE_PAD");
  return !(e && atoi(e) == 0);
}

// row blocks per CTA of the full (multi-block) instantiation of a group width
template <typename S>
int rpc_full(int gw) {
  int lpr = 1;
  switch (gw) {
    case 64: lpr = Lay<64, S>::LPR; break;
    case 32: lpr = Lay<32, S>::LPR; break;
    case 16: lpr = Lay<16, S>::LPR; break;
    case 8: lpr = Lay<8, S>::LPR; break;
    case 4: lpr = Lay<4, S>::LPR; break;
    case 2: lpr = Lay<2, S>::LPR; break;
    default: lpr = Lay<1, S>::LPR; break;
  }
  return lpr == 1 ? kRowsPerCta1 : kRowsPerCta;
}

// Row blocks per CTA: kRowsPerCta (L1 reuse across consecutive blocks) unless that leaves fewer
// than two CTAs per SM, in which case 1 (small, latency-bound problems such as config 0).
template <typename S>
int choose_rpc(int n, int gw, int groups, double near_frac = 1.0) {
  const char* renv = getenv("GS_RPC");  // read per call (tests force the multi-block kernels)
  const int forced = renv ? atoi(renv) : 0;
  if (forced == 1) return 1;
  if (forced > 1) return rpc_full<S>(gw);
  // several lanes per row and fewer than 32 columns (the degree-sorted layout; configs 2 and 4:
  // B = 8 and 16 fp64 on kNN graphs in R^30): consecutive row blocks share few L1 lines, so short
  // CTAs win by shrinking the tail wave (config 2: 416 -> 351 us; config 4: 217 -> 151 us at 4e5)
  // 64-byte narrow rows (config 2's B = 8 fp64) went back to four row blocks per CTA once the next
  // CSR chunk is prefetched (340 -> 328 us); 128-byte rows (config 4's B = 16) stay at one
  // (343 vs 463 us at n = 1e6)
  if (gw < 32 && gw * (int)sizeof(S) == 64) {
    const int64_t ctas = (int64_t)groups * ((n + rows_per_block<S>(gw) * kRowsPerCta - 1) /
                                            (rows_per_block<S>(gw) * kRowsPerCta));
    return ctas < 2 * 148 ? 1 : kRowsPerCta;
  }
  if (gw < 32 && gw * (int)sizeof(S) > 16) return 1;
  // graphs without index locality (kNN graphs in R^30: ~12% of entries within 256 rows in CM
  // order, against ~50% on the swiss roll) get no L1 reuse between row blocks either
  if (near_frac < 0.3) return 1;
  const int full = rpc_full<S>(gw);
  const int64_t ctas = (int64_t)groups * ((n + rows_per_block<S>(gw) * full - 1) / (rows_per_block<S>(gw) * full));
  return ctas < 2 * 148 ? 1 : full;
}

template <typename S, int GW, int RPC>
void launch_step_rpc(const StepArgs& A, int mode, cudaStream_t s) {
  dim3 grid((unsigned)(A.tiles * A.Gl));
  switch (mode) {
    case MODE_NONE: k_cheb_step<S, GW, MODE_NONE, RPC><<<grid, kStepThreads, 0, s>>>(A); break;
    case MODE_SK_PSI: k_cheb_step<S, GW, MODE_SK_PSI, RPC><<<grid, kStepThreads, 0, s>>>(A); break;
    case MODE_SK_PHI: k_cheb_step<S, GW, MODE_SK_PHI, RPC><<<grid, kStepThreads, 0, s>>>(A); break;
    default: k_cheb_step<S, GW, MODE_BARY_PSI, RPC><<<grid, kStepThreads, 0, s>>>(A); break;
  }
}

template <typename S, int GW, int MODE>
void launch_lane_mode(const StepArgs& A, cudaStream_t s) {
  constexpr int smem = lane_smem_bytes<S>();
  static std::vector<char> seen;  // the attribute is per device
  gs_once_per_device(seen, [] {
    cudaFuncSetAttribute(k_cheb_lane<S, GW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  k_cheb_lane<S, GW, MODE><<<dim3((unsigned)(A.tiles * A.Gl)), kStepThreads, smem, s>>>(A);
}

template <typename S, int GW>
void launch_lane(const StepArgs& A, int mode, cudaStream_t s) {
  switch (mode) {
    case MODE_NONE: launch_lane_mode<S, GW, MODE_NONE>(A, s); break;
    case MODE_SK_PSI: launch_lane_mode<S, GW, MODE_SK_PSI>(A, s); break;
    case MODE_SK_PHI: launch_lane_mode<S, GW, MODE_SK_PHI>(A, s); break;
    default: launch_lane_mode<S, GW, MODE_BARY_PSI>(A, s); break;
  }
}

template <typename S, int GW, int MODE, int RPC>
void launch_rec_mode(const StepArgs& A, cudaStream_t s) {
  constexpr int smem = rec_smem_bytes();
  static std::vector<char> seen;  // the attribute is per device
  gs_once_per_device(seen, [] {
    cudaFuncSetAttribute(k_cheb_rec<S, GW, MODE, RPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  k_cheb_rec<S, GW, MODE, RPC><<<dim3((unsigned)(A.tiles * A.Gl)), kStepThreads, smem, s>>>(A);
}

template <typename S, int GW, int RPC>
void launch_rec(const StepArgs& A, int mode, cudaStream_t s) {
  switch (mode) {
    case MODE_NONE: launch_rec_mode<S, GW, MODE_NONE, RPC>(A, s); break;
    case MODE_SK_PSI: launch_rec_mode<S, GW, MODE_SK_PSI, RPC>(A, s); break;
    case MODE_SK_PHI: launch_rec_mode<S, GW, MODE_SK_PHI, RPC>(A, s); break;
    default: launch_rec_mode<S, GW, MODE_BARY_PSI, RPC>(A, s); break;
  }
}

template <typename S, int GW>
void launch_step_gw(const StepArgs& A, int mode, int rpc, cudaStream_t s) {
  if constexpr (sizeof(S) == 8 && Lay<GW, S>::LPR > 1 && Lay<GW, S>::LPR < 32) {
    if (A.recs) {
      if (rpc == 1) launch_rec<S, GW, 1>(A, mode, s);
      else launch_rec<S, GW, kRowsPerCta>(A, mode, s);
      return;
    }
  }
  if (rpc == 1) launch_step_rpc<S, GW, 1>(A, mode, s);
  else if constexpr (Lay<GW, S>::LPR == 1) {
    if (A.lane) launch_lane<S, GW>(A, mode, s);
    else launch_step_rpc<S, GW, kRowsPerCta1>(A, mode, s);
  }
  else launch_step_rpc<S, GW, kRowsPerCta>(A, mode, s);
}

// Sliced step kernels (gs_sell.cuh): layouts with at least four rows per warp. Opt-in (GS_SELL=1,
// read per call so tests can compare them with k_cheb_step): bit-identical results, but measured
// slower than the register-gather kernel on the shapes they were written for -- config 2's
// 64-byte rows 413-555 vs 324 us, config 4's 128-byte rows 611-807 vs 401 us
// (profiles/r02_summary.md "Sliced store"): the step is bound by the registers that hold gathers
// in flight, not by the shuffles the sliced store removes.
inline bool sell_enabled() {
  const char* e = getenv("GS_SELL");
  return e && atoi(e) != 0;
}

// one row per lane (C = 32) through k_cheb_sell: opt-in (GS_SELL_C32=1) -- measured slower than
// k_cheb_step's one-row-per-lane path (config-3 shape at n = 2e6: 125-152 vs 75 us)
inline bool sell_c32_enabled() {
  const char* e = getenv("GS_SELL_C32");
  return e && atoi(e) != 0;
}

template <typename S>
int sell_height(int gw) {  // rows per warp of a group width (0: the sliced kernel does not apply)
  int c = 0;
  switch (gw) {
    case 32: c = Lay<32, S>::RPW; break;
    case 16: c = Lay<16, S>::RPW; break;
    case 8: c = Lay<8, S>::RPW; break;
    case 4: c = Lay<4, S>::RPW; break;
    case 2: c = Lay<2, S>::RPW; break;
    case 1: c = Lay<1, S>::RPW; break;
    default: c = 0; break;
  }
  return c >= 4 ? c : 0;
}

template <typename S, int GW, int SPW>
void launch_sell_spw(const StepArgs& A, const SellArgs& E, int mode, cudaStream_t s) {
  if constexpr (Lay<GW, S>::RPW >= 4) {
    const dim3 grid((unsigned)(A.tiles * A.Gl));
    switch (mode) {
      case MODE_NONE: k_cheb_sell<S, GW, MODE_NONE, SPW><<<grid, kStepThreads, 0, s>>>(A, E); break;
      case MODE_SK_PSI: k_cheb_sell<S, GW, MODE_SK_PSI, SPW><<<grid, kStepThreads, 0, s>>>(A, E); break;
      case MODE_SK_PHI: k_cheb_sell<S, GW, MODE_SK_PHI, SPW><<<grid, kStepThreads, 0, s>>>(A, E); break;
      default: k_cheb_sell<S, GW, MODE_BARY_PSI, SPW><<<grid, kStepThreads, 0, s>>>(A, E); break;
    }
  }
}

// warp-staged sliced kernel (k_cheb_sellw): rows of at least four lanes
template <typename S, int GW>
void launch_sellw_gw(const StepArgs& A, const SellArgs& E, int mode, cudaStream_t s) {
  if constexpr (Lay<GW, S>::RPW >= 4 && Lay<GW, S>::RPW <= 8) {
    const dim3 grid((unsigned)(A.tiles * A.Gl));
    switch (mode) {
      case MODE_NONE: k_cheb_sellw<S, GW, MODE_NONE><<<grid, kStepThreads, 0, s>>>(A, E); break;
      case MODE_SK_PSI: k_cheb_sellw<S, GW, MODE_SK_PSI><<<grid, kStepThreads, 0, s>>>(A, E); break;
      case MODE_SK_PHI: k_cheb_sellw<S, GW, MODE_SK_PHI><<<grid, kStepThreads, 0, s>>>(A, E); break;
      default: k_cheb_sellw<S, GW, MODE_BARY_PSI><<<grid, kStepThreads, 0, s>>>(A, E); break;
    }
  }
}

template <typename S, int GW>
int sellw_occupancy_gw() {  // resident CTAs per SM of the plain step
  int occ = 0;
  if constexpr (Lay<GW, S>::RPW >= 4 && Lay<GW, S>::RPW <= 8)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cheb_sellw<S, GW, MODE_NONE>, kStepThreads, 0);
  return occ;
}

template <typename S>
int sellw_occupancy(int gw) {
  switch (gw) {
    case 32: return sellw_occupancy_gw<S, 32>();
    case 16: return sellw_occupancy_gw<S, 16>();
    case 8: return sellw_occupancy_gw<S, 8>();
    case 4: return sellw_occupancy_gw<S, 4>();
    default: return 0;
  }
}

template <typename S>
void launch_step_sellw(gs_ctx* ctx, int gw, const StepArgs& A, const SellArgs& E, int mode) {
  gs_launch_begin(ctx, 0);
  switch (gw) {
    case 32: launch_sellw_gw<S, 32>(A, E, mode, ctx->stream); break;
    case 16: launch_sellw_gw<S, 16>(A, E, mode, ctx->stream); break;
    case 8: launch_sellw_gw<S, 8>(A, E, mode, ctx->stream); break;
    default: launch_sellw_gw<S, 4>(A, E, mode, ctx->stream); break;
  }
  gs_launch_end(ctx, 0);
}

template <typename S>
void launch_step_sell(gs_ctx* ctx, int gw, int spw, const StepArgs& A, const SellArgs& E, int mode) {
  gs_launch_begin(ctx, 0);
#define GS_SELL_CASE(W)                                                        \
  case W:                                                                      \
    if (spw == 1) launch_sell_spw<S, W, 1>(A, E, mode, ctx->stream);           \
    else launch_sell_spw<S, W, kSellSpw>(A, E, mode, ctx->stream);             \
    break;
  switch (gw) {
    GS_SELL_CASE(32)
    GS_SELL_CASE(16)
    GS_SELL_CASE(8)
    GS_SELL_CASE(4)
    GS_SELL_CASE(2)
    default:
      if (spw == 1) launch_sell_spw<S, 1, 1>(A, E, mode, ctx->stream);
      else launch_sell_spw<S, 1, kSellSpw>(A, E, mode, ctx->stream);
      break;
  }
#undef GS_SELL_CASE
  gs_launch_end(ctx, 0);
}

template <typename S>
void launch_step(gs_ctx* ctx, int gw, int rpc, const StepArgs& A, int mode) {
  gs_launch_begin(ctx, 0);
  if constexpr (sizeof(S) == 8) {
    if (A.rec_key) {  // 8-row block records (wide fp64 rows)
      const dim3 grid((unsigned)(A.tiles * A.Gl));
      switch (mode) {
        case MODE_NONE: k_cheb_blk<S, MODE_NONE><<<grid, kBlkWarps * 32, 0, ctx->stream>>>(A); break;
        case MODE_SK_PSI: k_cheb_blk<S, MODE_SK_PSI><<<grid, kBlkWarps * 32, 0, ctx->stream>>>(A); break;
        case MODE_SK_PHI: k_cheb_blk<S, MODE_SK_PHI><<<grid, kBlkWarps * 32, 0, ctx->stream>>>(A); break;
        default: k_cheb_blk<S, MODE_BARY_PSI><<<grid, kBlkWarps * 32, 0, ctx->stream>>>(A); break;
      }
      gs_launch_end(ctx, 0);
      return;
    }
  }
  if (A.warp_rows) {  // small one-column problems: one warp per row
    const dim3 grid((unsigned)(A.tiles * A.Gl));
    switch (mode) {
      case MODE_NONE: k_cheb_step_w1<S, MODE_NONE><<<grid, kThreads, 0, ctx->stream>>>(A); break;
      case MODE_SK_PSI: k_cheb_step_w1<S, MODE_SK_PSI><<<grid, kThreads, 0, ctx->stream>>>(A); break;
      case MODE_SK_PHI: k_cheb_step_w1<S, MODE_SK_PHI><<<grid, kThreads, 0, ctx->stream>>>(A); break;
      default: k_cheb_step_w1<S, MODE_BARY_PSI><<<grid, kThreads, 0, ctx->stream>>>(A); break;
    }
    gs_launch_end(ctx, 0);
    return;
  }
  switch (gw) {
    case 64: launch_step_gw<S, 64>(A, mode, rpc, ctx->stream); break;
    case 32: launch_step_gw<S, 32>(A, mode, rpc, ctx->stream); break;
    case 16: launch_step_gw<S, 16>(A, mode, rpc, ctx->stream); break;
    case 8: launch_step_gw<S, 8>(A, mode, rpc, ctx->stream); break;
    case 4: launch_step_gw<S, 4>(A, mode, rpc, ctx->stream); break;
    case 2: launch_step_gw<S, 2>(A, mode, rpc, ctx->stream); break;
    default: launch_step_gw<S, 1>(A, mode, rpc, ctx->stream); break;
  }
  gs_launch_end(ctx, 0);
}

// Windowed step kernel (gs_win.cuh) for wide rows: GS_WIN=0 turns it off (read per call).
inline bool win_enabled() {
  const char* e = getenv("GS_WIN");
  return !(e && atoi(e) == 0);
}

template <typename S, int GW, int MODE>
void launch_win_mode(const CUtensorMap& tm, const StepArgs& A, const WinArgs& WA, int G, cudaStream_t s) {
  constexpr int smem = win_smem_bytes<S, GW>();
  static std::vector<char> seen;  // the attribute is per device
  gs_once_per_device(seen, [] {
    cudaFuncSetAttribute(k_cheb_win<S, GW, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  k_cheb_win<S, GW, MODE><<<dim3((unsigned)(WA.nctas * G)), kWinThreads, smem, s>>>(tm, A, WA);
}

template <typename S, int GW>
void launch_win_gw(const CUtensorMap& tm, const StepArgs& A, const WinArgs& WA, int G, int mode, cudaStream_t s) {
  switch (mode) {
    case MODE_NONE: launch_win_mode<S, GW, MODE_NONE>(tm, A, WA, G, s); break;
    case MODE_SK_PSI: launch_win_mode<S, GW, MODE_SK_PSI>(tm, A, WA, G, s); break;
    case MODE_SK_PHI: launch_win_mode<S, GW, MODE_SK_PHI>(tm, A, WA, G, s); break;
    default: launch_win_mode<S, GW, MODE_BARY_PSI>(tm, A, WA, G, s); break;
  }
}

template <typename S>
void launch_step_win(gs_ctx* ctx, int gw, const CUtensorMap& tm, const StepArgs& A, const WinArgs& WA, int mode) {
  gs_launch_begin(ctx, 0);
  switch (gw) {
    case 64: launch_win_gw<S, 64>(tm, A, WA, A.Gl, mode, ctx->stream); break;
    case 32: launch_win_gw<S, 32>(tm, A, WA, A.Gl, mode, ctx->stream); break;
    case 16: launch_win_gw<S, 16>(tm, A, WA, A.Gl, mode, ctx->stream); break;
    default: launch_win_gw<S, 8>(tm, A, WA, A.Gl, mode, ctx->stream); break;
  }
  gs_launch_end(ctx, 0);
}

// Row sizes the windowed kernel takes: 256 bytes or more by default (GS_WIN_MIN_BYTES, at least
// 32). Narrower rows are the kNN graphs in R^30 (configs 2 and 4): at n = 1e6 a CTA's ring gets
// little reuse there (0.84 loads per entry) and the TMA gather4 issue rate (~75 cycles per
// instruction per SM) bounds the step at 1.5-1.9 ms, against 0.32-0.40 ms for the register-gather
// kernel (profiles/r02_summary.md).
template <typename S>
bool win_row_ok(int gw) {
  static const int min_bytes = [] {
    const char* e = getenv("GS_WIN_MIN_BYTES");
    return e ? atoi(e) : 256;
  }();
  return gw >= 8 && gw * (int)sizeof(S) >= min_bytes && gw * (int)sizeof(S) >= 32;
}

// GS_BLK=1 runs wide fp64 rows through the 8-row block kernel (k_cheb_blk). Off by default:
// it halves the gathered sectors (23.8M vs 49.7M per config-1 step) but doubles the
// instructions (predicated per-record fold) at 88 registers, 238 vs 117 us.
// Read per call, so tests can switch it.
inline bool blk_enabled() {
  const char* e = getenv("GS_BLK");
  return e && atoi(e) != 0;
}

__global__ void k_blk_keys(const int* __restrict__ offs, const int* __restrict__ cols,
                           const int* __restrict__ order, int n, unsigned long long* keys, int* idx) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long b = (unsigned long long)(i >> 3), r = (unsigned long long)(i & 7);
  for (int p = offs[i]; p < offs[i + 1]; ++p) {
    const unsigned long long oc = (unsigned)order[cols[p]];  // original column id
    keys[p] = (b << 34) | (oc << 3) | r;
    idx[p] = p;
  }
}

__global__ void k_blk_fill(const unsigned long long* __restrict__ keys, const int* __restrict__ idx,
                           const int* __restrict__ cols, const double* __restrict__ vals, int64_t nnz,
                           int* rec_key, double* rec_val) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nnz) return;
  const int p = idx[j];
  rec_key[j] = (cols[p] << 3) | (int)(keys[j] & 7ull);
  rec_val[j] = vals[p];
}

// 8-row block records of layout `l` (gs_layout::rec_key / rec_val), built once.
int gs_build_block_records(gs_ctx* ctx, gs_filter* f, int l) {
  gs_layout& Ly = f->lay[l];
  if (Ly.rec_key) return GS_OK;
  const gs_graph* G = Ly.perm;
  const int n = G->n;
  const int64_t nnz = G->nnz;
  if (n >= (1 << 28) || nnz >= (int64_t)INT32_MAX)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "block records: graph too large");
  cudaStream_t s = ctx->stream;
  DevBuf<unsigned long long> k0, k1;
  DevBuf<int> i0, i1;
  GS_CUDA(ctx, k0.alloc(nnz, s));
  GS_CUDA(ctx, k1.alloc(nnz, s));
  GS_CUDA(ctx, i0.alloc(nnz, s));
  GS_CUDA(ctx, i1.alloc(nnz, s));
  if (n > 0) {
    gs_launch_begin(ctx, 1);
    k_blk_keys<<<(n + 255) / 256, 256, 0, s>>>(G->offs, G->cols, Ly.order, n, k0.get(), i0.get());
    gs_launch_end(ctx, 1);
  }
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.get(), k1.get(), i0.get(), i1.get(), (int)nnz, 0, 64, s);
  DevBuf<unsigned char> tmp;
  GS_CUDA(ctx, tmp.alloc(tb, s));
  cub::DeviceRadixSort::SortPairs(tmp.get(), tb, k0.get(), k1.get(), i0.get(), i1.get(), (int)nnz, 0, 64, s);
  if (cudaMalloc((void**)&Ly.rec_key, (size_t)(nnz ? nnz : 1) * sizeof(int)) != cudaSuccess ||
      cudaMalloc((void**)&Ly.rec_val, (size_t)(nnz ? nnz : 1) * sizeof(double)) != cudaSuccess) {
    cudaFree(Ly.rec_key);
    Ly.rec_key = nullptr;
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "block record allocation failed");
  }
  if (nnz > 0) {
    gs_launch_begin(ctx, 1);
    k_blk_fill<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(k1.get(), i1.get(), G->cols, G->vals, nnz,
                                                               Ly.rec_key, Ly.rec_val);
    gs_launch_end(ctx, 1);
  }
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// GS_L2_PERSIST=1: the Chebyshev vectors T_{k-1} / T_k (gathered every step) are marked L2-
// persisting through the stream's access-policy window (kernel nodes captured into the sweep
// graphs inherit it), so the once-per-step streams (CSR, T_{k-2}, acc) do not evict them.
struct L2Window {
  cudaStream_t s = nullptr;
  bool on = false;
  L2Window(gs_ctx* ctx, const void* base, size_t bytes) {
    const char* e = getenv("GS_L2_PERSIST");
    if (!(e && atoi(e) != 0) || bytes == 0) return;
    int dev = 0, maxp = 0, maxw = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (maxp <= 0 || maxw <= 0) return;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp) != cudaSuccess) return;
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    v.accessPolicyWindow.num_bytes = std::min(bytes, (size_t)maxw);
    v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)maxp / (double)v.accessPolicyWindow.num_bytes);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    s = ctx->stream;
    on = cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
  }
  ~L2Window() {
    if (!on) return;
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
  }
};

template <typename S>
const void* layout_vals(const gs_layout& L) {
  if constexpr (sizeof(S) == 4) return L.vals32;
  else return L.perm->vals;
}

// Workspace for one batched run: grouped buffers (precision S) + per-column state.
template <typename S>
struct Work {
  int n = 0, B = 0, GW = 1, G = 1, Bpad = 1, tiles = 0, rpc = 1;
  int64_t ld = 0;  // rows per column group: n, or local + halo rows of a row partition
  int lay = 0;  // filter layout: 0 for one-warp-per-row groups, 1 (degree-sorted) for narrower
  bool w1 = false;  // one-column fp64 problem small enough for the warp-per-row kernel
  bool blk = false;  // wide fp64 rows through the 8-row block kernel (k_cheb_blk)
  bool win = false;  // wide rows through the windowed kernel (k_cheb_win, lay[2])
  const gs_winsched* ws = nullptr;
  const gs_sell* sell = nullptr;  // several rows per warp through the sliced kernel (k_cheb_sell)
  int spw = 1;                    // its slices per warp
  bool sellw = false;             // ... through the warp-staged persistent kernel (k_cheb_sellw)
  int tile_period = 0;            // k_cheb_step tiles per degree-sorted window (heaviest-first launch order)
  const void* recs = nullptr;     // fp64 rows shared by several lanes through the record kernel (k_cheb_rec)
  bool lane = false;              // one row per lane through the staged kernel (k_cheb_lane)
  const gs_lanepad* lp = nullptr;  // its odd-stride CSR copy (filter layouts; GS_LANE_PAD=0: none)
  DevBuf<int> wstart;             // its static split of the slices over the grid's warps
  alignas(64) CUtensorMap tmap[2];  // gather sources T[0], T[1] (win)
  struct TView {  // T[0], T[1]: halves of one allocation (one L2 access-policy window covers both)
    S* p = nullptr;
    S* get() const { return p; }
  };
  DevBuf<S> Tall, acc;
  TView T[2];
  DevBuf<unsigned long long> cmin, cmax;
  DevBuf<double> thr, errcol, part_err;
  DevBuf<int> active, gactive;
  DevBuf<gs_status> status;
  // 32-bit mode: the barycenter's psi in fp64 (the fp64 mode keeps it in acc)
  DevBuf<double> psi64;
  static constexpr bool kF32 = sizeof(S) == 4;
  int init(gs_ctx* ctx, int n_, int B_, bool want_err, int64_t ld_ = -1, const gs_filter* f = nullptr) {
    cudaStream_t s = ctx->stream;
    std::unique_lock<std::mutex> build_lock;
    if (f) build_lock = std::unique_lock<std::mutex>(const_cast<gs_filter*>(f)->build_mu);
    n = n_;
    B = B_;
    ld = ld_ < 0 ? n_ : ld_;
    GW = choose_gw(B);
    G = (B + GW - 1) / GW;
    Bpad = G * GW;
    lay = GW >= 32 ? 0 : 1;
    rpc = choose_rpc<S>(n, GW, G, f ? f->lay[lay].near_frac : 1.0);
    tiles = (n + rows_per_block<S>(GW) * rpc - 1) / (rows_per_block<S>(GW) * rpc);
    w1 = GW == 1 && sizeof(S) == 8 && n <= w1_max_rows();
    if (w1) tiles = (n + kThreads / 32 - 1) / (kThreads / 32);
    if (sizeof(S) == 8 && GW == 64 && f && ld_ < 0 && blk_enabled()) {  // not for row partitions
      GS_TRY(gs_build_block_records(ctx, const_cast<gs_filter*>(f), lay));
      blk = true;
      tiles = (n + kBlkRows * kBlkWarps - 1) / (kBlkRows * kBlkWarps);
    } else if (f && ld_ < 0 && n > 0 && win_enabled() && win_row_ok<S>(GW)) {
      const int rb = GW * (int)sizeof(S);
      const int rc = gs_win_build(ctx, const_cast<gs_filter*>(f), rb, (int)sizeof(S));
      if (rc == GS_OK) {
        win = true;
        ws = gs_win_get(f, rb, (int)sizeof(S));
        lay = 2;
        tiles = ws->nctas;
        rpc = 1;
      } else if (rc != GS_ERR_UNSUPPORTED) {
        return rc;
      }
    }
    if (f && ld_ < 0 && n > 0 && !w1 && !blk && !win && sell_enabled() && sell_height<S>(GW) > 0 &&
        (sell_height<S>(GW) <= 8 || sell_c32_enabled())) {
      const int C = sell_height<S>(GW);
      gs_layout& Ly = const_cast<gs_filter*>(f)->lay[lay];
      for (const gs_sell* e : Ly.sell)
        if (e->C == C && e->elem_bytes == (int)sizeof(S)) sell = e;
      if (!sell) {
        gs_sell* e = nullptr;
        GS_TRY(gs_sell_build(ctx, Ly.perm, Ly.vals32, C, (int)sizeof(S), &e));
        Ly.sell.push_back(e);
        sell = e;
      }
      const int warps = kStepThreads / 32;
      if (C <= 8) {  // warp-staged persistent kernel: one wave of CTAs over all column groups
        sellw = true;
        const int occ = std::max(1, sellw_occupancy<S>(GW));
        const int full = (sell->nslices + warps - 1) / warps;
        tiles = std::max(1, std::min(full, (148 * occ + G - 1) / G));
        GS_CUDA(ctx, wstart.alloc((size_t)tiles * warps + 1, s));
        GS_TRY(gs_sell_split(ctx, sell, tiles * warps, wstart.get()));
      } else {
        spw = (int64_t)G * ((sell->nslices + warps * kSellSpw - 1) / (warps * kSellSpw)) < 4 * 148 ? 1 : kSellSpw;
        tiles = (sell->nslices + warps * spw - 1) / (warps * spw);
      }
      rpc = 1;
    }
    if (sizeof(S) == 8 && f && ld_ < 0 && n > 0 && !w1 && !blk && !win && !sell && rpc_lpr<S>(GW) > 1 &&
        rpc_lpr<S>(GW) < 32 && rec_wanted<S>(GW, f)) {
      gs_layout& Ly = const_cast<gs_filter*>(f)->lay[lay];
      if (!Ly.recs) GS_TRY(gs_recs_build(ctx, Ly.perm->cols, Ly.perm->vals, Ly.perm->nnz, &Ly.recs));
      recs = Ly.recs;
    }
    // degree-sorted layout on k_cheb_step / k_cheb_rec: a window of sigma rows spans P tiles whose
    // cost falls from the first (the window's longest rows) to the last; launching every
    // window's first tile, then every second one, ... puts the short tiles into the tail wave
    // Only while the gathered block T_{k-1} fits the L2: the two classes walk the rows twice, and on
    // config 4 (n = 4e6, 512 MB) that second pass costs more than the tail it saves (step 1.485 ->
    // 1.581 ms), while config 2 (64 MB) gains 10% and the config-4 shape at n = 1e6 (128 MB) 3%.
    if (f && ld_ < 0 && lay == 1 && !w1 && !blk && !win && !sell && f->sigma > 0 && heavy_first_enabled() &&
        (size_t)n_ * (size_t)Bpad * sizeof(S) <= l2_bytes()) {
      const int tile_rows = rows_per_block<S>(GW) * rpc;
      if (f->sigma % tile_rows == 0 && f->sigma / tile_rows >= 2 && f->sigma / tile_rows <= 256)
        tile_period = f->sigma / tile_rows;
    }
    lane = !w1 && !blk && !win && !sell && rpc > 1 && rpc_lpr<S>(GW) == 1 && lane_enabled();
    if (lane && f && ld_ < 0 && n > 0 && lane_pad_enabled()) {
      gs_layout& Ly = const_cast<gs_filter*>(f)->lay[lay];
      for (const gs_lanepad* e : Ly.lanepad)
        if (e->elem_bytes == (int)sizeof(S)) lp = e;
      if (!lp) {
        gs_lanepad* e = nullptr;
        const int rc = gs_lanepad_build(ctx, Ly.perm->offs, Ly.perm->cols, layout_vals<S>(Ly), (int)sizeof(S), n,
                                        Ly.perm->nnz, &e);
        if (rc == GS_OK) {
          Ly.lanepad.push_back(e);
          lp = e;
        } else if (rc != GS_ERR_UNSUPPORTED) {
          return rc;
        }
      }
    }
    const size_t len = (size_t)Bpad * (ld > 0 ? ld : 1);
    GS_CUDA(ctx, Tall.alloc(2 * len, s));
    T[0].p = Tall.get();
    T[1].p = Tall.get() + len;
    if (win)
      for (int h = 0; h < 2; ++h)
        GS_TRY(gs_win_tensor_map(ctx, &tmap[h], T[h].p, (int64_t)G * ld, GW, (int)sizeof(S)));
    GS_CUDA(ctx, acc.alloc(len, s));
    GS_CUDA(ctx, cmin.alloc(Bpad, s));
    GS_CUDA(ctx, cmax.alloc(Bpad, s));
    GS_CUDA(ctx, thr.alloc(Bpad, s));
    GS_CUDA(ctx, errcol.alloc(Bpad, s));
    GS_CUDA(ctx, part_err.alloc(want_err ? (size_t)tiles * Bpad : 1, s));
    GS_CUDA(ctx, active.alloc(Bpad, s));
    GS_CUDA(ctx, gactive.alloc(G, s));
    {
      std::vector<int> ga(G);
      for (int g = 0; g < G; ++g) ga[g] = std::min(GW, B - g * GW);
      GS_CUDA(ctx, cudaMemcpyAsync(gactive.get(), ga.data(), G * sizeof(int), cudaMemcpyHostToDevice, s));
      GS_CUDA(ctx, cudaStreamSynchronize(s));
    }
    if constexpr (kF32) GS_CUDA(ctx, psi64.alloc(len, s));
    GS_CUDA(ctx, status.alloc(1, s));
    GS_CUDA(ctx, cudaMemsetAsync(status.get(), 0, sizeof(gs_status), s));
    GS_CUDA(ctx, cudaMemsetAsync(thr.get(), 0, Bpad * sizeof(double), s));
    GS_CUDA(ctx, cudaMemsetAsync(errcol.get(), 0, Bpad * sizeof(double), s));
    gs_launch_begin(ctx, 1);
    k_fill_key<<<grid_for(Bpad), kThreads, 0, s>>>(cmin.get(), Bpad, KEY_POS_INF);
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_fill_key<<<grid_for(Bpad), kThreads, 0, s>>>(cmax.get(), Bpad, KEY_ZERO);
    gs_launch_end(ctx, 1);
    return GS_OK;
  }
  ColState cs() {
    ColState c;
    c.active = active.get();
    c.gactive = gactive.get();
    c.cmin = cmin.get();
    c.cmax = cmax.get();
    c.thr = thr.get();
    c.errcol = errcol.get();
    c.part_err = part_err.get();
    return c;
  }
};

// Deferred-accumulation schedule (StepArgs::acc_terms): step k holds the own rows T_{k-2},
// T_{k-1}, T_k, so acc may lag by up to two steps; it is brought up to date whenever waiting one
// more step would leave a pending term out of reach, and at the last step. K = 30 updates acc at
// steps 2, 5, ..., 29, 30 instead of every step.
struct AccSchedule {
  int last = 0;       // highest T index already in acc
  bool init = false;  // acc holds (b_0 / 2) T_0 + ...
  void step(const gs_filter* f, int K, int k, StepArgs& A) {
    const bool must = k == K || (!init && k >= 2) || (init && last < k - 2);
    A.acc_terms = must ? k - last : 0;
    A.acc_init = must && !init;
    A.store_t = k < K;
    A.bk1 = k >= 1 ? f->coeffs[k - 1] : 0.0;
    A.bk2 = k >= 2 ? f->coeffs[k - 2] : 0.0;
    if (must) {
      last = k;
      init = true;
    }
  }
};

// One full filter application on the workspace: T0 in T[a0]; K steps; the last step uses `mode`
// with the given epilogue operands. Returns the buffer index holding the next T_0.
// BARY_PSI applies: the log-domain geometric mean fused into the last step's epilogue
struct BaryFuse {
  double* lb;
  const double* alphas;
  unsigned long long* lbmax;
  int m;
};

template <typename S>
int run_apply(gs_ctx* ctx, const gs_filter* f, Work<S>& w, int a0, int mode, const double* a,
              const double* M, const double* Vcur, double* Wout, bool use_active, bool use_status,
              const BaryFuse* bf = nullptr) {
  const gs_layout& Ly = f->lay[w.lay];
  const gs_graph* G = Ly.perm;
  const int K = f->degree;
  StepArgs A{};
  A.offs = G->offs;
  A.cols = G->cols;
  A.vals = layout_vals<S>(Ly);
  A.warp_rows = w.w1;
  A.lane = w.lane;
  A.recs = w.recs;
  A.tile_period = w.tile_period;
  if (w.lp) {
    A.offs = w.lp->offs;
    A.cols = w.lp->cols;
    A.vals = w.lp->vals;
  }
  if (w.blk) {
    A.rec_key = Ly.rec_key;
    A.rec_val = Ly.rec_val;
  }
  A.n = w.n;
  A.ld = w.ld;
  A.tiles = w.tiles;
  A.g0 = 0;
  A.Gl = w.G;
  A.Bpad = w.Bpad;
  A.acc = w.acc.get();
  A.b0h = f->coeffs[0] / 2.0;
  A.status = use_status ? w.status.get() : nullptr;
  A.cs = w.cs();
  if (!use_active) {
    A.cs.active = nullptr;
    A.cs.gactive = nullptr;
  }
  A.a = a;
  A.M = M;
  A.Vcur = Vcur;
  A.Wout = Wout;
  A.psi = w.psi64.get();
  if (bf && mode == MODE_BARY_PSI) {
    A.lb = bf->lb;
    A.alphas = bf->alphas;
    A.lbmax = bf->lbmax;
    A.m = bf->m;
  }
  WinArgs WA{};
  if (w.win) {
    WA.blk = static_cast<const WinBlk*>(w.ws->blk);
    WA.cta_blk = w.ws->cta_blk;
    WA.loads = w.ws->loads;
    WA.slot = w.ws->slot;
    WA.own = w.ws->own;
    WA.poffs = w.ws->poffs;
    WA.pvals = w.ws->pvals;
    WA.W = w.ws->W;
    WA.nctas = w.ws->nctas;
  }
  SellArgs SE{};
  if (w.sell) {
    SE.soff = w.sell->soff;
    SE.cols = w.sell->cols;
    SE.vals = w.sell->vals;
    SE.nslices = w.sell->nslices;
    SE.wstart = w.wstart.get();
  }
  // GS_WIN_CTATIME=1 (diagnostics): per-CTA start/end times of the apply's steps, summarised on
  // stderr (the tail of the persistent grid)
  static const bool ctatime = getenv("GS_WIN_CTATIME") && atoi(getenv("GS_WIN_CTATIME")) != 0;
  DevBuf<unsigned long long> ctt;
  if (w.win && ctatime) {
    GS_CUDA(ctx, ctt.alloc((size_t)2 * w.ws->nctas * w.G * K, ctx->stream));
  }
  const bool seq = seq_groups() && w.G > 1 && !w.win;
  for (int g = 0; g < (seq ? w.G : 1); ++g) {
    if (seq) {
      A.g0 = g;
      A.Gl = 1;
    }
    AccSchedule sched;
    for (int k = 1; k <= K; ++k) {
      A.k = k;
      A.bk = f->coeffs[k];
      sched.step(f, K, k, A);
      A.Tprev = w.T[(a0 + k - 1) & 1].get();
      A.Tout = w.T[(a0 + k) & 1].get();
      if (w.win && ctt.get()) WA.ctatime = ctt.get() + (size_t)2 * w.ws->nctas * w.G * (k - 1);
      if (w.win) launch_step_win<S>(ctx, w.GW, w.tmap[(a0 + k - 1) & 1], A, WA, k == K ? mode : MODE_NONE);
      else if (w.sellw) launch_step_sellw<S>(ctx, w.GW, A, SE, k == K ? mode : MODE_NONE);
      else if (w.sell) launch_step_sell<S>(ctx, w.GW, w.spw, A, SE, k == K ? mode : MODE_NONE);
      else launch_step<S>(ctx, w.GW, w.rpc, A, k == K ? mode : MODE_NONE);
    }
  }
  if (ctt.get()) {
    const int nb = w.ws->nctas * w.G;
    std::vector<unsigned long long> h((size_t)2 * nb * K);
    GS_CUDA(ctx, cudaMemcpyAsync(h.data(), ctt.get(), h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    for (int k = 1; k <= K; ++k) {
      const unsigned long long* t = h.data() + (size_t)2 * nb * (k - 1);
      unsigned long long s0 = ~0ull, e1 = 0;
      std::vector<double> dur(nb), endt(nb);
      for (int b = 0; b < nb; ++b) s0 = std::min(s0, t[2 * b]);
      for (int b = 0; b < nb; ++b) {
        dur[b] = (t[2 * b + 1] - t[2 * b]) * 1e-3;
        endt[b] = (t[2 * b + 1] - s0) * 1e-3;
        e1 = std::max(e1, t[2 * b + 1]);
      }
      std::sort(dur.begin(), dur.end());
      std::sort(endt.begin(), endt.end());
      fprintf(stderr, "[win step %2d] CTA duration us: min %.1f med %.1f max %.1f | end times: med %.1f p90 %.1f max %.1f\n",
              k, dur[0], dur[nb / 2], dur[nb - 1], endt[nb / 2], endt[nb * 9 / 10], endt[nb - 1]);
    }
  }
  return (a0 + K) & 1;
}

template <typename S>
void run_finalize(gs_ctx* ctx, Work<S>& w, int check, int has_next, int has_err, int knp_code,
                  bool use_active) {
  FinArgs F{};
  F.cs = w.cs();
  if (!use_active) F.cs.active = nullptr;
  F.B = w.B;
  F.tiles = w.tiles;
  F.Bpad = w.Bpad;
  F.check = check;
  F.has_next = has_next;
  F.has_err = has_err;
  F.status = w.status.get();
  F.knp_code = knp_code;
  F.slack = Prec<S>::slack;
  gs_launch_begin(ctx, 1);
  k_finalize<<<w.B, kThreads, 0, ctx->stream>>>(F);
  gs_launch_end(ctx, 1);
}

// Input staging: returns a device pointer to `count` doubles (the caller's when mem = DEVICE).
int stage_in(gs_ctx* ctx, DevBuf<double>& buf, const double* src, size_t count, int mem,
             const double** out) {
  if (mem == GS_MEM_DEVICE) {
    *out = src;
    return GS_OK;
  }
  GS_CUDA(ctx, buf.alloc(count, ctx->stream));
  GS_CUDA(ctx, cudaMemcpyAsync(buf.get(), src, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  *out = buf.get();
  return GS_OK;
}

int finish_out(gs_ctx* ctx, DevBuf<double>& buf, double* dst, size_t count, int mem) {
  if (mem == GS_MEM_DEVICE) return GS_OK;
  GS_CUDA(ctx, cudaMemcpyAsync(dst, buf.get(), count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  return GS_OK;
}

int validate_columns(gs_ctx* ctx, const double* d, int n, int P, std::vector<double>& sums,
                     std::vector<int>& nonfinite, std::vector<int>& negative) {
  cudaStream_t s = ctx->stream;
  DevBuf<double> dsum;
  DevBuf<int> dnf, dng;
  GS_CUDA(ctx, dsum.alloc(P, s));
  GS_CUDA(ctx, dnf.alloc(P, s));
  GS_CUDA(ctx, dng.alloc(P, s));
  GS_CUDA(ctx, cudaMemsetAsync(dnf.get(), 0, P * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(dng.get(), 0, P * sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_validate_cols<<<dim3(1, P), kThreads, 0, s>>>(d, n, dsum.get(), dnf.get(), dng.get());
  gs_launch_end(ctx, 1);
  sums.resize(P);
  nonfinite.resize(P);
  negative.resize(P);
  GS_CUDA(ctx, cudaMemcpyAsync(sums.data(), dsum.get(), P * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(nonfinite.data(), dnf.get(), P * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(negative.data(), dng.get(), P * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// Distribution::validate (transport.cpp:96-102) for one column
int check_distribution(gs_ctx* ctx, int n, double sum, int nonfinite, int negative) {
  if (n < 1) return gs_fail(ctx, ERRC_LENGTH_MISMATCH, "empty distribution");
  if (nonfinite) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "non-finite weights");
  if (negative) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "negative weights");
  if (!(std::fabs(sum - 1.0) <= 1e-12)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "distribution must sum to 1");
  return GS_OK;
}

int check_weights(gs_ctx* ctx, const double* da, int n) {
  DevBuf<int> bad;
  GS_CUDA(ctx, bad.alloc(1, ctx->stream));
  GS_CUDA(ctx, cudaMemsetAsync(bad.get(), 0, sizeof(int), ctx->stream));
  if (n > 0) {
    gs_launch_begin(ctx, 1);
    k_validate_weights<<<(n + 255) / 256, 256, 0, ctx->stream>>>(da, n, bad.get());
    gs_launch_end(ctx, 1);
  }
  int h = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return h ? gs_fail(ctx, ERRC_INVALID_ARGUMENT, "vertex weights must be positive") : GS_OK;
}

const char* kKnpTransport =
    "heat approximation produced negative mass; increase the degree or diffusion time";
// 32-bit mode: a non-finite marginal error or cost is reported, never returned as a value (the
// fp64 reference returns -inf costs for pairs whose v underflows; the 32-bit mode raises
// numerical_underflow for them, transport.cpp:284-289's errc)
const std::string kF32Range_msg = "fp32 mode: non-finite marginal error or cost; rerun in fp64. Pair ";
const char* kKnpBary =
    "heat filter produced negative mass; increase the Chebyshev degree or diffusion time";

// ---- filter apply (heat.cpp:116-131) -----------------------------------------------------------
template <typename S>
int filter_apply_impl(gs_ctx* ctx, const gs_filter* f, const double* dX, double* dY, int width) {
  const int n = f->scaled->n;
  cudaStream_t s = ctx->stream;
  Work<S> w;
  GS_TRY(w.init(ctx, n, width, false, -1, f));
  gs_launch_begin(ctx, 1);
  k_pack<S><<<grid_for((int64_t)w.Bpad * n), kThreads, 0, s>>>(dX, w.T[0].get(), n, width, w.GW, w.G, f->lay[w.lay].order, (int64_t)n);
  gs_launch_end(ctx, 1);
  run_apply<S>(ctx, f, w, 0, MODE_NONE, nullptr, nullptr, nullptr, nullptr, false, false);
  gs_launch_begin(ctx, 1);
  k_unpack<S><<<grid_for((int64_t)width * n), kThreads, 0, s>>>(w.acc.get(), dY, n, width, w.GW, nullptr, nullptr, f->lay[w.lay].newpos, (int64_t)n);
  gs_launch_end(ctx, 1);
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// fp32 mode: a non-finite cost is numerical_underflow (first such pair in pair order)
int check_finite_costs(gs_ctx* ctx, const double* dcost, int P) {
  std::vector<double> h(P);
  GS_CUDA(ctx, cudaMemcpyAsync(h.data(), dcost, P * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  for (int q = 0; q < P; ++q)
    if (!std::isfinite(h[q])) return gs_fail(ctx, ERRC_NUMERICAL_UNDERFLOW, kF32Range_msg + std::to_string(q));
  return GS_OK;
}

// ---- geodesic Sinkhorn batch (transport.cpp:108-255) --------------------------------------------
template <typename S>
int sinkhorn_impl(gs_ctx* ctx, const gs_filter* f, const double* da_user, const double* dmu,
                  const double* dnu, int P, int max_iter, double tol, int flags, int mem,
                  double* out_v, double* out_w, double* out_cost, double* out_kl, int* out_iters,
                  int* out_conv, double* out_err, int* fail_pair, int* fail_sweep) {
  const int n = f->scaled->n;
  cudaStream_t s = ctx->stream;
  Work<S> w;
  GS_TRY(w.init(ctx, n, P, true, -1, f));
  L2Window l2w(ctx, w.Tall.get(), w.Tall.n * sizeof(S));
  // vertex weights in the filter's locality order (the epilogue state is fp64 in both modes)
  DevBuf<double> aperm;
  GS_CUDA(ctx, aperm.alloc(n, s));
  gs_launch_begin(ctx, 1);
  k_gather_to<double><<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(da_user, f->lay[w.lay].order, n, aperm.get());
  gs_launch_end(ctx, 1);
  const double* da = aperm.get();
  const size_t len = (size_t)w.Bpad * n;
  DevBuf<double> M, N, V[2], W;
  GS_CUDA(ctx, M.alloc(len, s));
  GS_CUDA(ctx, N.alloc(len, s));
  GS_CUDA(ctx, V[0].alloc(len, s));
  GS_CUDA(ctx, V[1].alloc(len, s));
  GS_CUDA(ctx, W.alloc(len, s));
  DevBuf<int> iters, conv, stag, final_sweep;
  DevBuf<double> errv;
  GS_CUDA(ctx, iters.alloc(w.Bpad, s));
  GS_CUDA(ctx, conv.alloc(w.Bpad, s));
  GS_CUDA(ctx, stag.alloc(w.Bpad, s));
  GS_CUDA(ctx, final_sweep.alloc(w.Bpad, s));
  GS_CUDA(ctx, errv.alloc(w.Bpad, s));
  GS_CUDA(ctx, cudaMemsetAsync(iters.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(conv.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(stag.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(final_sweep.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(V[0].get(), 0, len * sizeof(double), s));
  GS_CUDA(ctx, cudaMemsetAsync(W.get(), 0, len * sizeof(double), s));
  {
    std::vector<int> act(w.Bpad, 0);
    for (int p = 0; p < P; ++p) act[p] = 1;
    GS_CUDA(ctx, cudaMemcpyAsync(w.active.get(), act.data(), w.Bpad * sizeof(int), cudaMemcpyHostToDevice, s));
    std::vector<double> inf(w.Bpad, INFINITY);
    GS_CUDA(ctx, cudaMemcpyAsync(errv.get(), inf.data(), w.Bpad * sizeof(double), cudaMemcpyHostToDevice, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
  }
  gs_launch_begin(ctx, 1);
  k_pack<double><<<grid_for((int64_t)len), kThreads, 0, s>>>(dmu, M.get(), n, P, w.GW, w.G, f->lay[w.lay].order, (int64_t)n);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_pack<double><<<grid_for((int64_t)len), kThreads, 0, s>>>(dnu, N.get(), n, P, w.GW, w.G, f->lay[w.lay].order, (int64_t)n);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_sk_init<S><<<grid_for((int64_t)len), kThreads, 0, s>>>(da, w.T[0].get(), n, w.GW, w.G, P, w.cmax.get(), (int64_t)n);
  gs_launch_end(ctx, 1);
  const int knp = ERRC_KERNEL_NOT_POSITIVE + 1;
  run_finalize<S>(ctx, w, 0, 1, 0, knp, true);  // threshold of the first apply
  // phi = H(a * 1) (transport.cpp:176); V_1 = M / max(phi, floor) in the epilogue
  int a0 = run_apply<S>(ctx, f, w, 0, MODE_SK_PHI, da, M.get(), V[0].get(), V[1].get(), true, true);
  run_finalize<S>(ctx, w, 1, 1, 0, knp, true);
  gs_status* hst = ctx->h_status;
  cudaEvent_t ev[2];
  cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
  CtlArgs C{};
  C.active = w.active.get();
  C.gactive = w.gactive.get();
  C.GW = w.GW;
  C.errcol = w.errcol.get();
  C.iters = iters.get();
  C.conv = conv.get();
  C.stag = stag.get();
  C.final_sweep = final_sweep.get();
  C.err_out = errv.get();
  C.status = w.status.get();
  C.P = P;
  C.max_iter = max_iter;
  C.no_abort = (flags & GS_FLAG_NO_STAGNATION_ABORT) ? 1 : 0;
  C.fp32 = w.kF32 ? 1 : 0;
  C.tol = tol;
  DevBuf<int> sweep_ctr;
  GS_CUDA(ctx, sweep_ctr.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(sweep_ctr.get(), 0, sizeof(int), s));
  C.sweep_ctr = sweep_ctr.get();
  // one sweep (transport.cpp:177-227); `parity` selects the V ping-pong buffers
  auto issue_sweep = [&](int parity) {
    // psi = H(a * V_s); W_s = N / max(psi, floor); T_0 = a * W_s
    a0 = run_apply<S>(ctx, f, w, a0, MODE_SK_PSI, da, N.get(), nullptr, W.get(), true, true);
    run_finalize<S>(ctx, w, 1, 1, 0, knp, true);
    // phi = H(a * W_s); err; V_{s+1} = M / max(phi, floor); T_0 = a * V_{s+1}
    a0 = run_apply<S>(ctx, f, w, a0, MODE_SK_PHI, da, M.get(), V[parity].get(), V[parity ^ 1].get(),
                      true, true);
    run_finalize<S>(ctx, w, 1, 1, 1, knp, true);
    gs_launch_begin(ctx, 1);
    k_sk_control<<<1, 1, 0, s>>>(C);
    gs_launch_end(ctx, 1);
  };
  // Small one-pair fp64 problems (config 0): every sweep in one persistent cluster kernel
  // (gs_persist.cuh); GS_PERSIST=0 keeps the per-step kernels.
  bool persisted = false;
  if constexpr (sizeof(S) == 8) {
    const char* penv = getenv("GS_PERSIST");
    const bool want = penv ? penv[0] != '0' : true;
    static const int CL = [] {  // CTAs per cluster (GS_PERSIST_CLUSTER: 8 portable, 16 opt-in)
      const char* e = getenv("GS_PERSIST_CLUSTER");
      const int v = e ? atoi(e) : 16;
      return v >= 2 && v <= kPersistClusterMax ? v : 16;
    }();
    const int kPersistCluster = CL;
    const int R = (n + kPersistCluster - 1) / kPersistCluster;
    if (want && P == 1 && w.GW == 1 && n >= kPersistCluster && R <= kPersistMaxRows && n <= kPersistMaxN) {
      const gs_graph* G = f->lay[w.lay].perm;
      std::vector<int> ho(n + 1);
      GS_CUDA(ctx, cudaMemcpyAsync(ho.data(), G->offs, (size_t)(n + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
      GS_CUDA(ctx, cudaStreamSynchronize(s));
      // ELL slice of the largest CTA: per warp of 32 rows, 32 x its longest row
      int64_t maxne = 0;
      for (int r = 0; r < kPersistCluster; ++r) {
        const int r0 = std::min(n, r * R), r1 = std::min(n, r0 + R);
        int64_t ne = 0;
        for (int w0 = r0; w0 < r1; w0 += 32) {
          int md = 0;
          for (int i = w0; i < std::min(r1, w0 + 32); ++i) md = std::max(md, ho[i + 1] - ho[i]);
          ne += 32 * (int64_t)md;
        }
        maxne = std::max(maxne, ne);
      }
      const size_t smem = (size_t)persist_rep_offset(n) + (size_t)2 * n * 8 + (size_t)maxne * 12;
      if (smem <= 220 * 1024) {  // + 768 bytes of static shared memory
        static std::vector<char> seen;  // the attributes are per device
        gs_once_per_device(seen, [] {
          cudaFuncSetAttribute(k_sk_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
          cudaFuncSetAttribute(k_sk_persist, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        });
        PersistArgs PA{};
        PA.n = n;
        PA.R = R;
        PA.K = f->degree;
        PA.max_iter = max_iter;
        PA.no_abort = (flags & GS_FLAG_NO_STAGNATION_ABORT) ? 1 : 0;
        PA.tol = tol;
        PA.slack = Prec<S>::slack;
        PA.coeffs = f->d_coeffs;
        PA.offs = G->offs;
        PA.cols = G->cols;
        PA.vals = G->vals;
        PA.a = da;
        PA.M = M.get();
        PA.N = N.get();
        PA.V0 = V[0].get();
        PA.V1 = V[1].get();
        PA.W = W.get();
        PA.T0 = reinterpret_cast<const double*>(w.T[a0].get());
        PA.thr = w.thr.get();
        PA.iters = iters.get();
        PA.conv = conv.get();
        PA.stag = stag.get();
        PA.final_sweep = final_sweep.get();
        PA.err_out = errv.get();
        PA.status = w.status.get();
        PA.knp_code = knp;
        const int threads = (R + 31) / 32 * 32;
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(kPersistCluster);
        lc.blockDim = dim3(threads);
        lc.dynamicSmemBytes = smem;
        lc.stream = s;
        cudaLaunchAttribute la[1];
        la[0].id = cudaLaunchAttributeClusterDimension;
        la[0].val.clusterDim.x = kPersistCluster;
        la[0].val.clusterDim.y = 1;
        la[0].val.clusterDim.z = 1;
        lc.attrs = la;
        lc.numAttrs = 1;
        gs_launch_begin(ctx, 0);
        GS_CUDA(ctx, cudaLaunchKernelEx(&lc, k_sk_persist, PA));
        gs_launch_end(ctx, 0);
        GS_CUDA(ctx, cudaGetLastError());
        persisted = true;
      }
    }
  }
  // Two sweeps (odd, even parity) are captured once as a CUDA graph and replayed: one host launch
  // per two sweeps instead of ~126, so the GPU never waits on the host's launch path (small
  // problems are launch-latency bound; on config 1 per-kernel launches left 11-25% of the GPU idle
  // under host-side stalls). Kernels of sweeps past convergence / max_iter exit immediately.
  // GS_GRAPH=0 selects per-kernel launches.
  const char* genv = getenv("GS_GRAPH");
  const bool use_graph = genv ? genv[0] != '0' : true;
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_launches = 0;
  if (!persisted && use_graph && max_iter >= 2) {
    cudaGraph_t graph = nullptr;
    const int64_t l0 = ctx->launches;
    ctx->capturing = true;
    cudaError_t ce = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (ce == cudaSuccess) {
      issue_sweep(1);
      issue_sweep(0);
      ce = cudaStreamEndCapture(s, &graph);
    }
    ctx->capturing = false;
    graph_launches = ctx->launches - l0;
    ctx->launches = l0;
    if (ce == cudaSuccess) ce = cudaGraphInstantiate(&gexec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (ce != cudaSuccess) {
      cudaGetLastError();
      gexec = nullptr;
    }
  }
  const int step_sweeps = gexec ? 2 : 1;
  for (int sweep = 1, it = 0; !persisted && sweep <= max_iter; sweep += step_sweeps, ++it) {
    if (it >= 2) {
      const int slot = (it - 2) & 1;
      cudaEventSynchronize(ev[slot]);
      const gs_status st = hst[slot];
      if (st.error || st.n_active == 0) break;
    }
    if (gexec) {
      GS_CUDA(ctx, cudaGraphLaunch(gexec, s));
      ctx->launches += graph_launches;
    } else {
      issue_sweep(sweep & 1);
    }
    const int slot = it & 1;
    cudaMemcpyAsync(&hst[slot], w.status.get(), sizeof(gs_status), cudaMemcpyDeviceToHost, s);
    cudaEventRecord(ev[slot], s);
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  gs_status st;
  GS_CUDA(ctx, cudaMemcpy(&st, w.status.get(), sizeof st, cudaMemcpyDeviceToHost));
  if (st.error) {
    if (st.error == ERRC_DISCONNECTED + 1) {
      if (fail_pair) *fail_pair = st.fail_pair;
      if (fail_sweep) *fail_sweep = st.fail_sweep;
      if (flags & GS_FLAG_SINGLE)
        return gs_fail(ctx, ERRC_DISCONNECTED,
                       "marginal error stagnated above 0.5; are mu and nu in the same graph component?");
      return gs_fail(ctx, ERRC_DISCONNECTED,
                     "marginal error stagnated above 0.5 for pair " + std::to_string(st.fail_pair));
    }
    if (st.error == ERRC_NUMERICAL_UNDERFLOW + 1) {
      if (fail_pair) *fail_pair = st.fail_pair;
      if (fail_sweep) *fail_sweep = st.fail_sweep;
      return gs_fail(ctx, ERRC_NUMERICAL_UNDERFLOW, kF32Range_msg + std::to_string(st.fail_pair));
    }
    return gs_fail(ctx, ERRC_KERNEL_NOT_POSITIVE, kKnpTransport);
  }
  // ---- cost / KL + outputs ------------------------------------------------------------------------
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  DevBuf<double> part, dcost, dkl;
  GS_CUDA(ctx, part.alloc((size_t)nchunks * P * 4, s));
  GS_CUDA(ctx, dcost.alloc(P, s));
  GS_CUDA(ctx, dkl.alloc(P, s));
  gs_launch_begin(ctx, 1);
  k_sk_cost_partial<double><<<dim3((unsigned)nchunks, P), kThreads, 0, s>>>(
      da, M.get(), N.get(), V[0].get(), V[1].get(), W.get(), final_sweep.get(), n, w.GW, part.get(), P,
      (int64_t)n);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_sk_cost_final<<<(P + 63) / 64, 64, 0, s>>>(part.get(), nchunks, P, 4.0 * f->t, dcost.get(), dkl.get());
  gs_launch_end(ctx, 1);
  if (w.kF32) GS_TRY(check_finite_costs(ctx, dcost.get(), P));
  DevBuf<double> ov, ow;
  double* dv = out_v;
  double* dw = out_w;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, ov.alloc((size_t)P * n, s));
    GS_CUDA(ctx, ow.alloc((size_t)P * n, s));
    dv = ov.get();
    dw = ow.get();
  }
  if (out_v) {
    gs_launch_begin(ctx, 1);
    k_unpack<double><<<grid_for((int64_t)P * n), kThreads, 0, s>>>(V[0].get(), dv, n, P, w.GW, V[1].get(), final_sweep.get(), f->lay[w.lay].newpos, (int64_t)n);
    gs_launch_end(ctx, 1);
    GS_TRY(finish_out(ctx, ov, out_v, (size_t)P * n, mem));
  }
  if (out_w) {
    gs_launch_begin(ctx, 1);
    k_unpack<double><<<grid_for((int64_t)P * n), kThreads, 0, s>>>(W.get(), dw, n, P, w.GW, nullptr, nullptr, f->lay[w.lay].newpos, (int64_t)n);
    gs_launch_end(ctx, 1);
    GS_TRY(finish_out(ctx, ow, out_w, (size_t)P * n, mem));
  }
  auto out_small = [&](void* dst, const void* src, size_t bytes) -> int {
    if (!dst) return GS_OK;
    GS_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes,
                                 mem == GS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    return GS_OK;
  };
  GS_TRY(out_small(out_cost, dcost.get(), P * sizeof(double)));
  GS_TRY(out_small(out_kl, dkl.get(), P * sizeof(double)));
  GS_TRY(out_small(out_iters, iters.get(), P * sizeof(int)));
  GS_TRY(out_small(out_conv, conv.get(), P * sizeof(int)));
  GS_TRY(out_small(out_err, errv.get(), P * sizeof(double)));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// ---- barycenter (barycenter.cpp:45-107) ------------------------------------------------------------
template <typename S>
int barycenter_impl(gs_ctx* ctx, const gs_filter* f, const double* da_user, const double* dmem, int m,
                    const std::vector<double>& al, int max_iter, double tol, int mem,
                    const gs_comm* comm, double* out_bary, double* out_V, double* out_W,
                    int* out_iters, int* out_conv, double* out_err) {
  const int n = f->scaled->n;
  cudaStream_t s = ctx->stream;
  Work<S> w;
  GS_TRY(w.init(ctx, n, m, true, -1, f));
  L2Window l2w(ctx, w.Tall.get(), w.Tall.n * sizeof(S));
  DevBuf<double> aperm;
  GS_CUDA(ctx, aperm.alloc(n, s));
  gs_launch_begin(ctx, 1);
  k_gather_to<double><<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(da_user, f->lay[w.lay].order, n, aperm.get());
  gs_launch_end(ctx, 1);
  const double* da = aperm.get();
  const size_t len = (size_t)w.Bpad * n;
  DevBuf<double> Mb, V[2], W;
  DevBuf<double> lb, bary, part, mass, dal, errbuf, derr;
  DevBuf<unsigned long long> lbmax;
  DevBuf<int> diters, dconv;
  GS_CUDA(ctx, Mb.alloc(len, s));
  GS_CUDA(ctx, V[0].alloc(len, s));
  GS_CUDA(ctx, V[1].alloc(len, s));
  GS_CUDA(ctx, W.alloc(len, s));
  GS_CUDA(ctx, lb.alloc(n, s));
  GS_CUDA(ctx, bary.alloc(n, s));
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  GS_CUDA(ctx, part.alloc(nchunks, s));
  GS_CUDA(ctx, mass.alloc(1, s));
  GS_CUDA(ctx, dal.alloc(m, s));
  GS_CUDA(ctx, errbuf.alloc(2, s));
  GS_CUDA(ctx, derr.alloc(1, s));
  GS_CUDA(ctx, lbmax.alloc(1, s));
  GS_CUDA(ctx, diters.alloc(1, s));
  GS_CUDA(ctx, dconv.alloc(1, s));
  GS_CUDA(ctx, cudaMemcpyAsync(dal.get(), al.data(), m * sizeof(double), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemsetAsync(V[0].get(), 0, len * sizeof(double), s));
  GS_CUDA(ctx, cudaMemsetAsync(diters.get(), 0, sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(dconv.get(), 0, sizeof(int), s));
  {
    const double inf = INFINITY;
    GS_CUDA(ctx, cudaMemcpyAsync(derr.get(), &inf, sizeof(double), cudaMemcpyHostToDevice, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
  }
  gs_launch_begin(ctx, 1);
  k_fill<<<grid_for(n), kThreads, 0, s>>>(bary.get(), n, 1.0 / n);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_pack<double><<<grid_for((int64_t)len), kThreads, 0, s>>>(dmem, Mb.get(), n, m, w.GW, w.G, f->lay[w.lay].order, (int64_t)n);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_sk_init<S><<<grid_for((int64_t)len), kThreads, 0, s>>>(da, w.T[0].get(), n, w.GW, w.G, m, w.cmax.get(), (int64_t)n);
  gs_launch_end(ctx, 1);
  run_finalize<S>(ctx, w, 0, 1, 0, 0, false);
  const int knp = ERRC_KERNEL_NOT_POSITIVE + 1;
  // phi = H(a * 1) (barycenter.cpp:68); V_1 = M / max(phi, floor) in the epilogue
  int a0 = run_apply<S>(ctx, f, w, 0, MODE_SK_PHI, da, Mb.get(), V[0].get(), V[1].get(), false, true);
  run_finalize<S>(ctx, w, 1, 1, 0, knp, false);
  gs_status* hst = ctx->h_status;
  cudaEvent_t ev[2];
  cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
  DevBuf<int> sweep_ctr;
  GS_CUDA(ctx, sweep_ctr.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(sweep_ctr.get(), 0, sizeof(int), s));
  const bool hooked = comm && comm->allreduce;
  int hook_rc = 0;
  // one sweep (barycenter.cpp:70-86); `parity` selects the V ping-pong buffers. Kernels of sweeps
  // past convergence / max_iter exit on the status word (or recompute unchanged values).
  // the log-sum (and, unsharded, its max) computed in the psi apply's last-step epilogue for one
  // column group (m <= 64); GS_BARY_UNFUSED=1 keeps the separate passes (k_bary_lb, k_max_key)
  const bool fuse = w.G == 1 && !(getenv("GS_BARY_UNFUSED") && atoi(getenv("GS_BARY_UNFUSED")) != 0);
  const BaryFuse bfuse{lb.get(), dal.get(), lbmax.get(), m};
  auto issue_sweep = [&](int parity) -> int {
    // psi = H(a * V) (barycenter.cpp:71)
    if (fuse) cudaMemsetAsync(lbmax.get(), 0, sizeof(unsigned long long), s);
    a0 = run_apply<S>(ctx, f, w, a0, MODE_BARY_PSI, da, nullptr, nullptr, nullptr, false, true,
                      fuse ? &bfuse : nullptr);
    run_finalize<S>(ctx, w, 1, 0, 0, knp, false);
    // log-domain geometric mean (barycenter.cpp:75-82)
    // psi in fp64: acc in the fp64 mode, psi64 in the 32-bit mode
    const double* psi = w.kF32 ? w.psi64.get() : reinterpret_cast<const double*>(w.acc.get());
    if (!fuse) {
      gs_launch_begin(ctx, 1);
      k_bary_lb<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(psi, dal.get(), n, m, w.GW, lb.get(), w.status.get());
      gs_launch_end(ctx, 1);
    }
    if (hooked) {
      const int rc = comm->allreduce(comm->user, lb.get(), n, 0, (void*)s);
      if (rc) return rc;
    }
    if (!fuse || hooked) {  // the max of the (allreduced) log-sum
      cudaMemsetAsync(lbmax.get(), 0, sizeof(unsigned long long), s);
      gs_launch_begin(ctx, 1);
      k_max_key<<<grid_for(n), kThreads, 0, s>>>(lb.get(), n, lbmax.get());
      gs_launch_end(ctx, 1);
    }
    gs_launch_begin(ctx, 1);
    k_bary_exp<<<(unsigned)nchunks, kThreads, 0, s>>>(lb.get(), lbmax.get(), n, bary.get(), part.get(), w.status.get());
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_fold<<<1, kThreads, 0, s>>>(part.get(), nchunks, mass.get());
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_bary_mass_check<<<1, 1, 0, s>>>(mass.get(), w.status.get());
    gs_launch_end(ctx, 1);
    // W = bary / max(psi, floor); T_0 = a * W (barycenter.cpp:84-85)
    gs_launch_begin(ctx, 1);
    k_bary_w<S><<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(
        bary.get(), mass.get(), psi, da, n, m, w.GW, W.get(), w.T[a0].get(), w.cmax.get(),
        w.status.get());
    gs_launch_end(ctx, 1);
    run_finalize<S>(ctx, w, 0, 1, 0, knp, false);
    // phi = H(a * W); err; V' = M / max(phi, floor) (barycenter.cpp:85-86, 70)
    a0 = run_apply<S>(ctx, f, w, a0, MODE_SK_PHI, da, Mb.get(), V[parity].get(), V[parity ^ 1].get(),
                      false, true);
    run_finalize<S>(ctx, w, 1, 1, 1, knp, false);
    gs_launch_begin(ctx, 1);
    k_bary_errlocal<<<1, 1, 0, s>>>(w.errcol.get(), m, errbuf.get(), w.status.get());
    gs_launch_end(ctx, 1);
    if (hooked) {
      const int rc = comm->allreduce(comm->user, errbuf.get(), 2, 1, (void*)s);
      if (rc) return rc;
    }
    gs_launch_begin(ctx, 1);
    k_bary_control<<<1, 1, 0, s>>>(errbuf.get(), w.status.get(), sweep_ctr.get(), tol, diters.get(),
                                   dconv.get(), derr.get(), max_iter, w.kF32 ? 1 : 0);
    gs_launch_end(ctx, 1);
    return 0;
  };
  // Two sweeps (odd, even parity) are captured once as a CUDA graph and replayed (as in
  // sinkhorn_impl) -- with no collective hooks, or with stream-ordered device collectives that may
  // be captured (GS_COMM_GRAPH_SAFE: the engine's NCCL communicator, gs_nccl.cu). Host-callback
  // hooks run every sweep without capture.
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_launches = 0;
  const char* genv = getenv("GS_GRAPH");
  const bool capturable = !hooked || (comm->flags & GS_COMM_GRAPH_SAFE);
  if (capturable && (genv ? genv[0] != '0' : true) && max_iter >= 2) {
    cudaGraph_t graph = nullptr;
    const int64_t l0 = ctx->launches;
    const int a0_saved = a0;
    ctx->capturing = true;
    cudaError_t ce = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (ce == cudaSuccess) {
      issue_sweep(1);
      issue_sweep(0);
      ce = cudaStreamEndCapture(s, &graph);
    }
    ctx->capturing = false;
    graph_launches = ctx->launches - l0;
    ctx->launches = l0;
    if (ce == cudaSuccess) ce = cudaGraphInstantiate(&gexec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (ce != cudaSuccess) {
      cudaGetLastError();
      gexec = nullptr;
    }
    a0 = a0_saved;  // two sweeps = 4 applies of K steps: the buffer parity returns to a0 (K even)
    if (gexec && ((4 * f->degree) & 1)) a0 ^= 1;
  }
  const int step_sweeps = gexec ? 2 : 1;
  for (int sweep = 1, it = 0; sweep <= max_iter; sweep += step_sweeps, ++it) {
    if (it >= 2) {
      const int slot = (it - 2) & 1;
      cudaEventSynchronize(ev[slot]);
      const gs_status st = hst[slot];
      if (st.error || st.done) break;
    }
    if (gexec) {
      GS_CUDA(ctx, cudaGraphLaunch(gexec, s));
      ctx->launches += graph_launches;
    } else {
      hook_rc = issue_sweep(sweep & 1);
      if (hook_rc) break;
    }
    const int slot = it & 1;
    cudaMemcpyAsync(&hst[slot], w.status.get(), sizeof(gs_status), cudaMemcpyDeviceToHost, s);
    cudaEventRecord(ev[slot], s);
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (hook_rc) {
    ctx->err = "NcclError: allreduce hook failed";
    return GS_ERR_NCCL;
  }
  gs_status st;
  GS_CUDA(ctx, cudaMemcpy(&st, w.status.get(), sizeof st, cudaMemcpyDeviceToHost));
  if (st.error) {
    if (st.error == 1000 + ERRC_KERNEL_NOT_POSITIVE + 1)
      return gs_fail(ctx, ERRC_KERNEL_NOT_POSITIVE, "barycenter iterate collapsed to zero");
    if (st.error == ERRC_NUMERICAL_UNDERFLOW + 1)
      return gs_fail(ctx, ERRC_NUMERICAL_UNDERFLOW,
                     "fp32 mode: non-finite barycenter marginal error; rerun in fp64");
    return gs_fail(ctx, ERRC_KERNEL_NOT_POSITIVE, kKnpBary);
  }
  int h_iters = 0;
  GS_CUDA(ctx, cudaMemcpy(&h_iters, diters.get(), sizeof(int), cudaMemcpyDeviceToHost));
  // bary /= sum (barycenter.cpp:94), then Distribution::from_weights divides twice more
  // (transport.cpp:86-94); every sum is the deterministic DET-chunk fold.
  for (int pass = 0; pass < 3; ++pass) {
    gs_launch_begin(ctx, 1);
    k_chunk_sum<<<(unsigned)nchunks, kThreads, 0, s>>>(bary.get(), n, part.get());
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_fold<<<1, kThreads, 0, s>>>(part.get(), nchunks, mass.get());
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_scale_div<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(bary.get(), mass.get(), n);
    gs_launch_end(ctx, 1);
  }
  {
    DevBuf<double> bu;
    GS_CUDA(ctx, bu.alloc(n, s));
    gs_launch_begin(ctx, 1);
    k_gather<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(bary.get(), f->lay[w.lay].newpos, n, bu.get());
    gs_launch_end(ctx, 1);
    GS_TRY(gs_copy_out(ctx, out_bary, bu.get(), (size_t)n * sizeof(double), mem));
  }
  // final V lives in V[iters & 1] (V_s of the last sweep), W is single-buffered
  DevBuf<int> sel;
  GS_CUDA(ctx, sel.alloc(m, s));
  {
    std::vector<int> hs(m, h_iters);
    GS_CUDA(ctx, cudaMemcpyAsync(sel.get(), hs.data(), m * sizeof(int), cudaMemcpyHostToDevice, s));
  }
  DevBuf<double> ov, ow;
  double* dv = out_V;
  double* dw = out_W;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, ov.alloc((size_t)m * n, s));
    GS_CUDA(ctx, ow.alloc((size_t)m * n, s));
    dv = ov.get();
    dw = ow.get();
  }
  if (out_V) {
    gs_launch_begin(ctx, 1);
    k_unpack<double><<<grid_for((int64_t)m * n), kThreads, 0, s>>>(V[0].get(), dv, n, m, w.GW, V[1].get(), sel.get(), f->lay[w.lay].newpos, (int64_t)n);
    gs_launch_end(ctx, 1);
    GS_TRY(finish_out(ctx, ov, out_V, (size_t)m * n, mem));
  }
  if (out_W) {
    gs_launch_begin(ctx, 1);
    k_unpack<double><<<grid_for((int64_t)m * n), kThreads, 0, s>>>(W.get(), dw, n, m, w.GW, nullptr, nullptr, f->lay[w.lay].newpos, (int64_t)n);
    gs_launch_end(ctx, 1);
    GS_TRY(finish_out(ctx, ow, out_W, (size_t)m * n, mem));
  }
  int h_conv = 0;
  double h_err = 0.0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h_conv, dconv.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(&h_err, derr.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (out_iters) *out_iters = h_iters;
  if (out_conv) *out_conv = h_conv;
  if (out_err) *out_err = h_err;
  return GS_OK;
}


// ============================================================================================
// Row-partitioned applies (gs_part.cu). The grouped buffers hold nl local rows
// followed by nh halo rows per column group (Work::ld = nl + nh); before every Chebyshev step the
// rows other ranks read are packed, exchanged through comm->alltoallv and unpacked into the halo.
// Per-column reductions are combined through comm->allreduce before any decision is taken, so all
// ranks follow the same control path (and make the same number of collective calls).
// ============================================================================================
template <typename S>
__global__ void k_halo_pack(const S* __restrict__ T, int64_t ld, int GW, int Bpad,
                            const int* __restrict__ rows, int ns, S* __restrict__ buf) {
  const int64_t total = (int64_t)ns * Bpad;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / Bpad), col = (int)(e % Bpad);
    buf[e] = T[((size_t)(col / GW) * ld + rows[j]) * GW + (col % GW)];
  }
}

template <typename S>
__global__ void k_halo_unpack(const S* __restrict__ buf, int nh, int nl, int64_t ld, int GW, int Bpad,
                              S* __restrict__ T) {
  const int64_t total = (int64_t)nh * Bpad;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / Bpad), col = (int)(e % Bpad);
    T[((size_t)(col / GW) * ld + nl + j) * GW + (col % GW)] = buf[e];
  }
}

// local half of k_finalize: fold this rank's error tiles; export -min and max of every column
__global__ void __launch_bounds__(kThreads) k_fin_local(const FinArgs F, double* stat) {
  const int col = blockIdx.x;
  if (col >= F.B) return;
  __shared__ double sh[kThreads];
  double acc = 0.0;
  if (F.has_err) {
    for (int t = threadIdx.x; t < F.tiles; t += kThreads) acc = acc + F.cs.part_err[(size_t)t * F.Bpad + col];
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  if (F.has_err) F.cs.errcol[col] = sh[0];
  stat[col] = -dunkey(F.cs.cmin[col]);
  stat[F.Bpad + col] = dunkey(F.cs.cmax[col]);
}

// global half: the positivity check and the next threshold from the combined column extrema
__global__ void k_fin_global(const FinArgs F, const double* stat) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= F.B) return;
  const bool act = !F.cs.active || F.cs.active[col];
  if (F.check && act && F.status->error == 0) {
    const double mn = -stat[col];
    if (!(mn >= -F.cs.thr[col])) atomicCAS(&F.status->error, 0, F.knp_code);
  }
  if (F.has_next) F.cs.thr[col] = F.slack * stat[F.Bpad + col];
  F.cs.cmin[col] = KEY_POS_INF;
  F.cs.cmax[col] = KEY_ZERO;
}

__global__ void k_sk_cost_sums(const double* part, int64_t nchunks, int P, double* sums) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= P) return;
  double s[4] = {0, 0, 0, 0};
  for (int64_t c = 0; c < nchunks; ++c)
    for (int q = 0; q < 4; ++q) s[q] = s[q] + part[((size_t)c * P + col) * 4 + q];
  for (int q = 0; q < 4; ++q) sums[(size_t)col * 4 + q] = s[q];
}

__global__ void k_sk_cost_from_sums(const double* sums, int P, double lambda, double* cost, double* kl) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= P) return;
  const double* s = sums + (size_t)col * 4;
  cost[col] = lambda * (s[0] + s[1]);
  kl[col] = s[2] + s[3] - 1.0;
}

__global__ void k_int_to_double(const int* __restrict__ x, int n, double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = (double)x[i];
}

int hook_fail(gs_ctx* ctx, const char* what) {
  ctx->err = std::string("NcclError: ") + what + " hook failed";
  return GS_ERR_NCCL;
}

int allreduce(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, double* buf, int64_t count, int op) {
  if (p->nparts == 1 || count == 0) return GS_OK;
  if (comm->allreduce(comm->user, buf, count, op, (void*)ctx->stream)) return hook_fail(ctx, "allreduce");
  return GS_OK;
}

template <typename S>
struct Halo {
  DevBuf<S> send, recv;
  std::vector<int64_t> sb, rb;  // bytes per rank
  int init(gs_ctx* ctx, const gs_part* p, int Bpad) {
    sb.resize(p->nparts);
    rb.resize(p->nparts);
    for (int q = 0; q < p->nparts; ++q) {
      sb[q] = p->send_counts[q] * Bpad * (int64_t)sizeof(S);
      rb[q] = p->recv_counts[q] * Bpad * (int64_t)sizeof(S);
    }
    GS_CUDA(ctx, send.alloc((size_t)p->ns * Bpad, ctx->stream));
    GS_CUDA(ctx, recv.alloc((size_t)p->nh * Bpad, ctx->stream));
    return GS_OK;
  }
};

// Row ranges of one partitioned step: the interior rows (no halo reads) run while the halo is in
// flight; the two boundary ranges after it has landed. One range when the part is alone.
struct PartRanges {
  int lo[3], hi[3], tile0[3], tiles[3], count, total;
};

inline PartRanges part_ranges(const gs_part* p, int rows_per_tile) {
  PartRanges R{};
  auto add = [&](int lo, int hi) {
    const int c = R.count++;
    R.lo[c] = lo;
    R.hi[c] = hi;
    R.tile0[c] = R.total;
    R.tiles[c] = hi > lo ? (hi - lo + rows_per_tile - 1) / rows_per_tile : 0;
    R.total += R.tiles[c];
  };
  if (p->nparts == 1) {
    add(0, p->nl);
  } else {
    add(p->int_lo, p->int_hi);  // [0]: interior
    add(0, p->int_lo);          // [1], [2]: boundary prefix and suffix
    add(p->int_hi, p->nl);
  }
  return R;
}

template <typename S>
int part_tiles(const gs_part* p, const Work<S>& w) {
  return part_ranges(p, rows_per_block<S>(w.GW) * w.rpc).total;
}

// pack the rows other parts read, then hand them to comm->alltoallv on the context's comm stream
// (after the pack); the caller launches the interior rows meanwhile and calls halo_finish
template <typename S>
int halo_start(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const Work<S>& w, const S* T, Halo<S>& h) {
  cudaStream_t s = ctx->stream;
  if (!ctx->comm_stream) {
    GS_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    GS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_packed, cudaEventDisableTiming));
    GS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_received, cudaEventDisableTiming));
  }
  if (p->ns > 0) {
    gs_launch_begin(ctx, 1);
    k_halo_pack<S><<<grid_for((int64_t)p->ns * w.Bpad), kThreads, 0, s>>>(T, w.ld, w.GW, w.Bpad, p->send_rows, p->ns, h.send.get());
    gs_launch_end(ctx, 1);
  }
  GS_CUDA(ctx, cudaEventRecord(ctx->ev_packed, s));
  GS_CUDA(ctx, cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_packed, 0));
  return GS_OK;
}

// One column group (Bpad == GW): the received rows land straight in T's halo rows [nl, nl + nh),
// whose layout equals the packed one, so no unpack pass follows.
template <typename S>
inline bool halo_direct(const Work<S>& w) {
  return w.G == 1;
}

template <typename S>
int halo_exchange(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const Work<S>& w, S* T, Halo<S>& h) {
  S* recv = halo_direct(w) ? T + (size_t)p->nl * w.GW : h.recv.get();
  if (comm->alltoallv(comm->user, h.send.get(), h.sb.data(), recv, h.rb.data(), p->nparts,
                      (void*)ctx->comm_stream))
    return hook_fail(ctx, "alltoallv");
  GS_CUDA(ctx, cudaEventRecord(ctx->ev_received, ctx->comm_stream));
  return GS_OK;
}

template <typename S>
int halo_finish(gs_ctx* ctx, const gs_part* p, const Work<S>& w, S* T, Halo<S>& h) {
  cudaStream_t s = ctx->stream;
  GS_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_received, 0));
  if (p->nh > 0 && !halo_direct(w)) {
    gs_launch_begin(ctx, 1);
    k_halo_unpack<S><<<grid_for((int64_t)p->nh * w.Bpad), kThreads, 0, s>>>(h.recv.get(), p->nh, p->nl, w.ld, w.GW, w.Bpad, T);
    gs_launch_end(ctx, 1);
  }
  return GS_OK;
}

// k_cheb_lane on a part's rows stages the odd-stride copy of its local CSR (gs_lane.cu): built
// once per part and precision, before any sweep is captured into a CUDA graph
template <typename S>
bool part_lane_wanted(const Work<S>& w) {
  return lane_enabled() && lane_pad_enabled() && w.rpc > 1 && rpc_lpr<S>(w.GW) == 1 && w.n > 0;
}
template <typename S>
const gs_lanepad* part_lane_copy(const gs_part* p, const Work<S>& w) {
  return part_lane_wanted<S>(w) ? p->lanepad[sizeof(S) == 4 ? 0 : 1] : nullptr;
}
template <typename S>
int part_lane_prepare(gs_ctx* ctx, const gs_part* p, const Work<S>& w) {
  if (!part_lane_wanted<S>(w)) return GS_OK;
  gs_lanepad*& lp = const_cast<gs_part*>(p)->lanepad[sizeof(S) == 4 ? 0 : 1];
  if (lp) return GS_OK;
  const void* vals = sizeof(S) == 4 ? static_cast<const void*>(p->vals32) : static_cast<const void*>(p->local->vals);
  const int rc = gs_lanepad_build(ctx, p->local->offs, p->local->cols, vals, (int)sizeof(S), p->local->n,
                                  p->local->nnz, &lp);
  return rc == GS_ERR_UNSUPPORTED ? GS_OK : rc;
}

// run_apply over this part's rows, one halo exchange of T_{k-1} before every step
template <typename S>
int run_apply_part(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, Work<S>& w, Halo<S>& h, int a0,
                   int mode, const double* a, const double* M, const double* Vcur, double* Wout,
                   bool use_active, bool use_status, int* next) {
  const gs_filter* f = p->f;
  const int K = f->degree;
  StepArgs A{};
  A.offs = p->local->offs;
  A.cols = p->local->cols;
  if constexpr (sizeof(S) == 4) A.vals = p->vals32;
  else A.vals = p->local->vals;
  A.lane = lane_enabled();
  if (const gs_lanepad* lp = part_lane_copy<S>(p, w)) {  // built by part_lane_prepare
    A.offs = lp->offs;
    A.cols = lp->cols;
    A.vals = lp->vals;
  }
  A.n = w.n;
  A.ld = w.ld;
  A.tiles = w.tiles;
  A.g0 = 0;
  A.Gl = w.G;
  A.Bpad = w.Bpad;
  A.acc = w.acc.get();
  A.b0h = f->coeffs[0] / 2.0;
  A.status = use_status ? w.status.get() : nullptr;
  A.cs = w.cs();
  if (!use_active) {
    A.cs.active = nullptr;
    A.cs.gactive = nullptr;
  }
  A.a = a;
  A.M = M;
  A.Vcur = Vcur;
  A.Wout = Wout;
  A.psi = w.psi64.get();
  const PartRanges R = part_ranges(p, rows_per_block<S>(w.GW) * w.rpc);
  auto launch_range = [&](int r, int m) {
    if (R.tiles[r] == 0) return;
    A.row0 = R.lo[r];
    A.n = R.hi[r];
    A.tiles = R.tiles[r];
    A.tile0 = R.tile0[r];
    launch_step<S>(ctx, w.GW, w.rpc, A, m);
  };
  AccSchedule sched;
  for (int k = 1; k <= K; ++k) {
    A.k = k;
    A.bk = f->coeffs[k];
    sched.step(f, K, k, A);
    S* Tprev = w.T[(a0 + k - 1) & 1].get();
    A.Tprev = Tprev;
    A.Tout = w.T[(a0 + k) & 1].get();
    const int m = k == K ? mode : MODE_NONE;
    if (p->nparts == 1) {
      launch_range(0, m);
      continue;
    }
    // T_{k-1}'s boundary rows go out while the interior rows (no halo reads) are computed
    GS_TRY(halo_start<S>(ctx, p, comm, w, Tprev, h));
    launch_range(0, m);
    GS_TRY(halo_exchange<S>(ctx, p, comm, w, Tprev, h));
    GS_TRY(halo_finish<S>(ctx, p, w, Tprev, h));
    launch_range(1, m);
    launch_range(2, m);
  }
  *next = (a0 + K) & 1;
  return GS_OK;
}

template <typename S>
int run_finalize_part(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, Work<S>& w, double* stat,
                      int check, int has_next, int has_err, int knp_code, bool use_active) {
  FinArgs F{};
  F.cs = w.cs();
  if (!use_active) F.cs.active = nullptr;
  F.B = w.B;
  F.tiles = w.tiles;
  F.Bpad = w.Bpad;
  F.check = check;
  F.has_next = has_next;
  F.has_err = has_err;
  F.status = w.status.get();
  F.knp_code = knp_code;
  F.slack = Prec<S>::slack;
  gs_launch_begin(ctx, 1);
  k_fin_local<<<w.B, kThreads, 0, ctx->stream>>>(F, stat);
  gs_launch_end(ctx, 1);
  GS_TRY(allreduce(ctx, p, comm, stat, 2 * (int64_t)w.Bpad, 1));
  if (has_err) GS_TRY(allreduce(ctx, p, comm, w.errcol.get(), w.B, 0));
  gs_launch_begin(ctx, 1);
  k_fin_global<<<(w.B + kThreads - 1) / kThreads, kThreads, 0, ctx->stream>>>(F, stat);
  gs_launch_end(ctx, 1);
  return GS_OK;
}

template <typename S>
int filter_apply_part_impl(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const double* dX,
                           double* dY, int width) {
  const int nl = p->nl;
  cudaStream_t s = ctx->stream;
  Work<S> w;
  GS_TRY(w.init(ctx, nl, width, false, (int64_t)nl + p->nh, p->f));
  GS_TRY(part_lane_prepare<S>(ctx, p, w));
  w.tiles = part_tiles<S>(p, w);
  Halo<S> h;
  GS_TRY(h.init(ctx, p, w.Bpad));
  if (nl > 0) {
    gs_launch_begin(ctx, 1);
    k_pack<S><<<grid_for((int64_t)w.Bpad * nl), kThreads, 0, s>>>(dX, w.T[0].get(), nl, width, w.GW, w.G, nullptr, w.ld);
    gs_launch_end(ctx, 1);
  }
  int next = 0;
  GS_TRY(run_apply_part<S>(ctx, p, comm, w, h, 0, MODE_NONE, nullptr, nullptr, nullptr, nullptr, false, false, &next));
  if (nl > 0) {
    gs_launch_begin(ctx, 1);
    k_unpack<S><<<grid_for((int64_t)width * nl), kThreads, 0, s>>>(w.acc.get(), dY, nl, width, w.GW, nullptr, nullptr, nullptr, w.ld);
    gs_launch_end(ctx, 1);
  }
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// geodesic Sinkhorn batch on one part (transport.cpp:144-239; same control as sinkhorn_impl)
template <typename S>
int sinkhorn_part_impl(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const double* da_user,
                       const double* dmu, const double* dnu, int P, int max_iter, double tol, int flags,
                       int mem, double* out_v, double* out_w, double* out_cost, double* out_kl,
                       int* out_iters, int* out_conv, double* out_err, int* fail_pair, int* fail_sweep) {
  const int nl = p->nl;
  cudaStream_t s = ctx->stream;
  Work<S> w;
  GS_TRY(w.init(ctx, nl, P, true, (int64_t)nl + p->nh, p->f));
  GS_TRY(part_lane_prepare<S>(ctx, p, w));
  w.tiles = part_tiles<S>(p, w);  // error partials: one per tile of the (up to) three row ranges
  GS_CUDA(ctx, w.part_err.alloc((size_t)(w.tiles ? w.tiles : 1) * w.Bpad, s));
  Halo<S> h;
  GS_TRY(h.init(ctx, p, w.Bpad));
  DevBuf<double> stat;
  GS_CUDA(ctx, stat.alloc(2 * (size_t)w.Bpad, s));
  DevBuf<double> aloc;
  GS_CUDA(ctx, aloc.alloc(nl, s));
  if (nl > 0) {
    gs_launch_begin(ctx, 1);
    k_gather_to<double><<<(nl + kThreads - 1) / kThreads, kThreads, 0, s>>>(da_user, nullptr, nl, aloc.get());
    gs_launch_end(ctx, 1);
  }
  const double* da = aloc.get();
  const size_t len = (size_t)w.Bpad * w.ld;
  DevBuf<double> M, N, V[2], W;
  GS_CUDA(ctx, M.alloc(len, s));
  GS_CUDA(ctx, N.alloc(len, s));
  GS_CUDA(ctx, V[0].alloc(len, s));
  GS_CUDA(ctx, V[1].alloc(len, s));
  GS_CUDA(ctx, W.alloc(len, s));
  DevBuf<int> iters, conv, stag, final_sweep;
  DevBuf<double> errv;
  GS_CUDA(ctx, iters.alloc(w.Bpad, s));
  GS_CUDA(ctx, conv.alloc(w.Bpad, s));
  GS_CUDA(ctx, stag.alloc(w.Bpad, s));
  GS_CUDA(ctx, final_sweep.alloc(w.Bpad, s));
  GS_CUDA(ctx, errv.alloc(w.Bpad, s));
  GS_CUDA(ctx, cudaMemsetAsync(iters.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(conv.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(stag.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(final_sweep.get(), 0, w.Bpad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(V[0].get(), 0, len * sizeof(double), s));
  GS_CUDA(ctx, cudaMemsetAsync(W.get(), 0, len * sizeof(double), s));
  {
    std::vector<int> act(w.Bpad, 0);
    for (int q = 0; q < P; ++q) act[q] = 1;
    GS_CUDA(ctx, cudaMemcpyAsync(w.active.get(), act.data(), w.Bpad * sizeof(int), cudaMemcpyHostToDevice, s));
    std::vector<double> inf(w.Bpad, INFINITY);
    GS_CUDA(ctx, cudaMemcpyAsync(errv.get(), inf.data(), w.Bpad * sizeof(double), cudaMemcpyHostToDevice, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
  }
  if (nl > 0) {
    gs_launch_begin(ctx, 1);
    k_pack<double><<<grid_for((int64_t)w.Bpad * nl), kThreads, 0, s>>>(dmu, M.get(), nl, P, w.GW, w.G, nullptr, w.ld);
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_pack<double><<<grid_for((int64_t)w.Bpad * nl), kThreads, 0, s>>>(dnu, N.get(), nl, P, w.GW, w.G, nullptr, w.ld);
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_sk_init<S><<<grid_for((int64_t)w.Bpad * nl), kThreads, 0, s>>>(da, w.T[0].get(), nl, w.GW, w.G, P, w.cmax.get(), w.ld);
    gs_launch_end(ctx, 1);
  }
  const int knp = ERRC_KERNEL_NOT_POSITIVE + 1;
  int a0 = 0;
  GS_TRY(run_finalize_part<S>(ctx, p, comm, w, stat.get(), 0, 1, 0, knp, true));
  GS_TRY(run_apply_part<S>(ctx, p, comm, w, h, 0, MODE_SK_PHI, da, M.get(), V[0].get(), V[1].get(), true, true, &a0));
  GS_TRY(run_finalize_part<S>(ctx, p, comm, w, stat.get(), 1, 1, 0, knp, true));
  CtlArgs C{};
  C.active = w.active.get();
  C.gactive = w.gactive.get();
  C.GW = w.GW;
  C.errcol = w.errcol.get();
  C.iters = iters.get();
  C.conv = conv.get();
  C.stag = stag.get();
  C.final_sweep = final_sweep.get();
  C.err_out = errv.get();
  C.status = w.status.get();
  C.P = P;
  C.max_iter = max_iter;
  C.no_abort = (flags & GS_FLAG_NO_STAGNATION_ABORT) ? 1 : 0;
  C.fp32 = w.kF32 ? 1 : 0;
  C.tol = tol;
  DevBuf<int> sweep_ctr;
  GS_CUDA(ctx, sweep_ctr.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(sweep_ctr.get(), 0, sizeof(int), s));
  C.sweep_ctr = sweep_ctr.get();
  gs_status* hst = ctx->h_status;
  cudaEvent_t ev[2];
  cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
  int rc = GS_OK;
  auto issue_sweep = [&](int parity) -> int {
    int r = run_apply_part<S>(ctx, p, comm, w, h, a0, MODE_SK_PSI, da, N.get(), nullptr, W.get(), true, true, &a0);
    if (!r) r = run_finalize_part<S>(ctx, p, comm, w, stat.get(), 1, 1, 0, knp, true);
    if (!r)
      r = run_apply_part<S>(ctx, p, comm, w, h, a0, MODE_SK_PHI, da, M.get(), V[parity].get(),
                            V[parity ^ 1].get(), true, true, &a0);
    if (!r) r = run_finalize_part<S>(ctx, p, comm, w, stat.get(), 1, 1, 1, knp, true);
    if (r) return r;
    gs_launch_begin(ctx, 1);
    k_sk_control<<<1, 1, 0, s>>>(C);
    gs_launch_end(ctx, 1);
    return GS_OK;
  };
  // With stream-ordered collectives (the engine's NCCL comm, or one part) two sweeps -- halo
  // exchanges on the comm stream and allreduces included -- are captured as one CUDA graph and
  // replayed, as in the unpartitioned sweep loop. Host-callback hooks run sweep by sweep.
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_launches = 0;
  {
    const char* genv = getenv("GS_GRAPH");
    const bool capturable = (!comm || (comm->flags & GS_COMM_GRAPH_SAFE)) && (genv ? genv[0] != '0' : true) &&
                            max_iter >= 2;
    if (capturable) {
      if (!ctx->comm_stream) {
        GS_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
        GS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_packed, cudaEventDisableTiming));
        GS_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_received, cudaEventDisableTiming));
      }
      cudaGraph_t graph = nullptr;
      const int64_t l0 = ctx->launches;
      const int a0_saved = a0;
      ctx->capturing = true;
      cudaError_t ce = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      int crc = GS_OK;
      if (ce == cudaSuccess) {
        crc = issue_sweep(1);
        if (!crc) crc = issue_sweep(0);
        ce = cudaStreamEndCapture(s, &graph);
      }
      ctx->capturing = false;
      graph_launches = ctx->launches - l0;
      ctx->launches = l0;
      if (ce == cudaSuccess && !crc) ce = cudaGraphInstantiate(&gexec, graph, 0);
      if (graph) cudaGraphDestroy(graph);
      if (ce != cudaSuccess || crc) {
        cudaGetLastError();
        if (gexec) cudaGraphExecDestroy(gexec);
        gexec = nullptr;
      }
      a0 = a0_saved;  // two sweeps = four K-step applies: the buffer parity returns
    }
  }
  const int step_sweeps = gexec ? 2 : 1;
  for (int sweep = 1, it = 0; sweep <= max_iter; sweep += step_sweeps, ++it) {
    if (it >= 2) {  // every rank sees the same status (same global reductions) -> same exit sweep
      const int slot = (it - 2) & 1;
      cudaEventSynchronize(ev[slot]);
      const gs_status st = hst[slot];
      if (st.error || st.n_active == 0) break;
    }
    if (gexec) {
      GS_CUDA(ctx, cudaGraphLaunch(gexec, s));
      ctx->launches += graph_launches;
    } else {
      rc = issue_sweep(sweep & 1);
      if (rc) break;
    }
    const int slot = it & 1;
    cudaMemcpyAsync(&hst[slot], w.status.get(), sizeof(gs_status), cudaMemcpyDeviceToHost, s);
    cudaEventRecord(ev[slot], s);
  }
  if (gexec) cudaGraphExecDestroy(gexec);
  cudaStreamSynchronize(s);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (rc) return rc;
  gs_status st;
  GS_CUDA(ctx, cudaMemcpy(&st, w.status.get(), sizeof st, cudaMemcpyDeviceToHost));
  if (st.error) {
    if (st.error == ERRC_DISCONNECTED + 1) {
      if (fail_pair) *fail_pair = st.fail_pair;
      if (fail_sweep) *fail_sweep = st.fail_sweep;
      if (flags & GS_FLAG_SINGLE)
        return gs_fail(ctx, ERRC_DISCONNECTED,
                       "marginal error stagnated above 0.5; are mu and nu in the same graph component?");
      return gs_fail(ctx, ERRC_DISCONNECTED,
                     "marginal error stagnated above 0.5 for pair " + std::to_string(st.fail_pair));
    }
    if (st.error == ERRC_NUMERICAL_UNDERFLOW + 1) {
      if (fail_pair) *fail_pair = st.fail_pair;
      if (fail_sweep) *fail_sweep = st.fail_sweep;
      return gs_fail(ctx, ERRC_NUMERICAL_UNDERFLOW, kF32Range_msg + std::to_string(st.fail_pair));
    }
    return gs_fail(ctx, ERRC_KERNEL_NOT_POSITIVE, kKnpTransport);
  }
  // ---- cost / KL: local DET-chunk partials, combined across ranks ---------------------------------
  const int64_t nchunks = (nl + DET_CHUNK - 1) / DET_CHUNK;
  DevBuf<double> part, sums, dcost, dkl;
  GS_CUDA(ctx, part.alloc((size_t)(nchunks ? nchunks : 1) * P * 4, s));
  GS_CUDA(ctx, sums.alloc((size_t)P * 4, s));
  GS_CUDA(ctx, dcost.alloc(P, s));
  GS_CUDA(ctx, dkl.alloc(P, s));
  if (nchunks > 0) {
    gs_launch_begin(ctx, 1);
    k_sk_cost_partial<double><<<dim3((unsigned)nchunks, P), kThreads, 0, s>>>(
        da, M.get(), N.get(), V[0].get(), V[1].get(), W.get(), final_sweep.get(), nl, w.GW, part.get(), P, w.ld);
    gs_launch_end(ctx, 1);
  }
  gs_launch_begin(ctx, 1);
  k_sk_cost_sums<<<(P + 63) / 64, 64, 0, s>>>(part.get(), nchunks, P, sums.get());
  gs_launch_end(ctx, 1);
  GS_TRY(allreduce(ctx, p, comm, sums.get(), 4 * (int64_t)P, 0));
  gs_launch_begin(ctx, 1);
  k_sk_cost_from_sums<<<(P + 63) / 64, 64, 0, s>>>(sums.get(), P, 4.0 * p->f->t, dcost.get(), dkl.get());
  gs_launch_end(ctx, 1);
  if (w.kF32) GS_TRY(check_finite_costs(ctx, dcost.get(), P));
  DevBuf<double> ov, ow;
  double* dv = out_v;
  double* dw = out_w;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, ov.alloc((size_t)P * nl, s));
    GS_CUDA(ctx, ow.alloc((size_t)P * nl, s));
    dv = ov.get();
    dw = ow.get();
  }
  if (out_v && nl > 0) {
    gs_launch_begin(ctx, 1);
    k_unpack<double><<<grid_for((int64_t)P * nl), kThreads, 0, s>>>(V[0].get(), dv, nl, P, w.GW, V[1].get(), final_sweep.get(), nullptr, w.ld);
    gs_launch_end(ctx, 1);
    GS_TRY(finish_out(ctx, ov, out_v, (size_t)P * nl, mem));
  }
  if (out_w && nl > 0) {
    gs_launch_begin(ctx, 1);
    k_unpack<double><<<grid_for((int64_t)P * nl), kThreads, 0, s>>>(W.get(), dw, nl, P, w.GW, nullptr, nullptr, nullptr, w.ld);
    gs_launch_end(ctx, 1);
    GS_TRY(finish_out(ctx, ow, out_w, (size_t)P * nl, mem));
  }
  auto out_small = [&](void* dst, const void* src, size_t bytes) -> int {
    if (!dst) return GS_OK;
    GS_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes,
                                 mem == GS_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    return GS_OK;
  };
  GS_TRY(out_small(out_cost, dcost.get(), P * sizeof(double)));
  GS_TRY(out_small(out_kl, dkl.get(), P * sizeof(double)));
  GS_TRY(out_small(out_iters, iters.get(), P * sizeof(int)));
  GS_TRY(out_small(out_conv, conv.get(), P * sizeof(int)));
  GS_TRY(out_small(out_err, errv.get(), P * sizeof(double)));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// Distribution::validate (transport.cpp:96-102) of P local column slices, sums combined across
// ranks: returns per-column global sum, non-finite and negative flags on the host.
int validate_columns_part(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const double* d, int P,
                          std::vector<double>& sums, std::vector<int>& nonfinite, std::vector<int>& negative) {
  cudaStream_t s = ctx->stream;
  DevBuf<double> dsum, dflags;
  DevBuf<int> dnf, dng;
  GS_CUDA(ctx, dsum.alloc(P, s));
  GS_CUDA(ctx, dflags.alloc(2 * (size_t)P, s));
  GS_CUDA(ctx, dnf.alloc(P, s));
  GS_CUDA(ctx, dng.alloc(P, s));
  GS_CUDA(ctx, cudaMemsetAsync(dnf.get(), 0, P * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(dng.get(), 0, P * sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_validate_cols<<<dim3(1, P), kThreads, 0, s>>>(d, p->nl, dsum.get(), dnf.get(), dng.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_int_to_double<<<(P + kThreads - 1) / kThreads, kThreads, 0, s>>>(dnf.get(), P, dflags.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_int_to_double<<<(P + kThreads - 1) / kThreads, kThreads, 0, s>>>(dng.get(), P, dflags.get() + P);
  gs_launch_end(ctx, 1);
  GS_TRY(allreduce(ctx, p, comm, dsum.get(), P, 0));
  GS_TRY(allreduce(ctx, p, comm, dflags.get(), 2 * (int64_t)P, 1));
  std::vector<double> fl(2 * (size_t)P);
  sums.resize(P);
  GS_CUDA(ctx, cudaMemcpyAsync(sums.data(), dsum.get(), P * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(fl.data(), dflags.get(), 2 * P * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  nonfinite.assign(P, 0);
  negative.assign(P, 0);
  for (int q = 0; q < P; ++q) {
    nonfinite[q] = fl[q] > 0.0;
    negative[q] = fl[P + q] > 0.0;
  }
  return GS_OK;
}

// collective half of check_weights: *bad = some rank holds a non-positive weight
int weights_bad_part(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const double* da, bool* bad_out) {
  cudaStream_t s = ctx->stream;
  DevBuf<int> bad;
  DevBuf<double> dbad;
  GS_CUDA(ctx, bad.alloc(1, s));
  GS_CUDA(ctx, dbad.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  if (p->nl > 0) {
    gs_launch_begin(ctx, 1);
    k_validate_weights<<<(p->nl + 255) / 256, 256, 0, s>>>(da, p->nl, bad.get());
    gs_launch_end(ctx, 1);
  }
  gs_launch_begin(ctx, 1);
  k_int_to_double<<<1, 1, 0, s>>>(bad.get(), 1, dbad.get());
  gs_launch_end(ctx, 1);
  GS_TRY(allreduce(ctx, p, comm, dbad.get(), 1, 1));
  double h = 0.0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h, dbad.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  *bad_out = h > 0.0;
  return GS_OK;
}

int check_part_comm(gs_ctx* ctx, const gs_part* p, const gs_comm* comm) {
  if (!p) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "null partition");
  if (p->nparts > 1 && (!comm || !comm->allreduce || !comm->alltoallv))
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "a partition of several ranks needs allreduce and alltoallv hooks");
  return GS_OK;
}

}  // namespace

// ============================================================================================
// HeatFilter (heat.cpp:72-96): scaled Laplacian copy + coefficients, both on the device.
// ============================================================================================
// Renumbered operator, fp32 value copy and index-locality statistic of layout l (its order and
// newpos already set).
static int finish_layout(gs_ctx* ctx, gs_filter* f, int l) {
  cudaStream_t s = ctx->stream;
  int rc = GS_OK;
  gs_layout& Ly = f->lay[l];
  gs_graph_destroy(Ly.perm);
  Ly.perm = nullptr;
  cudaFree(Ly.rec_key);
  cudaFree(Ly.rec_val);
  Ly.rec_key = nullptr;
  Ly.rec_val = nullptr;
  cudaFree(Ly.vals32);
  Ly.vals32 = nullptr;
  Ly.near_frac = 1.0;
  for (auto* w : Ly.win) gs_win_destroy(w);
  Ly.win.clear();
  for (auto* e : Ly.sell) gs_sell_destroy(e);
  Ly.sell.clear();
  for (auto* e : Ly.lanepad) gs_lanepad_destroy(e);
  Ly.lanepad.clear();
  cudaFree(Ly.recs);
  Ly.recs = nullptr;
  do {
    rc = gs_permute_graph(ctx, f->scaled, Ly.order, Ly.newpos, &Ly.perm);
    if (rc) break;
    const int64_t nnz = Ly.perm->nnz;  // fp32 copy of the permuted values (optional fp32 mode)
    if (cudaMalloc((void**)&Ly.vals32, (size_t)(nnz + kCsrPad) * sizeof(float)) != cudaSuccess) {
      rc = gs_fail(ctx, ERRC_INVALID_ARGUMENT, "fp32 value allocation failed");
    } else if (nnz > 0) {
      gs_launch_begin(ctx, 1);
      k_to_float<<<(unsigned)((nnz + 255) / 256), 256, 0, s>>>(Ly.perm->vals, nnz, Ly.vals32);
      gs_launch_end(ctx, 1);
      if (cudaStreamSynchronize(s) != cudaSuccess) rc = gs_fail(ctx, ERRC_INVALID_ARGUMENT, "fp32 copy failed");
    }
    if (!rc && nnz > 0) {  // index locality of this layout (choose_rpc)
      DevBuf<unsigned long long> cnt;
      unsigned long long h = 0;
      if (cnt.alloc(1, s) == cudaSuccess && cudaMemsetAsync(cnt.get(), 0, sizeof h, s) == cudaSuccess) {
        k_near_count<<<148 * 4, 256, 0, s>>>(Ly.perm->offs, Ly.perm->cols, Ly.perm->n, cnt.get());
        if (cudaMemcpyAsync(&h, cnt.get(), sizeof h, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
            cudaStreamSynchronize(s) == cudaSuccess)
          Ly.near_frac = (double)h / (double)nnz;
      }
    }
  } while (0);
  return rc;
}

extern "C" int gs_filter_create(gs_ctx* ctx, const gs_graph* L, int kind, double lambda_bound,
                                double t, int degree, gs_filter** out) {
  *out = nullptr;
  if (!(t > 0.0 && std::isfinite(t))) return gs_fail(ctx, ERRC_NON_POSITIVE_TIME, "diffusion time must be > 0");
  if (degree < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "Chebyshev degree must be >= 1");
  double scale;
  if (kind == GS_LAPLACIAN_NORMALIZED) {
    scale = 1.0;
  } else {
    if (!(lambda_bound >= 0.0 && std::isfinite(lambda_bound)))
      return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "bad lambda_max_bound");
    scale = lambda_bound > 1e-300 ? 2.0 / lambda_bound : 1.0;
  }
  gs_filter* f = new gs_filter();
  f->t = t;
  f->scale = scale;
  f->t_eff = t / scale;
  f->degree = degree;
  f->kind = kind;
  f->coeffs.assign(degree + 1, 0.0);
  cudaStream_t s = ctx->stream;
  int rc = gs_graph_alloc(ctx, L->n, L->nnz, &f->scaled);
  if (!rc) {
    cudaMemcpyAsync(f->scaled->offs, L->offs, ((size_t)L->n + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(f->scaled->cols, L->cols, (size_t)L->nnz * sizeof(int), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(f->scaled->vals, L->vals, (size_t)L->nnz * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (L->nnz > 0) {
      gs_launch_begin(ctx, 1);
      k_scale_vals<<<(unsigned)((L->nnz + 255) / 256), 256, 0, s>>>(f->scaled->vals, L->nnz, scale);
      gs_launch_end(ctx, 1);
    }
    if (cudaMalloc((void**)&f->d_coeffs, (degree + 1) * sizeof(double)) != cudaSuccess)
      rc = gs_fail(ctx, ERRC_INVALID_ARGUMENT, "coefficient allocation failed");
  }
  if (!rc) rc = gs_coefficients_impl(ctx, f->t_eff, degree, f->d_coeffs, f->coeffs.data());
  // two locality layouts (gs_reorder.cu): plain Cuthill-McKee, and CM with degree-sorted
  // windows of 256 rows for narrow batches (several rows per warp)
  int sigma = 256;
  if (const char* e = getenv("GS_SIGMA")) sigma = atoi(e);
  if (!rc) {
    const int n = L->n;
    for (int l = 0; l < 2 && !rc; ++l)
      if (cudaMalloc((void**)&f->lay[l].order, ((size_t)n + 1) * sizeof(int)) != cudaSuccess ||
          cudaMalloc((void**)&f->lay[l].newpos, ((size_t)n + 1) * sizeof(int)) != cudaSuccess)
        rc = gs_fail(ctx, ERRC_INVALID_ARGUMENT, "permutation allocation failed");
  }
  // Cuthill-McKee order first; its index locality picks the window of the degree sort unless
  // GS_SIGMA fixes it: graphs without locality (kNN in R^30: ~12% of the entries within 256 rows)
  // lose nothing to wider windows and gain rows of equal length per warp (config 2 step 293 -> 280
  // us, config 4 1442 -> 1326 us with 2048), the swiss roll (~50%) keeps 256 (config 3's gathers
  // live on that locality: 60 -> 94 us at 2048 on the n = 2e6 shape)
  if (!rc) rc = gs_bfs_order(ctx, f->scaled, f->lay[0].order, f->lay[0].newpos, 0, nullptr, nullptr);
  if (!rc) rc = finish_layout(ctx, f, 0);
  // (large graphs only: the member-sharded leg at n = 2e5 -- two waves of tiles -- ran 209
  // barycenter sweeps/s with 256-row windows and 162 with 2048)
  if (!rc && !getenv("GS_SIGMA") && f->lay[0].near_frac < 0.3 && L->n >= 500000) sigma = 2048;
  if (!rc) {
    if (sigma > 1) {
      rc = gs_sigma_order(ctx, f->scaled, f->lay[0].newpos, sigma, f->lay[1].order, f->lay[1].newpos);
    } else {
      const size_t nb = (size_t)L->n * sizeof(int);
      if (cudaMemcpy(f->lay[1].order, f->lay[0].order, nb, cudaMemcpyDeviceToDevice) != cudaSuccess ||
          cudaMemcpy(f->lay[1].newpos, f->lay[0].newpos, nb, cudaMemcpyDeviceToDevice) != cudaSuccess)
        rc = gs_fail(ctx, ERRC_INVALID_ARGUMENT, "order copy failed");
    }
  }
  if (!rc) rc = finish_layout(ctx, f, 1);
  if (rc) {
    gs_filter_destroy(f);
    return rc;
  }
  f->sigma = sigma;
  *out = f;
  return GS_OK;
}

extern "C" void gs_filter_destroy(gs_filter* f) {
  if (!f) return;
  gs_graph_destroy(f->scaled);
  for (auto& Ly : f->lay) {
    gs_graph_destroy(Ly.perm);
    cudaFree(Ly.order);
    cudaFree(Ly.newpos);
    cudaFree(Ly.vals32);
    cudaFree(Ly.rec_key);
    cudaFree(Ly.rec_val);
    for (auto* w : Ly.win) gs_win_destroy(w);
    for (auto* e : Ly.sell) gs_sell_destroy(e);
    for (auto* e : Ly.lanepad) gs_lanepad_destroy(e);
    cudaFree(Ly.recs);
  }
  cudaFree(f->d_coeffs);
  delete f;
}

extern "C" int gs_filter_info(const gs_filter* f, int* n, double* t, double* t_eff, double* scale,
                              int* degree, int* kind) {
  if (n) *n = f->scaled->n;
  if (t) *t = f->t;
  if (t_eff) *t_eff = f->t_eff;
  if (scale) *scale = f->scale;
  if (degree) *degree = f->degree;
  if (kind) *kind = f->kind;
  return GS_OK;
}

extern "C" int gs_filter_coefficients(const gs_filter* f, double* out) {
  memcpy(out, f->coeffs.data(), f->coeffs.size() * sizeof(double));
  return GS_OK;
}

extern "C" const gs_graph* gs_filter_scaled(const gs_filter* f) { return f->scaled; }

extern "C" int gs_filter_order(gs_ctx* ctx, const gs_filter* f, int* order, int mem) {
  GS_TRY(gs_copy_out(ctx, order, f->lay[0].order, (size_t)f->scaled->n * sizeof(int), mem));
  return gs_ctx_synchronize(ctx);
}

// Caller-supplied locality order for layout `layout` (0: wide column groups, 1: narrow ones).
// Results do not depend on it: every row keeps its entries in the original column order.
__global__ void k_newpos_from_order(const int* order, int n, int* newpos, int* bad) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int o = order[r];
  if (o < 0 || o >= n) {
    *bad = 1;
    return;
  }
  if (atomicExch(newpos + o, r) != -1) *bad = 1;
}

extern "C" int gs_filter_set_order(gs_ctx* ctx, gs_filter* f, int layout, const int* order, int mem) {
  if (!f || layout < 0 || layout > 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "gs_filter_set_order: bad layout");
  if (layout == 1) f->sigma = 0;  // a caller's order has no degree-sorted windows
  const int n = f->scaled->n;
  if (n == 0) return GS_OK;
  cudaStream_t s = ctx->stream;
  gs_layout& Ly = f->lay[layout];
  GS_CUDA(ctx, cudaMemcpyAsync(Ly.order, order, (size_t)n * sizeof(int),
                               mem == GS_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
  GS_CUDA(ctx, cudaMemsetAsync(Ly.newpos, 0xff, (size_t)n * sizeof(int), s));
  DevBuf<int> bad;
  GS_CUDA(ctx, bad.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_newpos_from_order<<<(n + 255) / 256, 256, 0, s>>>(Ly.order, n, Ly.newpos, bad.get());
  gs_launch_end(ctx, 1);
  int hb = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (hb) {  // restore a valid state: identity
    std::vector<int> id(n);
    for (int i = 0; i < n; ++i) id[i] = i;
    cudaMemcpy(Ly.order, id.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemcpy(Ly.newpos, id.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice);
    finish_layout(ctx, f, layout);
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "gs_filter_set_order: order is not a permutation of 0..n-1");
  }
  return finish_layout(ctx, f, layout);
}

int gs_layout_from_order(gs_ctx* ctx, gs_filter* f, int l, const int* h_order) {
  const int n = f->scaled->n;
  gs_layout& Ly = f->lay[l];
  cudaStream_t s = ctx->stream;
  if (!Ly.order) {
    GS_CUDA(ctx, cudaMalloc((void**)&Ly.order, ((size_t)n + 1) * sizeof(int)));
    GS_CUDA(ctx, cudaMalloc((void**)&Ly.newpos, ((size_t)n + 1) * sizeof(int)));
  }
  if (n == 0) return finish_layout(ctx, f, l);
  GS_CUDA(ctx, cudaMemcpyAsync(Ly.order, h_order, (size_t)n * sizeof(int), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemsetAsync(Ly.newpos, 0xff, (size_t)n * sizeof(int), s));
  DevBuf<int> bad;
  GS_CUDA(ctx, bad.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_newpos_from_order<<<(n + 255) / 256, 256, 0, s>>>(Ly.order, n, Ly.newpos, bad.get());
  gs_launch_end(ctx, 1);
  int hb = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (hb) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "layout order is not a permutation");
  return finish_layout(ctx, f, l);
}

// heat.cpp:116-131
extern "C" int gs_filter_apply_ex(gs_ctx* ctx, const gs_filter* f, const double* X, double* Y,
                                  int width, int mem, int flags) {
  const int n = f->scaled->n;
  if (width < 0) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "width");
  if (width == 0 || n == 0) return GS_OK;
  DevBuf<double> xin, yout;
  const double* dX = nullptr;
  GS_TRY(stage_in(ctx, xin, X, (size_t)width * n, mem, &dX));
  double* dY = Y;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, yout.alloc((size_t)width * n, ctx->stream));
    dY = yout.get();
  }
  const int rc = (flags & GS_FLAG_FP32) ? filter_apply_impl<float>(ctx, f, dX, dY, width)
                                        : filter_apply_impl<double>(ctx, f, dX, dY, width);
  if (rc) return rc;
  GS_TRY(finish_out(ctx, yout, Y, (size_t)width * n, mem));
  GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GS_OK;
}

extern "C" int gs_filter_apply(gs_ctx* ctx, const gs_filter* f, const double* X, double* Y,
                               int width, int mem) {
  return gs_filter_apply_ex(ctx, f, X, Y, width, mem, 0);
}

// sparse.cpp:70-99 (fp64, the graph's own vertex order)
extern "C" int gs_graph_multiply(gs_ctx* ctx, const gs_graph* g, const double* x, double* y,
                                 int width, int mem) {
  const int n = g->n;
  if (width <= 0 || n == 0) return GS_OK;
  cudaStream_t s = ctx->stream;
  Work<double> w;
  GS_TRY(w.init(ctx, n, width, false));
  DevBuf<double> xin, yout;
  const double* dX = nullptr;
  GS_TRY(stage_in(ctx, xin, x, (size_t)width * n, mem, &dX));
  double* dY = y;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, yout.alloc((size_t)width * n, s));
    dY = yout.get();
  }
  gs_launch_begin(ctx, 1);
  k_pack<double><<<grid_for((int64_t)w.Bpad * n), kThreads, 0, s>>>(dX, w.T[0].get(), n, width, w.GW, w.G, nullptr, (int64_t)n);
  gs_launch_end(ctx, 1);
  StepArgs A{};
  A.offs = g->offs;
  A.cols = g->cols;
  A.vals = g->vals;
  A.lane = lane_enabled();
  A.n = n;
  A.ld = n;
  A.tiles = w.tiles;
  A.Gl = w.G;
  A.Bpad = w.Bpad;
  A.k = 0;
  A.Tprev = w.T[0].get();
  A.Tout = w.T[1].get();
  launch_step<double>(ctx, w.GW, w.rpc, A, MODE_NONE);
  gs_launch_begin(ctx, 1);
  k_unpack<double><<<grid_for((int64_t)width * n), kThreads, 0, s>>>(w.T[1].get(), dY, n, width, w.GW, nullptr, nullptr, nullptr, (int64_t)n);
  gs_launch_end(ctx, 1);
  GS_TRY(finish_out(ctx, yout, y, (size_t)width * n, mem));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// ============================================================================================
// Geodesic Sinkhorn batch (transport.cpp:108-255)
// ============================================================================================
extern "C" int gs_sinkhorn(gs_ctx* ctx, const gs_filter* f, const double* a, const double* mus,
                           const double* nus, int P, int max_iter, double tol, int flags, int mem,
                           double* out_v, double* out_w, double* out_cost, double* out_kl,
                           int* out_iters, int* out_conv, double* out_err, int* fail_pair,
                           int* fail_sweep) {
  if (fail_pair) *fail_pair = -1;
  if (fail_sweep) *fail_sweep = 0;
  const int n = f->scaled->n;
  if (P < 0) return gs_fail(ctx, ERRC_SIZE_MISMATCH, "pair lists differ in length");
  if (P == 0) return GS_OK;
  // ---- stage + validate (check_transport_inputs, transport.cpp:56-66) -------------------------
  DevBuf<double> bmu, bnu, ba;
  const double *dmu, *dnu, *da;
  GS_TRY(stage_in(ctx, bmu, mus, (size_t)P * n, mem, &dmu));
  GS_TRY(stage_in(ctx, bnu, nus, (size_t)P * n, mem, &dnu));
  GS_TRY(stage_in(ctx, ba, a, (size_t)n, mem, &da));
  GS_TRY(gs_check_transport_inputs(ctx, n, dmu, dnu, da, P, max_iter, tol));
  if (flags & GS_FLAG_FP32)
    return sinkhorn_impl<float>(ctx, f, da, dmu, dnu, P, max_iter, tol, flags, mem, out_v, out_w,
                                out_cost, out_kl, out_iters, out_conv, out_err, fail_pair, fail_sweep);
  return sinkhorn_impl<double>(ctx, f, da, dmu, dnu, P, max_iter, tol, flags, mem, out_v, out_w,
                               out_cost, out_kl, out_iters, out_conv, out_err, fail_pair, fail_sweep);
}

// ============================================================================================
// Barycenter (barycenter.cpp:45-107)
// ============================================================================================
extern "C" int gs_barycenter_ex(gs_ctx* ctx, const gs_filter* f, const double* a,
                                const double* members, int m, const double* alphas, int max_iter,
                                double tol, int mem, const gs_comm* comm, int flags,
                                double* out_bary, double* out_V, double* out_W, int* out_iters,
                                int* out_conv, double* out_err) {
  const int n = f->scaled->n;
  DevBuf<double> bmem, ba;
  const double *dmem = nullptr, *da = nullptr;
  std::vector<double> al(m > 0 ? m : 1);
  // validation (barycenter.cpp:32-43 family.validate, weights, parameters); with a comm the
  // outcome is agreed across the member shards before anyone returns, so a rank that fails
  // never leaves the others waiting in a collective
  auto validate = [&]() -> int {
    if (m < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "family must be non-empty");
    GS_TRY(stage_in(ctx, bmem, members, (size_t)m * n, mem, &dmem));
    GS_TRY(stage_in(ctx, ba, a, (size_t)n, mem, &da));
    {
      std::vector<double> sm;
      std::vector<int> fm, gm;
      GS_TRY(validate_columns(ctx, dmem, n, m, sm, fm, gm));
      for (int c = 0; c < m; ++c) GS_TRY(check_distribution(ctx, n, sm[c], fm[c], gm[c]));
    }
    if (alphas) {
      if (mem == GS_MEM_DEVICE) {
        GS_CUDA(ctx, cudaMemcpy(al.data(), alphas, m * sizeof(double), cudaMemcpyDeviceToHost));
      } else {
        memcpy(al.data(), alphas, m * sizeof(double));
      }
    } else {
      for (int c = 0; c < m; ++c) al[c] = 1.0 / (double)m;
    }
    double asum = 0.0;
    for (int c = 0; c < m; ++c) {
      if (!(al[c] >= 0.0)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "alphas must be non-negative");
      asum += al[c];
    }
    if (!comm && !(std::fabs(asum - 1.0) <= 1e-9)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "alphas must sum to 1");
    GS_TRY(check_weights(ctx, da, n));
    if (!(tol > 0.0 && max_iter >= 1)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "bad parameters");
    return GS_OK;
  };
  int vrc = validate();
  if (comm && comm->allreduce) {
    DevBuf<double> flag;
    GS_CUDA(ctx, flag.alloc(1, ctx->stream));
    const double hv = (double)vrc;
    GS_CUDA(ctx, cudaMemcpyAsync(flag.get(), &hv, sizeof hv, cudaMemcpyHostToDevice, ctx->stream));
    if (comm->allreduce(comm->user, flag.get(), 1, 1, (void*)ctx->stream)) {
      ctx->err = "NcclError: allreduce hook failed";
      return GS_ERR_NCCL;
    }
    double agreed = 0.0;
    GS_CUDA(ctx, cudaMemcpyAsync(&agreed, flag.get(), sizeof agreed, cudaMemcpyDeviceToHost, ctx->stream));
    GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (vrc == 0 && agreed != 0.0) {
      const int code = (int)agreed;
      if (code >= 1 && code <= 16) return gs_fail(ctx, code - 1, "barycenter inputs rejected on another rank");
      ctx->err = "barycenter inputs rejected on another rank";
      return code;
    }
  }
  if (vrc) return vrc;
  if (flags & GS_FLAG_FP32)
    return barycenter_impl<float>(ctx, f, da, dmem, m, al, max_iter, tol, mem, comm, out_bary,
                                  out_V, out_W, out_iters, out_conv, out_err);
  return barycenter_impl<double>(ctx, f, da, dmem, m, al, max_iter, tol, mem, comm, out_bary, out_V,
                                 out_W, out_iters, out_conv, out_err);
}

extern "C" int gs_barycenter(gs_ctx* ctx, const gs_filter* f, const double* a,
                             const double* members, int m, const double* alphas, int max_iter,
                             double tol, int mem, const gs_comm* comm, double* out_bary,
                             double* out_V, double* out_W, int* out_iters, int* out_conv,
                             double* out_err) {
  return gs_barycenter_ex(ctx, f, a, members, m, alphas, max_iter, tol, mem, comm, 0, out_bary,
                          out_V, out_W, out_iters, out_conv, out_err);
}

// ============================================================================================
// Plan rows (transport.cpp:314-324): row i of diag(v) H_t diag(a .* w) through one filter
// application to the unit impulse e_i, clamped at zero -- batched over `nrows` impulses, which is
// the same Chebyshev kernel with B = nrows (the paper's displacement-interpolation use case).
// ============================================================================================
namespace {
__global__ void k_impulses(const int* rows, int nrows, int n, double* X) {
  const int64_t total = (int64_t)nrows * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(e / n), i = (int)(e % n);
    X[e] = i == rows[q] ? 1.0 : 0.0;
  }
}

__global__ void k_plan_rows(const int* rows, int nrows, int n, const double* a, const double* v,
                            const double* w, double* Y) {
  const int64_t total = (int64_t)nrows * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(e / n), j = (int)(e % n);
    const double r = v[rows[q]] * (Y[e] * (a[j] * w[j]));
    Y[e] = fmax(r, 0.0);
  }
}
}  // namespace

extern "C" int gs_plan_rows(gs_ctx* ctx, const gs_filter* f, const double* a, const double* v,
                            const double* w, const int* rows, int nrows, int mem, double* out) {
  const int n = f->scaled->n;
  if (nrows <= 0) return GS_OK;
  cudaStream_t s = ctx->stream;
  std::vector<int> hrows(nrows);
  if (mem == GS_MEM_DEVICE) {
    GS_CUDA(ctx, cudaMemcpy(hrows.data(), rows, nrows * sizeof(int), cudaMemcpyDeviceToHost));
  } else {
    memcpy(hrows.data(), rows, nrows * sizeof(int));
  }
  for (int q = 0; q < nrows; ++q)
    if (hrows[q] < 0 || hrows[q] >= n) return gs_fail(ctx, ERRC_INDEX_OUT_OF_RANGE, "plan row index");
  DevBuf<double> ba, bv, bw, X, Y;
  DevBuf<int> drows;
  const double *da, *dv, *dw;
  GS_TRY(stage_in(ctx, ba, a, n, mem, &da));
  GS_TRY(stage_in(ctx, bv, v, n, mem, &dv));
  GS_TRY(stage_in(ctx, bw, w, n, mem, &dw));
  GS_CUDA(ctx, drows.alloc(nrows, s));
  GS_CUDA(ctx, cudaMemcpyAsync(drows.get(), hrows.data(), nrows * sizeof(int), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, X.alloc((size_t)nrows * n, s));
  GS_CUDA(ctx, Y.alloc((size_t)nrows * n, s));
  gs_launch_begin(ctx, 1);
  k_impulses<<<grid_for((int64_t)nrows * n), kThreads, 0, s>>>(drows.get(), nrows, n, X.get());
  gs_launch_end(ctx, 1);
  GS_TRY(filter_apply_impl<double>(ctx, f, X.get(), Y.get(), nrows));
  gs_launch_begin(ctx, 1);
  k_plan_rows<<<grid_for((int64_t)nrows * n), kThreads, 0, s>>>(drows.get(), nrows, n, da, dv, dw, Y.get());
  gs_launch_end(ctx, 1);
  GS_TRY(gs_copy_out(ctx, out, Y.get(), (size_t)nrows * n * sizeof(double), mem));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// ============================================================================================
// Row-partitioned entry points (gs_part.cu)
// ============================================================================================
extern "C" int gs_part_filter_apply(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const double* X,
                                    double* Y, int width, int flags, int mem) {
  GS_TRY(check_part_comm(ctx, p, comm));
  if (width < 0) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "width");
  if (width == 0) return GS_OK;
  const int nl = p->nl;
  DevBuf<double> xin, yout;
  const double* dX = nullptr;
  GS_TRY(stage_in(ctx, xin, X, (size_t)width * nl, mem, &dX));
  double* dY = Y;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, yout.alloc((size_t)width * nl, ctx->stream));
    dY = yout.get();
  }
  const int rc = (flags & GS_FLAG_FP32) ? filter_apply_part_impl<float>(ctx, p, comm, dX, dY, width)
                                        : filter_apply_part_impl<double>(ctx, p, comm, dX, dY, width);
  if (rc) return rc;
  GS_TRY(finish_out(ctx, yout, Y, (size_t)width * nl, mem));
  GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GS_OK;
}

extern "C" int gs_part_sinkhorn(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const double* a,
                                const double* mus, const double* nus, int P, int max_iter, double tol,
                                int flags, int mem, double* out_v, double* out_w, double* out_cost,
                                double* out_kl, int* out_iters, int* out_conv, double* out_err,
                                int* fail_pair, int* fail_sweep) {
  if (fail_pair) *fail_pair = -1;
  if (fail_sweep) *fail_sweep = 0;
  GS_TRY(check_part_comm(ctx, p, comm));
  const int nl = p->nl;
  if (P < 0) return gs_fail(ctx, ERRC_SIZE_MISMATCH, "pair lists differ in length");
  if (P == 0) return GS_OK;
  DevBuf<double> bmu, bnu, ba;
  const double *dmu, *dnu, *da;
  GS_TRY(stage_in(ctx, bmu, mus, (size_t)P * nl, mem, &dmu));
  GS_TRY(stage_in(ctx, bnu, nus, (size_t)P * nl, mem, &dnu));
  GS_TRY(stage_in(ctx, ba, a, (size_t)nl, mem, &da));
  {  // check_transport_inputs (transport.cpp:56-66) on the combined column sums, pair order
    std::vector<double> smu, snu;
    std::vector<int> fmu, gmu, fnu, gnu;
    GS_TRY(validate_columns_part(ctx, p, comm, dmu, P, smu, fmu, gmu));
    GS_TRY(validate_columns_part(ctx, p, comm, dnu, P, snu, fnu, gnu));
    bool wbad = false;
    GS_TRY(weights_bad_part(ctx, p, comm, da, &wbad));  // collective: every rank calls it once
    const int n = p->n_global;
    for (int q = 0; q < P; ++q) {
      GS_TRY(check_distribution(ctx, n, smu[q], fmu[q], gmu[q]));
      GS_TRY(check_distribution(ctx, n, snu[q], fnu[q], gnu[q]));
      if (q == 0 && wbad) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "vertex weights must be positive");
      if (!(tol > 0.0)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "tolerance must be positive");
      if (max_iter < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "max_iter must be >= 1");
    }
  }
  if (flags & GS_FLAG_FP32)
    return sinkhorn_part_impl<float>(ctx, p, comm, da, dmu, dnu, P, max_iter, tol, flags, mem, out_v, out_w,
                                     out_cost, out_kl, out_iters, out_conv, out_err, fail_pair, fail_sweep);
  return sinkhorn_part_impl<double>(ctx, p, comm, da, dmu, dnu, P, max_iter, tol, flags, mem, out_v, out_w,
                                    out_cost, out_kl, out_iters, out_conv, out_err, fail_pair, fail_sweep);
}

int gs_group_width(int B) { return choose_gw(B); }

int gs_spmm_grouped(gs_ctx* ctx, const gs_graph* g, const double* x, double* y, int B) {
  const int n = g->n;
  if (n == 0 || B <= 0) return GS_OK;
  const int GW = choose_gw(B), G = (B + GW - 1) / GW;
  const int rpc = choose_rpc<double>(n, GW, G);
  StepArgs A{};
  A.offs = g->offs;
  A.cols = g->cols;
  A.vals = g->vals;
  A.lane = lane_enabled();
  A.n = n;
  A.ld = n;
  A.tiles = (n + rows_per_block<double>(GW) * rpc - 1) / (rows_per_block<double>(GW) * rpc);
  A.Gl = G;
  A.Bpad = G * GW;
  A.k = 0;
  A.Tprev = x;
  A.Tout = y;
  launch_step<double>(ctx, GW, rpc, A, MODE_NONE);
  GS_CUDA(ctx, cudaGetLastError());
  return GS_OK;
}

// check_transport_inputs (transport.cpp:56-66) over P device column pairs, in pair order
int gs_check_transport_inputs(gs_ctx* ctx, int n, const double* dmu, const double* dnu, const double* da,
                              int P, int max_iter, double tol) {
  std::vector<double> smu, snu;
  std::vector<int> fmu, gmu, fnu, gnu;
  GS_TRY(validate_columns(ctx, dmu, n, P, smu, fmu, gmu));
  GS_TRY(validate_columns(ctx, dnu, n, P, snu, fnu, gnu));
  bool a_checked = false;
  for (int p = 0; p < P; ++p) {
    GS_TRY(check_distribution(ctx, n, smu[p], fmu[p], gmu[p]));
    GS_TRY(check_distribution(ctx, n, snu[p], fnu[p], gnu[p]));
    if (!a_checked) {
      GS_TRY(check_weights(ctx, da, n));
      a_checked = true;
    }
    if (!(tol > 0.0)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "tolerance must be positive");
    if (max_iter < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "max_iter must be >= 1");
  }
  return GS_OK;
}
