// gs_dense.cu -- dense entropic Sinkhorn on the device (proj/src/transport.cpp:271-311) and the
// kNN benchmark's dense baselines (proj/src/bench.cpp:311-331, squared_distances bench.cpp:32-39;
// the dense_sinkhorn_w1 / dense_sinkhorn_w2 rows of the benchmark table).
//
// A batch of P independent problems (pairs of point groups in the benchmark, one caller matrix in
// gs_dense_sinkhorn). Per pair the cost C (r x c) and the kernel K = exp(-C / lambda) are formed
// once on the device, K in both orientations so that each matrix-vector product reads it
// coalesced: phi = K w with one thread per row i over the column-major copy, psi = K^T v with
// one thread per column j over the row-major copy. Summation orders are the oracle's
// (go_dense_sinkhorn): sequential fma chains in index order for phi_i, psi_j and the cost, a
// sequential sum for the marginal error, so every value produced by + - * / fma matches it bit
// for bit; exp and log come from libdevice (<= 1 ulp from glibc). Converged pairs are masked, as
// running each pair's loop separately would leave them.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "gs_internal.cuh"
#include "geosink_b200.h"

namespace {

constexpr int kT = 256;

struct DensePairs {  // device arrays, P pairs
  int P = 0;
  DevBuf<int> r, c;           // sizes
  DevBuf<long long> koff;     // offset of pair p's r*c block
  DevBuf<long long> roff, coff;  // offsets of its r- and c-vectors
  DevBuf<double> C, K, Kt;    // r x c row-major (C, K) and column-major (Kt)
  DevBuf<double> mu, nu, v, w, phi, e, t;
  DevBuf<int> active, iters, conv, bad;
  DevBuf<double> err, cost, kl;
  int max_r = 0, max_c = 0;
  long long total_rc = 0, total_r = 0, total_c = 0;
};

__global__ void k_dense_cost_groups(const double* __restrict__ X, int d, const int* __restrict__ gidx,
                                    const int* __restrict__ goff, const int* __restrict__ pa,
                                    const int* __restrict__ pb, const long long* __restrict__ koff,
                                    const int* __restrict__ rr, const int* __restrict__ cc, int squared,
                                    double* __restrict__ C) {
  const int p = blockIdx.y;
  const int r = rr[p], c = cc[p];
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)r * c) return;
  const int i = (int)(q / c), j = (int)(q % c);
  const double* x = X + (size_t)gidx[goff[pa[p]] + i] * d;
  const double* y = X + (size_t)gidx[goff[pb[p]] + j] * d;
  double xn = 0.0, yn = 0.0, dot = 0.0;
  for (int k = 0; k < d; ++k) xn = fma(x[k], x[k], xn);
  for (int k = 0; k < d; ++k) {
    yn = fma(y[k], y[k], yn);
    dot = fma(x[k], y[k], dot);
  }
  double v = fmax((-2.0 * dot + xn) + yn, 0.0);  // bench.cpp:32-39
  if (!squared) v = sqrt(v);                     // cost.cwiseSqrt(), bench.cpp:327
  C[koff[p] + q] = v;
}

// K = exp(-C / lambda) (transport.cpp:282), both orientations
__global__ void k_dense_kernel(const double* __restrict__ C, const long long* __restrict__ koff,
                               const int* __restrict__ rr, const int* __restrict__ cc, double lambda,
                               double* __restrict__ K, double* __restrict__ Kt, int* __restrict__ nonfinite) {
  const int p = blockIdx.y;
  const int r = rr[p], c = cc[p];
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)r * c) return;
  const int i = (int)(q / c), j = (int)(q % c);
  const double cv = C[koff[p] + q];
  if (!isfinite(cv)) nonfinite[p] = 1;
  const double k = exp(-cv / lambda);
  K[koff[p] + q] = k;
  Kt[koff[p] + (long long)j * r + i] = k;
}

// per pair: some row / column of K is all zero (transport.cpp:283-288); bad = 1 row, 2 column
__global__ void k_dense_underflow(const double* __restrict__ K, const double* __restrict__ Kt,
                                  const long long* __restrict__ koff, const int* __restrict__ rr,
                                  const int* __restrict__ cc, int* __restrict__ bad) {
  const int p = blockIdx.y;
  const int r = rr[p], c = cc[p];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < r) {  // row t: contiguous in K
    double mx = 0.0;
    for (int j = 0; j < c; ++j) mx = fmax(mx, K[koff[p] + (long long)t * c + j]);
    if (!(mx > 0.0)) atomicOr(bad + p, 1);
  }
  if (t < c) {  // column t: contiguous in Kt
    double mx = 0.0;
    for (int i = 0; i < r; ++i) mx = fmax(mx, Kt[koff[p] + (long long)t * r + i]);
    if (!(mx > 0.0)) atomicOr(bad + p, 2);
  }
}

__global__ void k_dense_init(const long long* __restrict__ roff, const long long* __restrict__ coff,
                             const int* __restrict__ rr, const int* __restrict__ cc, double* v, double* w) {
  const int p = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < rr[p]) v[roff[p] + t] = 0.0;
  if (t < cc[p]) w[coff[p] + t] = 1.0;
}

// phi_i = sum_j K_ij w_j (fma chain, j ascending); with `mu`: e_i = |v_i phi_i - mu_i|
__global__ void k_dense_rows(const double* __restrict__ Kt, const long long* __restrict__ koff,
                             const long long* __restrict__ roff, const long long* __restrict__ coff,
                             const int* __restrict__ rr, const int* __restrict__ cc,
                             const int* __restrict__ active, const double* __restrict__ w,
                             const double* __restrict__ v, const double* __restrict__ mu,
                             double* __restrict__ phi, double* __restrict__ e) {
  const int p = blockIdx.y;
  if (active && !active[p]) return;
  const int r = rr[p], c = cc[p];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r) return;
  const double* __restrict__ kp = Kt + koff[p] + i;
  const double* __restrict__ wp = w + coff[p];
  double s = 0.0;
#pragma unroll 8
  for (int j = 0; j < c; ++j) s = fma(__ldg(kp + (long long)j * r), __ldg(wp + j), s);
  phi[roff[p] + i] = s;
  if (mu) e[roff[p] + i] = fabs(v[roff[p] + i] * s - mu[roff[p] + i]);  // transport.cpp:300
}

// v_i = mu_i / max(phi_i, floor) (transport.cpp:297)
__global__ void k_dense_v(const long long* __restrict__ roff, const int* __restrict__ rr,
                          const int* __restrict__ active, const double* __restrict__ mu,
                          const double* __restrict__ phi, double* __restrict__ v) {
  const int p = blockIdx.y;
  if (!active[p]) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rr[p]) v[roff[p] + i] = mu[roff[p] + i] / fmax(phi[roff[p] + i], GS_FLOOR);
}

// w_j = nu_j / max(sum_i K_ij v_i, floor) (transport.cpp:298; fma chain, i ascending)
__global__ void k_dense_cols(const double* __restrict__ K, const long long* __restrict__ koff,
                             const long long* __restrict__ roff, const long long* __restrict__ coff,
                             const int* __restrict__ rr, const int* __restrict__ cc,
                             const int* __restrict__ active, const double* __restrict__ v,
                             const double* __restrict__ nu, double* __restrict__ w) {
  const int p = blockIdx.y;
  if (!active[p]) return;
  const int r = rr[p], c = cc[p];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= c) return;
  const double* __restrict__ kp = K + koff[p] + j;
  const double* __restrict__ vp = v + roff[p];
  double s = 0.0;
#pragma unroll 8
  for (int i = 0; i < r; ++i) s = fma(__ldg(kp + (long long)i * c), __ldg(vp + i), s);
  w[coff[p] + j] = nu[coff[p] + j] / fmax(s, GS_FLOOR);
}

// per pair (one thread): err = sequential sum of e_i; iterations, convergence (transport.cpp:300-305)
__global__ void k_dense_ctl(const long long* __restrict__ roff, const int* __restrict__ rr, int P, int it,
                            double tol, const double* __restrict__ e, int* active, int* iters, int* conv,
                            double* err, int* n_active) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P || !active[p]) return;
  double s = 0.0;
  for (int i = 0; i < rr[p]; ++i) s = s + e[roff[p] + i];
  err[p] = s;
  iters[p] = it;
  if (s <= tol) {
    conv[p] = 1;
    active[p] = 0;
    atomicSub(n_active, 1);
  }
}

// t_i = sum_j (K_ij C_ij) w_j (transport.cpp:308, inner products)
__global__ void k_dense_cost_rows(const double* __restrict__ K, const double* __restrict__ C,
                                  const long long* __restrict__ koff, const long long* __restrict__ roff,
                                  const long long* __restrict__ coff, const int* __restrict__ rr,
                                  const int* __restrict__ cc, const double* __restrict__ w,
                                  double* __restrict__ t) {
  const int p = blockIdx.y;
  const int r = rr[p], c = cc[p];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r) return;
  const double* kp = K + koff[p] + (long long)i * c;
  const double* cp = C + koff[p] + (long long)i * c;
  const double* wp = w + coff[p];
  double s = 0.0;
  for (int j = 0; j < c; ++j) s = fma(kp[j] * cp[j], wp[j], s);
  t[roff[p] + i] = s;
}

// cost = v . t (fma chain); kl = plain_log_sum(mu, max(v, floor)) + plain_log_sum(nu, max(w, floor)) - 1
__global__ void k_dense_final(const long long* __restrict__ roff, const long long* __restrict__ coff,
                              const int* __restrict__ rr, const int* __restrict__ cc, int P,
                              const double* __restrict__ v, const double* __restrict__ w,
                              const double* __restrict__ t, const double* __restrict__ mu,
                              const double* __restrict__ nu, double* cost, double* kl) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double cs = 0.0;
  for (int i = 0; i < rr[p]; ++i) cs = fma(v[roff[p] + i], t[roff[p] + i], cs);
  cost[p] = cs;
  double k1 = 0.0, k2 = 0.0;
  for (int i = 0; i < rr[p]; ++i) {
    const double m = mu[roff[p] + i];
    if (m > 0.0) k1 = k1 + m * log(fmax(v[roff[p] + i], GS_FLOOR));
  }
  for (int j = 0; j < cc[p]; ++j) {
    const double m = nu[coff[p] + j];
    if (m > 0.0) k2 = k2 + m * log(fmax(w[coff[p] + j], GS_FLOOR));
  }
  kl[p] = k1 + k2 - 1.0;
}

// uniform marginals 1/size (Distribution::uniform)
__global__ void k_dense_uniform(const long long* __restrict__ roff, const long long* __restrict__ coff,
                                const int* __restrict__ rr, const int* __restrict__ cc, double* mu, double* nu) {
  const int p = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < rr[p]) mu[roff[p] + t] = 1.0 / (double)rr[p];
  if (t < cc[p]) nu[coff[p] + t] = 1.0 / (double)cc[p];
}

// Distribution::validate's blocked sum (the oracle's blocked_sum, transport.cpp:96-102)
double host_blocked_sum(const double* x, int64_t n) {
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  double total = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) {
    double v[DET_T];
    for (int t = 0; t < DET_T; ++t) {
      double acc = 0.0;
      for (int j = 0; j < DET_J; ++j) {
        const int64_t idx = c * DET_CHUNK + (int64_t)j * DET_T + t;
        if (idx < n) acc = acc + x[idx];
      }
      v[t] = acc;
    }
    for (int s = DET_T / 2; s > 0; s >>= 1)
      for (int t = 0; t < s; ++t) v[t] = v[t] + v[t + s];
    total = total + v[0];
  }
  return total;
}

int host_validate_distribution(gs_ctx* ctx, const std::vector<double>& w) {
  if (w.empty()) return gs_fail(ctx, ERRC_LENGTH_MISMATCH, "empty distribution");
  for (double x : w)
    if (!std::isfinite(x)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "non-finite weights");
  for (double x : w)
    if (!(x >= 0.0)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "negative weights");
  if (!(std::fabs(host_blocked_sum(w.data(), (int64_t)w.size()) - 1.0) <= 1e-12))
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "distribution must sum to 1");
  return GS_OK;
}

// Shapes (host) -> device offsets and buffers.
int dense_setup(gs_ctx* ctx, DensePairs& D, const std::vector<int>& hr, const std::vector<int>& hc) {
  cudaStream_t s = ctx->stream;
  const int P = (int)hr.size();
  D.P = P;
  std::vector<long long> ko(P), ro(P), co(P);
  for (int p = 0; p < P; ++p) {
    ko[p] = D.total_rc;
    ro[p] = D.total_r;
    co[p] = D.total_c;
    D.total_rc += (long long)hr[p] * hc[p];
    D.total_r += hr[p];
    D.total_c += hc[p];
    D.max_r = std::max(D.max_r, hr[p]);
    D.max_c = std::max(D.max_c, hc[p]);
  }
  GS_CUDA(ctx, D.r.alloc(P, s));
  GS_CUDA(ctx, D.c.alloc(P, s));
  GS_CUDA(ctx, D.koff.alloc(P, s));
  GS_CUDA(ctx, D.roff.alloc(P, s));
  GS_CUDA(ctx, D.coff.alloc(P, s));
  GS_CUDA(ctx, cudaMemcpyAsync(D.r.get(), hr.data(), P * sizeof(int), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemcpyAsync(D.c.get(), hc.data(), P * sizeof(int), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemcpyAsync(D.koff.get(), ko.data(), P * sizeof(long long), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemcpyAsync(D.roff.get(), ro.data(), P * sizeof(long long), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemcpyAsync(D.coff.get(), co.data(), P * sizeof(long long), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, D.C.alloc(D.total_rc, s));
  GS_CUDA(ctx, D.K.alloc(D.total_rc, s));
  GS_CUDA(ctx, D.Kt.alloc(D.total_rc, s));
  GS_CUDA(ctx, D.mu.alloc(D.total_r, s));
  GS_CUDA(ctx, D.v.alloc(D.total_r, s));
  GS_CUDA(ctx, D.phi.alloc(D.total_r, s));
  GS_CUDA(ctx, D.e.alloc(D.total_r, s));
  GS_CUDA(ctx, D.t.alloc(D.total_r, s));
  GS_CUDA(ctx, D.nu.alloc(D.total_c, s));
  GS_CUDA(ctx, D.w.alloc(D.total_c, s));
  GS_CUDA(ctx, D.active.alloc(P + 1, s));  // [P]: number of active pairs
  GS_CUDA(ctx, D.iters.alloc(P, s));
  GS_CUDA(ctx, D.conv.alloc(P, s));
  GS_CUDA(ctx, D.bad.alloc(P, s));
  GS_CUDA(ctx, D.err.alloc(P, s));
  GS_CUDA(ctx, D.cost.alloc(P, s));
  GS_CUDA(ctx, D.kl.alloc(P, s));
  GS_CUDA(ctx, cudaMemsetAsync(D.bad.get(), 0, P * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(D.iters.get(), 0, P * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(D.conv.get(), 0, P * sizeof(int), s));
  std::vector<int> act(P + 1, 1);
  act[P] = P;
  GS_CUDA(ctx, cudaMemcpyAsync(D.active.get(), act.data(), (P + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
  std::vector<double> inf(P, INFINITY);
  GS_CUDA(ctx, cudaMemcpyAsync(D.err.get(), inf.data(), P * sizeof(double), cudaMemcpyHostToDevice, s));
  return GS_OK;
}

inline dim3 grid2(long long work, int P) {
  return dim3((unsigned)((work + kT - 1) / kT > 0 ? (work + kT - 1) / kT : 1), (unsigned)P);
}

// K from C, underflow checks, then the Sinkhorn loop and the final cost / kl. `fail_pair`: the
// first pair whose kernel underflows (or whose cost has non-finite entries), -1 otherwise.
int dense_run(gs_ctx* ctx, DensePairs& D, double lambda, int max_iter, double tol, int* fail_pair) {
  cudaStream_t s = ctx->stream;
  const int P = D.P;
  if (fail_pair) *fail_pair = -1;
  DevBuf<int> nonfinite;
  GS_CUDA(ctx, nonfinite.alloc(P, s));
  GS_CUDA(ctx, cudaMemsetAsync(nonfinite.get(), 0, P * sizeof(int), s));
  const long long max_rc = (long long)D.max_r * D.max_c;
  gs_launch_begin(ctx, 1);
  k_dense_kernel<<<grid2(max_rc, P), kT, 0, s>>>(D.C.get(), D.koff.get(), D.r.get(), D.c.get(), lambda,
                                                  D.K.get(), D.Kt.get(), nonfinite.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_dense_underflow<<<grid2(std::max(D.max_r, D.max_c), P), kT, 0, s>>>(D.K.get(), D.Kt.get(), D.koff.get(),
                                                                         D.r.get(), D.c.get(), D.bad.get());
  gs_launch_end(ctx, 1);
  std::vector<int> hbad(P), hnf(P);
  GS_CUDA(ctx, cudaMemcpyAsync(hbad.data(), D.bad.get(), P * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(hnf.data(), nonfinite.get(), P * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  for (int p = 0; p < P; ++p) {  // pairs run in order in the reference: the first failure throws
    if (hnf[p]) {
      if (fail_pair) *fail_pair = p;
      return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "cost matrix has non-finite entries");
    }
    if (hbad[p] & 1) {
      if (fail_pair) *fail_pair = p;
      return gs_fail(ctx, ERRC_NUMERICAL_UNDERFLOW, "kernel row underflowed to zero; increase lambda");
    }
    if (hbad[p] & 2) {
      if (fail_pair) *fail_pair = p;
      return gs_fail(ctx, ERRC_NUMERICAL_UNDERFLOW, "kernel column underflowed to zero; increase lambda");
    }
  }
  const dim3 gr = grid2(D.max_r, P), gc = grid2(D.max_c, P), gb = grid2(std::max(D.max_r, D.max_c), P);
  gs_launch_begin(ctx, 1);
  k_dense_init<<<gb, kT, 0, s>>>(D.roff.get(), D.coff.get(), D.r.get(), D.c.get(), D.v.get(), D.w.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);  // phi = K w (transport.cpp:295)
  k_dense_rows<<<gr, kT, 0, s>>>(D.Kt.get(), D.koff.get(), D.roff.get(), D.coff.get(), D.r.get(), D.c.get(),
                                 nullptr, D.w.get(), nullptr, nullptr, D.phi.get(), nullptr);
  gs_launch_end(ctx, 1);
  int* d_nact = D.active.get() + P;
  int h_nact = P;
  const int poll = 16;
  for (int it = 1; it <= max_iter && h_nact > 0; ++it) {
    gs_launch_begin(ctx, 0);
    k_dense_v<<<gr, kT, 0, s>>>(D.roff.get(), D.r.get(), D.active.get(), D.mu.get(), D.phi.get(), D.v.get());
    gs_launch_end(ctx, 0);
    gs_launch_begin(ctx, 0);
    k_dense_cols<<<gc, kT, 0, s>>>(D.K.get(), D.koff.get(), D.roff.get(), D.coff.get(), D.r.get(), D.c.get(),
                                   D.active.get(), D.v.get(), D.nu.get(), D.w.get());
    gs_launch_end(ctx, 0);
    gs_launch_begin(ctx, 0);
    k_dense_rows<<<gr, kT, 0, s>>>(D.Kt.get(), D.koff.get(), D.roff.get(), D.coff.get(), D.r.get(), D.c.get(),
                                   D.active.get(), D.w.get(), D.v.get(), D.mu.get(), D.phi.get(), D.e.get());
    gs_launch_end(ctx, 0);
    gs_launch_begin(ctx, 1);
    k_dense_ctl<<<(P + kT - 1) / kT, kT, 0, s>>>(D.roff.get(), D.r.get(), P, it, tol, D.e.get(), D.active.get(),
                                                 D.iters.get(), D.conv.get(), D.err.get(), d_nact);
    gs_launch_end(ctx, 1);
    if (it % poll == 0) {
      GS_CUDA(ctx, cudaMemcpyAsync(&h_nact, d_nact, sizeof(int), cudaMemcpyDeviceToHost, s));
      GS_CUDA(ctx, cudaStreamSynchronize(s));
    }
  }
  gs_launch_begin(ctx, 1);
  k_dense_cost_rows<<<gr, kT, 0, s>>>(D.K.get(), D.C.get(), D.koff.get(), D.roff.get(), D.coff.get(), D.r.get(),
                                      D.c.get(), D.w.get(), D.t.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_dense_final<<<(P + kT - 1) / kT, kT, 0, s>>>(D.roff.get(), D.coff.get(), D.r.get(), D.c.get(), P, D.v.get(),
                                                 D.w.get(), D.t.get(), D.mu.get(), D.nu.get(), D.cost.get(),
                                                 D.kl.get());
  gs_launch_end(ctx, 1);
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

}  // namespace

// transport.cpp:271-311
extern "C" int gs_dense_sinkhorn(gs_ctx* ctx, const double* C, int r, int c, const double* mu,
                                 const double* nu, double lambda, int max_iter, double tol, int mem,
                                 double* out_v, double* out_w, double* out_cost, double* out_kl,
                                 int* out_iters, int* out_conv, double* out_err) {
  if (r < 0 || c < 0) return gs_fail(ctx, ERRC_LENGTH_MISMATCH, "cost matrix shape does not match the marginals");
  cudaStream_t s = ctx->stream;
  std::vector<double> hmu(r), hnu(c);
  if (mem == GS_MEM_HOST) {
    if (r) memcpy(hmu.data(), mu, (size_t)r * sizeof(double));
    if (c) memcpy(hnu.data(), nu, (size_t)c * sizeof(double));
  } else {
    GS_CUDA(ctx, cudaMemcpy(hmu.data(), mu, (size_t)r * sizeof(double), cudaMemcpyDeviceToHost));
    GS_CUDA(ctx, cudaMemcpy(hnu.data(), nu, (size_t)c * sizeof(double), cudaMemcpyDeviceToHost));
  }
  GS_TRY(host_validate_distribution(ctx, hmu));
  GS_TRY(host_validate_distribution(ctx, hnu));
  if (!(lambda > 0.0)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "lambda must be positive");
  if (!(tol > 0.0 && max_iter >= 1)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "bad Sinkhorn parameters");
  DensePairs D;
  GS_TRY(dense_setup(ctx, D, std::vector<int>{r}, std::vector<int>{c}));
  GS_TRY(gs_copy_in(ctx, D.C.get(), C, (size_t)r * c * sizeof(double), mem));
  GS_CUDA(ctx, cudaMemcpyAsync(D.mu.get(), hmu.data(), r * sizeof(double), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemcpyAsync(D.nu.get(), hnu.data(), c * sizeof(double), cudaMemcpyHostToDevice, s));
  GS_TRY(dense_run(ctx, D, lambda, max_iter, tol, nullptr));
  GS_TRY(gs_copy_out(ctx, out_v, D.v.get(), (size_t)r * sizeof(double), mem));
  GS_TRY(gs_copy_out(ctx, out_w, D.w.get(), (size_t)c * sizeof(double), mem));
  GS_TRY(gs_copy_out(ctx, out_cost, D.cost.get(), sizeof(double), mem));
  GS_TRY(gs_copy_out(ctx, out_kl, D.kl.get(), sizeof(double), mem));
  GS_TRY(gs_copy_out(ctx, out_iters, D.iters.get(), sizeof(int), mem));
  GS_TRY(gs_copy_out(ctx, out_conv, D.conv.get(), sizeof(int), mem));
  GS_TRY(gs_copy_out(ctx, out_err, D.err.get(), sizeof(double), mem));
  return gs_ctx_synchronize(ctx);
}

// bench.cpp:311-331: dense baselines over pairs of point groups (uniform marginals)
extern "C" int gs_dense_sinkhorn_groups(gs_ctx* ctx, const double* X, int n, int d, const int* group_idx,
                                        const int* group_off, int ngroups, const int* pair_a,
                                        const int* pair_b, int P, int squared, double lambda, int max_iter,
                                        double tol, double* out_cost, double* out_kl, int* out_iters,
                                        int* out_conv, double* out_err, int* fail_pair) {
  if (fail_pair) *fail_pair = -1;
  if (P <= 0) return GS_OK;
  if (n < 0 || d < 1 || ngroups < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "bad point groups");
  if (!(lambda > 0.0)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "lambda must be positive");
  if (!(tol > 0.0 && max_iter >= 1)) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "bad Sinkhorn parameters");
  cudaStream_t s = ctx->stream;
  std::vector<int> hr(P), hc(P);
  for (int p = 0; p < P; ++p) {
    const int a = pair_a[p], b = pair_b[p];
    if (a < 0 || a >= ngroups || b < 0 || b >= ngroups)
      return gs_fail(ctx, ERRC_INDEX_OUT_OF_RANGE, "pair refers to a missing group");
    hr[p] = group_off[a + 1] - group_off[a];
    hc[p] = group_off[b + 1] - group_off[b];
    if (hr[p] < 1 || hc[p] < 1) return gs_fail(ctx, ERRC_LENGTH_MISMATCH, "empty distribution");
  }
  for (int q = 0; q < group_off[ngroups]; ++q)
    if (group_idx[q] < 0 || group_idx[q] >= n) return gs_fail(ctx, ERRC_INDEX_OUT_OF_RANGE, "group index out of range");
  DensePairs D;
  GS_TRY(dense_setup(ctx, D, hr, hc));
  DevBuf<double> dX;
  DevBuf<int> dgi, dgo, dpa, dpb;
  GS_CUDA(ctx, dX.alloc((size_t)n * d, s));
  GS_CUDA(ctx, dgi.alloc(group_off[ngroups], s));
  GS_CUDA(ctx, dgo.alloc(ngroups + 1, s));
  GS_CUDA(ctx, dpa.alloc(P, s));
  GS_CUDA(ctx, dpb.alloc(P, s));
  GS_CUDA(ctx, cudaMemcpyAsync(dX.get(), X, (size_t)n * d * sizeof(double), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemcpyAsync(dgi.get(), group_idx, group_off[ngroups] * sizeof(int), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemcpyAsync(dgo.get(), group_off, (ngroups + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemcpyAsync(dpa.get(), pair_a, P * sizeof(int), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemcpyAsync(dpb.get(), pair_b, P * sizeof(int), cudaMemcpyHostToDevice, s));
  const long long max_rc = (long long)D.max_r * D.max_c;
  gs_launch_begin(ctx, 1);
  k_dense_cost_groups<<<grid2(max_rc, P), kT, 0, s>>>(dX.get(), d, dgi.get(), dgo.get(), dpa.get(), dpb.get(),
                                                       D.koff.get(), D.r.get(), D.c.get(), squared, D.C.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_dense_uniform<<<grid2(std::max(D.max_r, D.max_c), P), kT, 0, s>>>(D.roff.get(), D.coff.get(), D.r.get(),
                                                                       D.c.get(), D.mu.get(), D.nu.get());
  gs_launch_end(ctx, 1);
  GS_TRY(dense_run(ctx, D, lambda, max_iter, tol, fail_pair));
  GS_CUDA(ctx, cudaMemcpyAsync(out_cost, D.cost.get(), P * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(out_kl, D.kl.get(), P * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(out_iters, D.iters.get(), P * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(out_conv, D.conv.get(), P * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(out_err, D.err.get(), P * sizeof(double), cudaMemcpyDeviceToHost, s));
  return gs_ctx_synchronize(ctx);
}
