// gs_euler.cu -- EulerHeat on the device (proj/src/heat.cpp:133-219): the
// implicit-Euler competitor of the Chebyshev filter. The system I + (t/steps) L is built on the
// device, renumbered by Cuthill-McKee (entries keep their column order, so every product row is
// the reference's fma chain), and each of the `steps` solves is the reference's lockstep conjugate
// gradient over the whole batch (Solver::lockstep_cg; the reference's automatic mode factorises
// with Eigen's LDLT below n = 4000, which has no device counterpart here).
//
// Per-column sums use the blocked order of the oracle (go_detdot over the ORIGINAL vertex order;
// Eigen's colwise().sum() order is unpinned) and the updates x + p*alpha,
// r - ap*alpha, r + p*beta are unfused, so device and oracle agree bit for bit.
#include <cub/cub.cuh>

#include <cmath>
#include <memory>
#include <algorithm>
#include <string>
#include <vector>

#include "gs_internal.cuh"
#include "geosink_b200.h"

struct gs_euler {
  int n = 0, steps = 1;
  double t = 0.0;
  gs_graph* system = nullptr;  // caller's vertex order
  gs_graph* perm = nullptr;    // Cuthill-McKee order
  int* order = nullptr;        // order[new] = old
  int* newpos = nullptr;       // newpos[old] = new
  // direct branch (heat.cpp:157-162: Solver::direct, or automatic with n <= 4000): the inverse
  // Cholesky factor Y = L^-1 of the system in the CM order (n x n row-major, lower triangle);
  // a solve is x <- Y^T (Y x)
  bool direct = false;
  double* Y = nullptr;
};

namespace {

constexpr int kT = 256;
inline unsigned blocks_for(int64_t work) { return (unsigned)((work + kT - 1) / kT); }

// ---- system I + h L (heat.cpp:139-153, then from_triplets mirrors the upper triangle) --------------
__device__ __forceinline__ bool euler_entry(const int* offs, const int* cols, const double* vals, int i,
                                            int p, double h, int* j_out, double* v_out) {
  const int j = cols[p];
  // the reference scales the upper triangle and mirrors it; L is symmetric bit for bit, so the
  // lower entries equal h * L(i, j) computed from their own row
  double v = h * vals[p];
  if (j == i) v = v + 1.0;
  *j_out = j;
  *v_out = v;
  return v != 0.0;  // from_triplets drops explicit zeros (sparse.cpp:25)
}

__global__ void k_euler_count(const int* __restrict__ offs, const int* __restrict__ cols,
                              const double* __restrict__ vals, int n, double h, int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  bool diag = false;
  for (int p = offs[i]; p < offs[i + 1]; ++p) {
    int j;
    double v;
    if (cols[p] == i) diag = true;
    if (euler_entry(offs, cols, vals, i, p, h, &j, &v)) ++c;
  }
  cnt[i] = c + (diag ? 0 : 1);  // a missing diagonal becomes 1 (heat.cpp:152)
}

__global__ void k_euler_fill(const int* __restrict__ offs, const int* __restrict__ cols,
                             const double* __restrict__ vals, int n, double h, const int* __restrict__ out_offs,
                             int* __restrict__ out_cols, double* __restrict__ out_vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int q = out_offs[i];
  bool diag = false;
  for (int p = offs[i]; p < offs[i + 1]; ++p) {
    if (!diag && cols[p] > i) {  // no diagonal in this (column-sorted) row: insert the unit one
      out_cols[q] = i;
      out_vals[q] = 1.0;
      ++q;
      diag = true;
    }
    if (cols[p] == i) diag = true;
    int j;
    double v;
    if (euler_entry(offs, cols, vals, i, p, h, &j, &v)) {
      out_cols[q] = j;
      out_vals[q] = v;
      ++q;
    }
  }
  if (!diag) {
    out_cols[q] = i;
    out_vals[q] = 1.0;
  }
}

// ---- blocked column sums in the original vertex order (go_detdot restated per column) ----------
// grouped layout: column col of vertex i lives at ((col / GW) * n + newpos[i]) * GW + col % GW
__global__ void k_colsum_partial(const double* __restrict__ x, const double* __restrict__ y, int n, int GW,
                                 const int* __restrict__ newpos, double* __restrict__ part, int B) {
  const int col = blockIdx.y;
  const int64_t c = blockIdx.x;
  const size_t gb = (size_t)(col / GW) * n;
  const int cc = col % GW;
  double acc = 0.0;
  for (int j = 0; j < DET_J; ++j) {
    const int64_t i = c * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
    if (i < n) {
      const size_t e = (gb + newpos[i]) * GW + cc;
      acc = fma(x[e], y[e], acc);
    }
  }
  __shared__ double sh[DET_T];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = DET_T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(size_t)col * gridDim.x + c] = sh[0];
}

__global__ void k_colsum_fold(const double* __restrict__ part, int64_t nchunks, double* __restrict__ out) {
  const int col = blockIdx.x;
  __shared__ double sh[DET_T];
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < nchunks; q += DET_T) acc = acc + part[(size_t)col * nchunks + q];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = DET_T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[col] = nchunks ? sh[0] : 0.0;
}

// ---- CG vector updates (heat.cpp:176-199), grouped layout, column = (e / GW) / n * GW + e % GW ----
__device__ __forceinline__ int col_of(int64_t e, int n, int GW) {
  return (int)((e / GW) / n) * GW + (int)(e % GW);
}

__global__ void k_cg_start(const double* __restrict__ b, const double* __restrict__ ap, int64_t len,
                           double* __restrict__ r, double* __restrict__ p) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    const double v = b[e] - ap[e];
    r[e] = v;
    p[e] = v;
  }
}

__global__ void k_cg_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                        const double* __restrict__ ap, const double* __restrict__ alpha, int64_t len, int n,
                        int GW) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
    const double a = alpha[col_of(e, n, GW)];
    x[e] = x[e] + p[e] * a;
    r[e] = r[e] - ap[e] * a;
  }
}

__global__ void k_cg_p(double* __restrict__ p, const double* __restrict__ r, const double* __restrict__ beta,
                       int64_t len, int n, int GW) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x)
    p[e] = r[e] + p[e] * beta[col_of(e, n, GW)];
}

// alpha = pap > 0 ? rs / pap : 0
__global__ void k_cg_alpha(const double* __restrict__ rs, const double* __restrict__ pap, int B,
                           double* __restrict__ alpha) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < B) alpha[c] = pap[c] > 0.0 ? rs[c] / pap[c] : 0.0;
}

// beta = rs > 0 ? rs_new / rs : 0; rs = rs_new; *busy = any column with rs > tol2 * |b|^2
__global__ void k_cg_beta(double* __restrict__ rs, const double* __restrict__ rs_new,
                          const double* __restrict__ bn, int B, double tol2, double* __restrict__ beta,
                          int* __restrict__ busy) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  beta[c] = rs[c] > 0.0 ? rs_new[c] / rs[c] : 0.0;
  rs[c] = rs_new[c];
  if (rs_new[c] > tol2 * bn[c]) atomicOr(busy, 1);
}

__global__ void k_cg_init_norms(const double* __restrict__ rs, double* __restrict__ bn, int B, double tol2,
                                int* __restrict__ busy) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  bn[c] = fmax(bn[c], 1e-300);
  if (rs[c] > tol2 * bn[c]) atomicOr(busy, 1);
}

__global__ void k_pack_cols(const double* __restrict__ src, double* __restrict__ dst, int n, int B, int GW,
                            int G, const int* __restrict__ order) {
  const int64_t total = (int64_t)G * n * GW;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % GW);
    const int64_t r = e / GW;
    const int i = (int)(r % n);
    const int col = (int)(r / n) * GW + c;
    dst[e] = col < B ? src[(size_t)col * n + order[i]] : 0.0;
  }
}

__global__ void k_unpack_cols(const double* __restrict__ src, double* __restrict__ dst, int n, int B, int GW,
                              const int* __restrict__ newpos) {
  const int64_t total = (int64_t)B * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(e / n), i = (int)(e % n);
    dst[e] = src[((size_t)(col / GW) * n + newpos[i]) * GW + col % GW];
  }
}

unsigned grid_for(int64_t work) {
  int64_t b = (work + kT - 1) / kT;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

struct Col {  // per-column device scalars, padded to the grouped width (padding stays 0)
  DevBuf<double> v;
  int alloc(gs_ctx* ctx, int Bpad) {
    GS_CUDA(ctx, v.alloc(Bpad, ctx->stream));
    GS_CUDA(ctx, cudaMemsetAsync(v.get(), 0, Bpad * sizeof(double), ctx->stream));
    return GS_OK;
  }
};

int colsum(gs_ctx* ctx, const gs_euler* E, const double* x, const double* y, int B, int GW,
           DevBuf<double>& part, double* out) {
  const int n = E->n;
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  cudaStream_t s = ctx->stream;
  if (nchunks > 0) {
    gs_launch_begin(ctx, 1);
    k_colsum_partial<<<dim3((unsigned)nchunks, B), DET_T, 0, s>>>(x, y, n, GW, E->newpos, part.get(), B);
    gs_launch_end(ctx, 1);
  }
  gs_launch_begin(ctx, 1);
  k_colsum_fold<<<B, DET_T, 0, s>>>(part.get(), nchunks, out);
  gs_launch_end(ctx, 1);
  return GS_OK;
}

// ---- direct branch: dense Cholesky of I + hL (n <= 4096), its inverse factor, triangular products
constexpr int kNb = 32;  // Cholesky block

__global__ void k_dense_fill(const int* __restrict__ offs, const int* __restrict__ cols,
                             const double* __restrict__ vals, int n, double* __restrict__ A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int p = offs[i]; p < offs[i + 1]; ++p) A[(size_t)i * n + cols[p]] = vals[p];
}

// factor the b x b diagonal block at k0 in place (lower triangle); fail on a non-positive pivot
__global__ void k_chol_diag(double* A, int n, int k0, int b, int* fail) {
  __shared__ double blk[kNb][kNb + 1];
  const int t = threadIdx.x;  // row within the block
  for (int c = 0; c < b; ++c) blk[t][c] = t < b ? A[(size_t)(k0 + t) * n + k0 + c] : 0.0;
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    if (t == 0) {
      const double d = blk[j][j];
      if (!(d > 0.0)) *fail = 1;
      blk[j][j] = sqrt(d > 0.0 ? d : 1.0);
    }
    __syncthreads();
    if (t > j && t < b) blk[t][j] = blk[t][j] / blk[j][j];
    __syncthreads();
    if (t > j && t < b)
      for (int c = j + 1; c <= t; ++c) blk[t][c] = blk[t][c] - blk[t][j] * blk[c][j];
    __syncthreads();
  }
  if (t < b)
    for (int c = 0; c <= t; ++c) A[(size_t)(k0 + t) * n + k0 + c] = blk[t][c];
}

// panel below the diagonal block: L21 = A21 L11^-T (one thread per row, forward substitution)
__global__ void k_chol_panel(double* A, int n, int k0, int b) {
  __shared__ double L11[kNb][kNb + 1];
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) L11[e / b][e % b] = A[(size_t)(k0 + e / b) * n + k0 + e % b];
  __syncthreads();
  const int i = k0 + b + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x[kNb];
  for (int j = 0; j < b; ++j) {
    double v = A[(size_t)i * n + k0 + j];
    for (int q = 0; q < j; ++q) v = v - x[q] * L11[j][q];
    x[j] = v / L11[j][j];
  }
  for (int j = 0; j < b; ++j) A[(size_t)i * n + k0 + j] = x[j];
}

// trailing update of the lower triangle: A22 -= L21 L21^T (32 x 32 tiles)
__global__ void k_chol_update(double* A, int n, int k0, int b) {
  const int r0 = k0 + b + blockIdx.y * kNb, c0 = k0 + b + blockIdx.x * kNb;
  if (c0 > r0 + kNb - 1) return;  // strictly upper tile
  __shared__ double Li[kNb][kNb + 1], Lc[kNb][kNb + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < kNb; r += 8) {
    Li[r][tx] = (r0 + r < n && tx < b) ? A[(size_t)(r0 + r) * n + k0 + tx] : 0.0;
    Lc[r][tx] = (c0 + r < n && tx < b) ? A[(size_t)(c0 + r) * n + k0 + tx] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < kNb; r += 8) {
    const int i = r0 + r, c = c0 + tx;
    if (i >= n || c >= n || c > i) continue;
    double acc = 0.0;
    for (int q = 0; q < b; ++q) acc = fma(Li[r][q], Lc[tx][q], acc);
    A[(size_t)i * n + c] -= acc;
  }
}

// Y = L^-1 (lower): thread j solves column j; the warp's threads walk the same rows so the L rows
// are broadcast loads; Y is zero above the diagonal, so the sums start at the warp's first column
__global__ void k_tri_inverse(const double* __restrict__ L, int n, double* __restrict__ Y) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int j0 = blockIdx.x * blockDim.x;
  for (int i = j0; i < n; ++i) {
    double sacc = 0.0;
    for (int p = j0; p < i; ++p) sacc = fma(L[(size_t)i * n + p], j < n ? Y[(size_t)p * n + j] : 0.0, sacc);
    if (j < n) Y[(size_t)i * n + j] = i < j ? 0.0 : ((i == j ? 1.0 : 0.0) - sacc) / L[(size_t)i * n + i];
    __syncwarp();
  }
}

// out = op(Y) x on the grouped block (B columns in groups of GW): op = Y (lower) or Y^T
template <bool TRANS>
__global__ void k_tri_apply(const double* __restrict__ Y, int n, const double* __restrict__ x, double* __restrict__ out,
                            int GW, int G) {
  __shared__ double Ys[kNb][kNb + 1];
  __shared__ double Xs[kNb][64];
  const int g = blockIdx.y;
  const int r0 = blockIdx.x * kNb;
  const int tx = threadIdx.x, ty = threadIdx.y;  // GW-wide column lanes x 8 row lanes
  double acc[kNb / 8];
#pragma unroll
  for (int u = 0; u < kNb / 8; ++u) acc[u] = 0.0;
  const int pb = TRANS ? r0 : 0, pe = TRANS ? n : min(n, r0 + kNb);
  for (int p0 = pb - pb % kNb; p0 < pe; p0 += kNb) {
    __syncthreads();
    for (int e = ty * blockDim.x + tx; e < kNb * kNb; e += blockDim.x * blockDim.y) {
      const int a = e / kNb, c = e % kNb;  // Ys[row i - r0][p - p0]
      const int i = r0 + a, pp = p0 + c;
      double v = 0.0;
      if (i < n && pp < n) v = TRANS ? (pp >= i ? Y[(size_t)pp * n + i] : 0.0) : (pp <= i ? Y[(size_t)i * n + pp] : 0.0);
      Ys[a][c] = v;
    }
    for (int e = ty * blockDim.x + tx; e < kNb * GW; e += blockDim.x * blockDim.y) {
      const int pp = p0 + e / GW, c = e % GW;
      Xs[e / GW][c] = pp < n ? x[((size_t)g * n + pp) * GW + c] : 0.0;
    }
    __syncthreads();
    if (tx < GW)
#pragma unroll
      for (int u = 0; u < kNb / 8; ++u) {
        const int a = ty + 8 * u;
        double sacc = acc[u];
        for (int c = 0; c < kNb; ++c) sacc = fma(Ys[a][c], Xs[c][tx], sacc);
        acc[u] = sacc;
      }
  }
  if (tx < GW)
#pragma unroll
    for (int u = 0; u < kNb / 8; ++u) {
      const int i = r0 + ty + 8 * u;
      if (i < n) out[((size_t)g * n + i) * GW + tx] = acc[u];
    }
}

int euler_factor(gs_ctx* ctx, gs_euler* E) {
  const int n = E->n;
  cudaStream_t s = ctx->stream;
  DevBuf<double> A;
  DevBuf<int> fail;
  GS_CUDA(ctx, A.alloc((size_t)n * n, s));
  GS_CUDA(ctx, fail.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(A.get(), 0, (size_t)n * n * sizeof(double), s));
  GS_CUDA(ctx, cudaMemsetAsync(fail.get(), 0, sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_dense_fill<<<blocks_for(n), kT, 0, s>>>(E->perm->offs, E->perm->cols, E->perm->vals, n, A.get());
  gs_launch_end(ctx, 1);
  for (int k0 = 0; k0 < n; k0 += kNb) {
    const int b = std::min(kNb, n - k0);
    gs_launch_begin(ctx, 1);
    k_chol_diag<<<1, kNb, 0, s>>>(A.get(), n, k0, b, fail.get());
    gs_launch_end(ctx, 1);
    const int rest = n - k0 - b;
    if (rest > 0) {
      gs_launch_begin(ctx, 1);
      k_chol_panel<<<(rest + 127) / 128, 128, 0, s>>>(A.get(), n, k0, b);
      gs_launch_end(ctx, 1);
      const int tiles = (rest + kNb - 1) / kNb;
      gs_launch_begin(ctx, 1);
      k_chol_update<<<dim3(tiles, tiles), dim3(32, 8), 0, s>>>(A.get(), n, k0, b);
      gs_launch_end(ctx, 1);
    }
  }
  int hf = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&hf, fail.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (hf) return gs_fail(ctx, ERRC_SOLVE_FAILURE, "sparse LDLT factorisation failed");
  GS_CUDA(ctx, cudaMalloc((void**)&E->Y, (size_t)n * n * sizeof(double)));
  gs_launch_begin(ctx, 1);
  k_tri_inverse<<<(n + 31) / 32, 32, 0, s>>>(A.get(), n, E->Y);
  gs_launch_end(ctx, 1);
  GS_CUDA(ctx, cudaGetLastError());
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// one solve (I + hL) x = b on the grouped block: x <- Y^T (Y x)
int euler_direct_solve(gs_ctx* ctx, const gs_euler* E, double* x, int B) {
  const int n = E->n;
  const int GW = gs_group_width(B), G = (B + GW - 1) / GW;
  cudaStream_t s = ctx->stream;
  DevBuf<double> z;
  GS_CUDA(ctx, z.alloc((size_t)G * GW * n, s));
  const dim3 grid((n + kNb - 1) / kNb, G), blk(GW < 32 ? 32 : GW, 8);
  gs_launch_begin(ctx, 1);
  k_tri_apply<false><<<grid, blk, 0, s>>>(E->Y, n, x, z.get(), GW, G);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_tri_apply<true><<<grid, blk, 0, s>>>(E->Y, n, z.get(), x, GW, G);
  gs_launch_end(ctx, 1);
  GS_CUDA(ctx, cudaGetLastError());
  return GS_OK;
}

// heat.cpp:166-201 on the grouped block x (B columns); *iters = CG iterations
int euler_solve(gs_ctx* ctx, const gs_euler* E, double* x, int B, int* iters) {
  if (E->direct) {  // heat.cpp:167-173
    if (iters) *iters = 0;
    return euler_direct_solve(ctx, E, x, B);
  }
  const int n = E->n;
  const int GW = gs_group_width(B), G = (B + GW - 1) / GW;
  const int64_t len = (int64_t)G * GW * n;
  cudaStream_t s = ctx->stream;
  DevBuf<double> b, r, p, ap, part;
  Col rs, rn, bn, pap, alpha, beta;
  GS_CUDA(ctx, b.alloc(len, s));
  GS_CUDA(ctx, r.alloc(len, s));
  GS_CUDA(ctx, p.alloc(len, s));
  GS_CUDA(ctx, ap.alloc(len, s));
  GS_CUDA(ctx, part.alloc((size_t)B * ((n + DET_CHUNK - 1) / DET_CHUNK + 1), s));
  for (Col* c : {&rs, &rn, &bn, &pap, &alpha, &beta}) GS_TRY(c->alloc(ctx, G * GW));
  DevBuf<int> busy;
  GS_CUDA(ctx, busy.alloc(1, s));
  GS_CUDA(ctx, cudaMemcpyAsync(b.get(), x, len * sizeof(double), cudaMemcpyDeviceToDevice, s));
  GS_TRY(gs_spmm_grouped(ctx, E->perm, x, ap.get(), B));
  gs_launch_begin(ctx, 1);
  k_cg_start<<<grid_for(len), kT, 0, s>>>(b.get(), ap.get(), len, r.get(), p.get());
  gs_launch_end(ctx, 1);
  GS_TRY(colsum(ctx, E, r.get(), r.get(), B, GW, part, rs.v.get()));
  GS_TRY(colsum(ctx, E, b.get(), b.get(), B, GW, part, bn.v.get()));
  const double tol2 = 1e-10 * 1e-10;
  const long max_iter = 10L * n;
  GS_CUDA(ctx, cudaMemsetAsync(busy.get(), 0, sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_cg_init_norms<<<(B + kT - 1) / kT, kT, 0, s>>>(rs.v.get(), bn.v.get(), B, tol2, busy.get());
  gs_launch_end(ctx, 1);
  long it = 0;
  for (;;) {
    int h_busy = 0;
    GS_CUDA(ctx, cudaMemcpyAsync(&h_busy, busy.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    if (!h_busy) break;
    if (!(it < max_iter)) return gs_fail(ctx, ERRC_SOLVE_FAILURE, "conjugate gradient exceeded 10 n iterations");
    ++it;
    GS_TRY(gs_spmm_grouped(ctx, E->perm, p.get(), ap.get(), B));
    GS_TRY(colsum(ctx, E, p.get(), ap.get(), B, GW, part, pap.v.get()));
    gs_launch_begin(ctx, 1);
    k_cg_alpha<<<(B + kT - 1) / kT, kT, 0, s>>>(rs.v.get(), pap.v.get(), B, alpha.v.get());
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_cg_xr<<<grid_for(len), kT, 0, s>>>(x, r.get(), p.get(), ap.get(), alpha.v.get(), len, n, GW);
    gs_launch_end(ctx, 1);
    GS_TRY(colsum(ctx, E, r.get(), r.get(), B, GW, part, rn.v.get()));
    GS_CUDA(ctx, cudaMemsetAsync(busy.get(), 0, sizeof(int), s));
    gs_launch_begin(ctx, 1);
    k_cg_beta<<<(B + kT - 1) / kT, kT, 0, s>>>(rs.v.get(), rn.v.get(), bn.v.get(), B, tol2, beta.v.get(),
                                               busy.get());
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_cg_p<<<grid_for(len), kT, 0, s>>>(p.get(), r.get(), beta.v.get(), len, n, GW);
    gs_launch_end(ctx, 1);
  }
  if (iters) *iters = (int)it;
  return GS_OK;
}

// ---- euler_sinkhorn[_batch] (transport.cpp:144-239 over EulerHeat, transport.cpp:257-269) ------
// Per-pair vectors are column-major (pair p at p * n, caller's vertex order). The lockstep CG runs
// until every column of its batch converges, so the batch must hold exactly the reference's
// active pairs in order: finished pairs are dropped after every sweep (transport.cpp:210-226).
__global__ void k_es_weighted(const double* __restrict__ a, const double* __restrict__ src,
                              const int* __restrict__ cols, int n, int B, double* __restrict__ out) {
  const int64_t total = (int64_t)B * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n), i = (int)(e % n);
    out[e] = a[i] * (src ? src[(size_t)cols[c] * n + i] : 1.0);
  }
}

// filter_checked (transport.cpp:21-38): min of the output vs 1e-12 max |input|, per column
__global__ void k_es_check(const double* __restrict__ x, const double* __restrict__ y, int n,
                           int* __restrict__ bad) {
  const int c = blockIdx.x;
  __shared__ double smn[kT], smx[kT];
  double mn = INFINITY, mx = 0.0;
  for (int i = threadIdx.x; i < n; i += kT) {
    mn = fmin(mn, y[(size_t)c * n + i]);
    mx = fmax(mx, fabs(x[(size_t)c * n + i]));
  }
  smn[threadIdx.x] = mn;
  smx[threadIdx.x] = mx;
  __syncthreads();
  for (int s = kT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      smn[threadIdx.x] = fmin(smn[threadIdx.x], smn[threadIdx.x + s]);
      smx[threadIdx.x] = fmax(smx[threadIdx.x], smx[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && !(smn[0] >= -(1e-12 * smx[0]))) atomicExch(bad, 1);
}

// dst[pair] = num[pair] / max(den_c, floor) for the active pairs (den: batch column c)
__global__ void k_es_divide(const double* __restrict__ num, const double* __restrict__ den,
                            const int* __restrict__ cols, int n, int B, double* __restrict__ dst) {
  const int64_t total = (int64_t)B * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n), i = (int)(e % n);
    const size_t o = (size_t)cols[c] * n + i;
    dst[o] = num[o] / fmax(den[e], 1e-300);
  }
}

// marginal L1 error per active pair, summed in vertex order as the oracle does
__global__ void k_es_err(const double* __restrict__ V, const double* __restrict__ phi,
                         const double* __restrict__ M, const int* __restrict__ cols, int n, int B,
                         double* __restrict__ err) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  const size_t o = (size_t)cols[c] * n;
  double e = 0.0;
  for (int i = 0; i < n; ++i) e += fabs(V[o + i] * phi[(size_t)c * n + i] - M[o + i]);
  err[c] = e;
}

// transport.cpp:41-54 (host, the oracle's order and libm)
double plain_log_sum(const double* a, const double* mu, const double* s, int n) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i)
    if (mu[i] > 0.0) acc += a[i] * mu[i] * std::log(s[i]);
  return acc;
}

}  // namespace

extern "C" int gs_euler_create_ex(gs_ctx* ctx, const gs_graph* L, double t, int steps, int solver,
                                  gs_euler** out);

// the reference's default (Solver::automatic): direct below n = 4000, lockstep CG above
extern "C" int gs_euler_create(gs_ctx* ctx, const gs_graph* L, double t, int steps, gs_euler** out) {
  return gs_euler_create_ex(ctx, L, t, steps, GS_EULER_AUTOMATIC, out);
}

extern "C" int gs_euler_create_ex(gs_ctx* ctx, const gs_graph* L, double t, int steps, int solver,
                                  gs_euler** out) {
  if (!ctx || !L || !out) return GS_ERR_UNSUPPORTED;
  *out = nullptr;
  if (!(t > 0.0 && std::isfinite(t))) return gs_fail(ctx, ERRC_NON_POSITIVE_TIME, "diffusion time must be > 0");
  if (steps < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "substep count must be >= 1");
  cudaStream_t s = ctx->stream;
  std::unique_ptr<gs_euler> E(new gs_euler());
  const int n = L->n;
  E->n = n;
  E->t = t;
  E->steps = steps;
  const double h = t / steps;
  DevBuf<int> cnt;
  GS_CUDA(ctx, cnt.alloc((size_t)n + 1, s));
  GS_CUDA(ctx, cudaMemsetAsync(cnt.get(), 0, ((size_t)n + 1) * sizeof(int), s));
  if (n > 0) {
    gs_launch_begin(ctx, 1);
    k_euler_count<<<blocks_for(n), kT, 0, s>>>(L->offs, L->cols, L->vals, n, h, cnt.get());
    gs_launch_end(ctx, 1);
  }
  DevBuf<int> offs;
  GS_CUDA(ctx, offs.alloc((size_t)n + 1, s));
  size_t tb = 0;
  GS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), offs.get(), n + 1, s));
  DevBuf<unsigned char> tmp;
  GS_CUDA(ctx, tmp.alloc(tb, s));
  GS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt.get(), offs.get(), n + 1, s));
  int nnz = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&nnz, offs.get() + n, sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  GS_TRY(gs_graph_alloc(ctx, n, nnz, &E->system));
  GS_CUDA(ctx, cudaMemcpyAsync(E->system->offs, offs.get(), ((size_t)n + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s));
  if (n > 0) {
    gs_launch_begin(ctx, 1);
    k_euler_fill<<<blocks_for(n), kT, 0, s>>>(L->offs, L->cols, L->vals, n, h, offs.get(), E->system->cols,
                                              E->system->vals);
    gs_launch_end(ctx, 1);
  }
  GS_CUDA(ctx, cudaMalloc((void**)&E->order, ((size_t)n + 1) * sizeof(int)));
  GS_CUDA(ctx, cudaMalloc((void**)&E->newpos, ((size_t)n + 1) * sizeof(int)));
  GS_TRY(gs_bfs_order(ctx, E->system, E->order, E->newpos, 1, nullptr, nullptr));
  GS_TRY(gs_permute_graph(ctx, E->system, E->order, E->newpos, &E->perm));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (solver < GS_EULER_AUTOMATIC || solver > GS_EULER_LOCKSTEP_CG)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "unknown solver");
  E->direct = solver == GS_EULER_DIRECT || (solver == GS_EULER_AUTOMATIC && n <= 4000);
  if (E->direct && n > 0) {
    if (n > 16384) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "direct solver: n <= 16384 on the device");
    GS_TRY(euler_factor(ctx, E.get()));
  }
  *out = E.release();
  return GS_OK;
}

extern "C" void gs_euler_destroy(gs_euler* E) {
  if (!E) return;
  gs_graph_destroy(E->system);
  gs_graph_destroy(E->perm);
  cudaFree(E->order);
  cudaFree(E->newpos);
  cudaFree(E->Y);
  delete E;
}

extern "C" const gs_graph* gs_euler_system(const gs_euler* E) { return E ? E->system : nullptr; }

// EulerHeat::apply on device column blocks (width contiguous n-vectors, caller's vertex order)
static int euler_apply_dev(gs_ctx* ctx, const gs_euler* E, const double* dX, double* dY, int width, int* it) {
  const int n = E->n;
  cudaStream_t s = ctx->stream;
  const int GW = gs_group_width(width), G = (width + GW - 1) / GW;
  const int64_t len = (int64_t)G * GW * n;
  DevBuf<double> blk;
  GS_CUDA(ctx, blk.alloc(len, s));
  gs_launch_begin(ctx, 1);
  k_pack_cols<<<grid_for(len), kT, 0, s>>>(dX, blk.get(), n, width, GW, G, E->order);
  gs_launch_end(ctx, 1);
  for (int step = 0; step < E->steps; ++step) GS_TRY(euler_solve(ctx, E, blk.get(), width, it));
  gs_launch_begin(ctx, 1);
  k_unpack_cols<<<grid_for((int64_t)width * n), kT, 0, s>>>(blk.get(), dY, n, width, GW, E->newpos);
  gs_launch_end(ctx, 1);
  return GS_OK;
}

extern "C" int gs_euler_apply(gs_ctx* ctx, const gs_euler* E, const double* X, double* Y, int width,
                              int mem, int* iters_out) {
  if (!ctx || !E) return GS_ERR_UNSUPPORTED;
  if (iters_out) *iters_out = 0;
  if (width < 0) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "width");
  const int n = E->n;
  if (width == 0 || n == 0) return GS_OK;
  cudaStream_t s = ctx->stream;
  DevBuf<double> xin, yout, blk;
  const double* dX = X;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, xin.alloc((size_t)width * n, s));
    GS_CUDA(ctx, cudaMemcpyAsync(xin.get(), X, (size_t)width * n * sizeof(double), cudaMemcpyHostToDevice, s));
    dX = xin.get();
  }
  double* dY = Y;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, yout.alloc((size_t)width * n, s));
    dY = yout.get();
  }
  const int GW = gs_group_width(width), G = (width + GW - 1) / GW;
  const int64_t len = (int64_t)G * GW * n;
  GS_CUDA(ctx, blk.alloc(len, s));
  gs_launch_begin(ctx, 1);
  k_pack_cols<<<grid_for(len), kT, 0, s>>>(dX, blk.get(), n, width, GW, G, E->order);
  gs_launch_end(ctx, 1);
  int it = 0;
  for (int step = 0; step < E->steps; ++step) GS_TRY(euler_solve(ctx, E, blk.get(), width, &it));
  gs_launch_begin(ctx, 1);
  k_unpack_cols<<<grid_for((int64_t)width * n), kT, 0, s>>>(blk.get(), dY, n, width, GW, E->newpos);
  gs_launch_end(ctx, 1);
  if (mem != GS_MEM_DEVICE)
    GS_CUDA(ctx, cudaMemcpyAsync(Y, dY, (size_t)width * n * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (iters_out) *iters_out = it;
  return GS_OK;
}

extern "C" int gs_euler_sinkhorn(gs_ctx* ctx, const gs_euler* E, const double* a, const double* mus,
                                 const double* nus, int P, int max_iter, double tol, int flags, int mem,
                                 double* out_v, double* out_w, double* out_cost, double* out_kl,
                                 int* out_iters, int* out_conv, double* out_err, int* fail_pair,
                                 int* fail_sweep) {
  if (!ctx || !E) return GS_ERR_UNSUPPORTED;
  if (fail_pair) *fail_pair = -1;
  if (fail_sweep) *fail_sweep = 0;
  const int n = E->n;
  if (P < 0) return gs_fail(ctx, ERRC_SIZE_MISMATCH, "pair lists differ in length");
  if (P == 0) return GS_OK;
  cudaStream_t s = ctx->stream;
  const size_t len = (size_t)P * n;
  DevBuf<double> bmu, bnu, ba;
  const double *dM = mus, *dN = nus, *da = a;
  auto stage = [&](DevBuf<double>& b, const double* src, size_t count, const double** out) -> int {
    GS_CUDA(ctx, b.alloc(count, s));
    GS_CUDA(ctx, cudaMemcpyAsync(b.get(), src, count * sizeof(double), cudaMemcpyHostToDevice, s));
    *out = b.get();
    return GS_OK;
  };
  if (mem != GS_MEM_DEVICE) {
    GS_TRY(stage(bmu, mus, len, &dM));
    GS_TRY(stage(bnu, nus, len, &dN));
    GS_TRY(stage(ba, a, n, &da));
  }
  GS_TRY(gs_check_transport_inputs(ctx, n, dM, dN, da, P, max_iter, tol));
  DevBuf<double> V, W, X, phi, psi, OV, OW, derr;
  DevBuf<int> cols, bad;
  for (DevBuf<double>* b : {&V, &W, &X, &phi, &psi, &OV, &OW}) GS_CUDA(ctx, b->alloc(len, s));
  GS_CUDA(ctx, derr.alloc(P, s));
  GS_CUDA(ctx, cols.alloc(P, s));
  GS_CUDA(ctx, bad.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(V.get(), 0, len * sizeof(double), s));
  std::vector<int> active(P), stagnant(P, 0), iters(P, 0), conv(P, 0);
  std::vector<double> errs(P, INFINITY);
  for (int p = 0; p < P; ++p) active[p] = p;
  const char* knp = "heat approximation produced negative mass; increase the degree or diffusion time";
  // X = a .* src[active] (src null: W = 1); out = E(X) checked
  auto apply = [&](const double* src, int B, double* out) -> int {
    gs_launch_begin(ctx, 1);
    k_es_weighted<<<grid_for((int64_t)B * n), kT, 0, s>>>(da, src, cols.get(), n, B, X.get());
    gs_launch_end(ctx, 1);
    int it = 0;
    GS_TRY(euler_apply_dev(ctx, E, X.get(), out, B, &it));
    GS_CUDA(ctx, cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    gs_launch_begin(ctx, 1);
    k_es_check<<<B, kT, 0, s>>>(X.get(), out, n, bad.get());
    gs_launch_end(ctx, 1);
    int h = 0;
    GS_CUDA(ctx, cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    return h ? gs_fail(ctx, ERRC_KERNEL_NOT_POSITIVE, knp) : GS_OK;
  };
  GS_CUDA(ctx, cudaMemcpyAsync(cols.get(), active.data(), P * sizeof(int), cudaMemcpyHostToDevice, s));
  GS_TRY(apply(nullptr, P, phi.get()));  // phi = H(a * 1)
  int na = P;
  for (int it = 1; it <= max_iter && na > 0; ++it) {
    const int B = na;
    gs_launch_begin(ctx, 1);
    k_es_divide<<<grid_for((int64_t)B * n), kT, 0, s>>>(dM, phi.get(), cols.get(), n, B, V.get());
    gs_launch_end(ctx, 1);
    GS_TRY(apply(V.get(), B, psi.get()));
    gs_launch_begin(ctx, 1);
    k_es_divide<<<grid_for((int64_t)B * n), kT, 0, s>>>(dN, psi.get(), cols.get(), n, B, W.get());
    gs_launch_end(ctx, 1);
    GS_TRY(apply(W.get(), B, phi.get()));
    gs_launch_begin(ctx, 1);
    k_es_err<<<(B + kT - 1) / kT, kT, 0, s>>>(V.get(), phi.get(), dM, cols.get(), n, B, derr.get());
    gs_launch_end(ctx, 1);
    std::vector<double> e(B);
    GS_CUDA(ctx, cudaMemcpyAsync(e.data(), derr.get(), B * sizeof(double), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    std::vector<int> keep;
    for (int c = 0; c < B; ++c) {
      const int pair = active[c];
      iters[pair] = it;
      errs[pair] = e[c];
      const bool done = e[c] <= tol;
      if (done) conv[pair] = 1;
      if (done || it == max_iter) {  // transport.cpp:196-200: finalise v, w
        GS_CUDA(ctx, cudaMemcpyAsync(OV.get() + (size_t)pair * n, V.get() + (size_t)pair * n, n * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
        GS_CUDA(ctx, cudaMemcpyAsync(OW.get() + (size_t)pair * n, W.get() + (size_t)pair * n, n * sizeof(double),
                                     cudaMemcpyDeviceToDevice, s));
      }
      if (!done) {
        stagnant[pair] = e[c] > 0.5 ? stagnant[pair] + 1 : 0;
        if (!(flags & GS_FLAG_NO_STAGNATION_ABORT) && !(stagnant[pair] < 50)) {
          if (fail_pair) *fail_pair = pair;
          if (fail_sweep) *fail_sweep = it;
          if (flags & GS_FLAG_SINGLE)
            return gs_fail(ctx, ERRC_DISCONNECTED,
                           "marginal error stagnated above 0.5; are mu and nu in the same graph component?");
          return gs_fail(ctx, ERRC_DISCONNECTED, "marginal error stagnated above 0.5 for pair " + std::to_string(pair));
        }
        keep.push_back(c);
      }
    }
    if ((int)keep.size() != B) {  // compaction (transport.cpp:210-226): phi keeps its batch order
      for (int c = 0; c < (int)keep.size(); ++c)
        if (keep[c] != c)
          GS_CUDA(ctx, cudaMemcpyAsync(phi.get() + (size_t)c * n, phi.get() + (size_t)keep[c] * n, n * sizeof(double),
                                       cudaMemcpyDeviceToDevice, s));
      std::vector<int> still;
      for (int c : keep) still.push_back(active[c]);
      active = still;
      na = (int)active.size();
      if (na > 0)
        GS_CUDA(ctx, cudaMemcpyAsync(cols.get(), active.data(), na * sizeof(int), cudaMemcpyHostToDevice, s));
    }
  }
  // ---- outputs; cost / KL on the host in the oracle's order (transport.cpp:137-140) ----------------
  std::vector<double> hv(len), hw(len), hmu(len), hnu(len), ha(n);
  GS_CUDA(ctx, cudaMemcpyAsync(hv.data(), OV.get(), len * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(hw.data(), OW.get(), len * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(hmu.data(), dM, len * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(hnu.data(), dN, len * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(ha.data(), da, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  const double lambda = 4.0 * E->t;
  std::vector<double> cost(P), kl(P);
  for (int p = 0; p < P; ++p) {
    const double *mu = &hmu[(size_t)p * n], *nu = &hnu[(size_t)p * n];
    const double *v = &hv[(size_t)p * n], *w = &hw[(size_t)p * n];
    cost[p] = lambda * (plain_log_sum(ha.data(), mu, v, n) + plain_log_sum(ha.data(), nu, w, n));
    double k1 = 0.0, k2 = 0.0;
    for (int i = 0; i < n; ++i)
      if (mu[i] > 0.0) k1 += mu[i] * std::log(v[i]);
    for (int i = 0; i < n; ++i)
      if (nu[i] > 0.0) k2 += nu[i] * std::log(std::fmax(ha[i] * w[i], 1e-300));
    kl[p] = k1 + k2 - 1.0;
  }
  auto put = [&](void* dst, const void* src, size_t bytes, bool host_src) -> int {
    if (!dst) return GS_OK;
    cudaMemcpyKind k = mem == GS_MEM_DEVICE ? (host_src ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice)
                                            : (host_src ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost);
    GS_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, k, s));
    return GS_OK;
  };
  GS_TRY(put(out_v, OV.get(), len * sizeof(double), false));
  GS_TRY(put(out_w, OW.get(), len * sizeof(double), false));
  GS_TRY(put(out_cost, cost.data(), P * sizeof(double), true));
  GS_TRY(put(out_kl, kl.data(), P * sizeof(double), true));
  GS_TRY(put(out_iters, iters.data(), P * sizeof(int), true));
  GS_TRY(put(out_conv, conv.data(), P * sizeof(int), true));
  GS_TRY(put(out_err, errs.data(), P * sizeof(double), true));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}
