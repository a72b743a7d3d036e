// gs_graph.cu -- operator construction on the device:
//   select_knn / knn_alpha_decay_graph   proj/src/graph.cpp:30-108
//   laplacian                            proj/src/graph.cpp:110-165
//   estimate_lambda_max                  proj/src/graph.cpp:167-194
//   heat_chebyshev_coefficients          proj/src/heat.cpp:14-70
//
// kNN: exact brute force, one thread per query, candidate tiles staged in shared memory,
// d^2 = max(0, (|xi|^2 + |xj|^2) - 2<xi,xj>) with fma chains in dimension order (the oracle's
// formula, so selections agree bit for bit), register top-k kept sorted by (d^2, index); the
// candidate scan is in increasing index order, so a tie never displaces the lower index.
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>

#include "gs_internal.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kKnnThreads = 128;
constexpr int kKnnTile = 128;
#ifndef GS_KNN_IL
#define GS_KNN_IL 4  // candidates whose inner products run as interleaved fma chains
#endif

__device__ __forceinline__ double row_sqnorm(const double* p, int d) {
  double s = 0.0;
  for (int q = 0; q < d; ++q) s = fma(p[q], p[q], s);
  return s;
}

__device__ __forceinline__ double exact_d2(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int q = 0; q < d; ++q) {
    const double diff = a[q] - b[q];
    s = fma(diff, diff, s);
  }
  return s;
}

__global__ void k_sqnorms(const double* __restrict__ pts, int n, int d, double* __restrict__ sq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) sq[i] = row_sqnorm(pts + (size_t)i * d, d);
}

__global__ void k_check_finite(const double* __restrict__ x, int64_t m, int* bad) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[e])) atomicExch(bad, 1);
}

template <int KMAX, int DMAX>
__global__ void __launch_bounds__(kKnnThreads) k_knn(const double* __restrict__ pts,
                                                     const double* __restrict__ sq, int n, int d,
                                                     int k, int* __restrict__ nbrs,
                                                     double* __restrict__ eps,
                                                     const int* __restrict__ qlist = nullptr, int nq = 0) {
  extern __shared__ double smem[];
  double* s_x = smem;                    // kKnnTile * d
  double* s_sq = smem + kKnnTile * d;    // kKnnTile
  // queries: all n rows, or the nq rows of qlist (the tensor-core path's fallback, gs_knn_tc.cu)
  const int qslot = blockIdx.x * kKnnThreads + threadIdx.x;
  const int qi = qlist ? (qslot < nq ? qlist[qslot] : n) : qslot;
  const bool valid = qi < n;
  double xq[DMAX];
#pragma unroll
  for (int q = 0; q < DMAX; ++q) xq[q] = (valid && q < d) ? pts[(size_t)qi * d + q] : 0.0;
  const double sqq = valid ? sq[qi] : 0.0;
  double bd[KMAX];
  int bi[KMAX];
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    bd[s] = INFINITY;
    bi[s] = 0x7fffffff;
  }
  for (int base = 0; base < n; base += kKnnTile) {
    const int cnt = min(kKnnTile, n - base);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * d; e += kKnnThreads) s_x[e] = pts[(size_t)base * d + e];
    for (int e = threadIdx.x; e < cnt; e += kKnnThreads) s_sq[e] = sq[base + e];
    __syncthreads();
    if (!valid) continue;
    // four candidates' inner products as independent fma chains (each in dimension order, as
    // the oracle's), then the selection in ascending candidate order
    constexpr int IL = GS_KNN_IL;
    for (int j0 = 0; j0 < cnt; j0 += IL) {
      double gg[IL];
#pragma unroll
      for (int u = 0; u < IL; ++u) gg[u] = 0.0;
#pragma unroll
      for (int q = 0; q < DMAX; ++q)
        if (q < d)
#pragma unroll
          for (int u = 0; u < IL; ++u)
            if (j0 + u < cnt) gg[u] = fma(xq[q], s_x[(j0 + u) * d + q], gg[u]);
#pragma unroll
      for (int u = 0; u < IL; ++u) {
      const int jj = j0 + u;
      if (jj >= cnt) break;
      const int j = base + jj;
      double d2 = (sqq + s_sq[jj]) - 2.0 * gg[u];
      if (!(d2 > 0.0)) d2 = 0.0;
      if (j == qi) continue;
      // current worst kept candidate is slot k-1
      double worst = bd[0];
#pragma unroll
      for (int s = 0; s < KMAX; ++s)
        if (s == k - 1) worst = bd[s];
      if (!(d2 < worst)) continue;
#pragma unroll
      for (int s = KMAX - 1; s > 0; --s) {
        if (s < k) {
          if (bd[s - 1] > d2) {
            bd[s] = bd[s - 1];
            bi[s] = bi[s - 1];
          } else if (bd[s] > d2) {
            bd[s] = d2;
            bi[s] = j;
          }
        }
      }
      if (bd[0] > d2) {
        bd[0] = d2;
        bi[0] = j;
      }
      }
    }
  }
  if (!valid) return;
  int last = 0;
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    if (s < k) nbrs[(size_t)qi * k + s] = bi[s];
    if (s == k - 1) last = bi[s];
  }
  double xl[DMAX];
#pragma unroll
  for (int q = 0; q < DMAX; ++q) xl[q] = q < d ? pts[(size_t)last * d + q] : 0.0;
  double s2 = 0.0;
#pragma unroll
  for (int q = 0; q < DMAX; ++q)
    if (q < d) {
      const double diff = xq[q] - xl[q];
      s2 = fma(diff, diff, s2);
    }
  eps[qi] = sqrt(s2);
}

template <int KMAX>
void launch_knn_k(const double* pts, const double* sq, int n, int d, int k, int* nb, double* eps,
                  cudaStream_t s, const int* qlist = nullptr, int nq = 0) {
  const size_t shm = (size_t)kKnnTile * (d + 1) * sizeof(double);
  const int rows = qlist ? nq : n;
  const unsigned grid = (unsigned)((rows + kKnnThreads - 1) / kKnnThreads);
  if (rows == 0) return;
  if (d <= 4) {
    k_knn<KMAX, 4><<<grid, kKnnThreads, shm, s>>>(pts, sq, n, d, k, nb, eps, qlist, nq);
  } else if (d <= 8) {
    k_knn<KMAX, 8><<<grid, kKnnThreads, shm, s>>>(pts, sq, n, d, k, nb, eps, qlist, nq);
  } else {
    cudaFuncSetAttribute(k_knn<KMAX, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
    k_knn<KMAX, 32><<<grid, kKnnThreads, shm, s>>>(pts, sq, n, d, k, nb, eps, qlist, nq);
  }
}

// ---- exact kNN on a uniform grid for low-dimensional clouds (d <= 3) --------------------------
// Same distance arithmetic as k_knn and the same (d2, index) order -- candidates are compared
// lexicographically, so the visiting order does not matter and the result equals the brute-force
// selection bit for bit (select_knn, graph.cpp:30-71). Cells are visited in cube shells of growing
// Chebyshev radius R around the query's cell; the search stops once the k-th candidate is closer
// than R cell widths (with a rounding slack for the Gram-form distance), or the grid is exhausted.
struct Grid {
  double lo[3], inv_h, h;
  int dim[3];
  int d;
};

__device__ __forceinline__ int grid_coord(const Grid& G, double x, int q) {
  int c = (int)floor((x - G.lo[q]) * G.inv_h);
  return c < 0 ? 0 : (c >= G.dim[q] ? G.dim[q] - 1 : c);
}

__device__ __forceinline__ long long grid_cell(const Grid& G, const double* x) {
  long long id = 0;
  for (int q = G.d - 1; q >= 0; --q) id = id * G.dim[q] + grid_coord(G, x[q], q);
  return id;
}

__global__ void k_grid_count(const double* __restrict__ pts, int n, Grid G, int* __restrict__ cell,
                             int* __restrict__ counts) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = (int)grid_cell(G, pts + (size_t)i * G.d);
  cell[i] = c;
  atomicAdd(counts + c, 1);
}

__global__ void k_grid_fill(const int* __restrict__ cell, int n, int* __restrict__ cursor,
                            int* __restrict__ items) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) items[atomicAdd(cursor + cell[i], 1)] = i;
}

template <int KMAX>
__global__ void __launch_bounds__(128) k_knn_grid(const double* __restrict__ pts,
                                                  const double* __restrict__ sq, int n, Grid G,
                                                  const int* __restrict__ start,
                                                  const int* __restrict__ items, double max_sq, int k,
                                                  int* __restrict__ nbrs, double* __restrict__ eps) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int qi = items[t];  // queries in cell order: neighbouring threads search the same cells
  const int d = G.d;
  double xq[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < d; ++q) xq[q] = pts[(size_t)qi * d + q];
  const double sqq = sq[qi];
  int cq[3] = {0, 0, 0};
  for (int q = 0; q < d; ++q) cq[q] = grid_coord(G, xq[q], q);
  double bd[KMAX];
  int bi[KMAX];
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    bd[s] = INFINITY;
    bi[s] = 0x7fffffff;
  }
  // Gram-form d2 differs from the exact squared distance by a few ulps of |xq|^2 + |xj|^2
  const double slack = 1e-9 * (sqq + max_sq) + 1e-300;
  const int rmax = max(G.dim[0], max(d > 1 ? G.dim[1] : 1, d > 2 ? G.dim[2] : 1));
  for (int R = 0; R <= rmax; ++R) {
    const int lo0 = cq[0] - R, hi0 = cq[0] + R;
    const int lo1 = d > 1 ? cq[1] - R : 0, hi1 = d > 1 ? cq[1] + R : 0;
    const int lo2 = d > 2 ? cq[2] - R : 0, hi2 = d > 2 ? cq[2] + R : 0;
    for (int c2 = lo2; c2 <= hi2; ++c2) {
      if (d > 2 && (c2 < 0 || c2 >= G.dim[2])) continue;
      for (int c1 = lo1; c1 <= hi1; ++c1) {
        if (d > 1 && (c1 < 0 || c1 >= G.dim[1])) continue;
        const bool inner12 = (d < 3 || (c2 > lo2 && c2 < hi2)) && (d < 2 || (c1 > lo1 && c1 < hi1));
        // on the shell: interior (c1, c2) rows only contribute their two end cells
        for (int c0 = lo0; c0 <= hi0; c0 += (inner12 && R > 0) ? (hi0 - lo0) : 1) {
          if (c0 < 0 || c0 >= G.dim[0]) {
            if (inner12 && R > 0 && c0 == hi0) break;
            continue;
          }
          const long long cell = ((long long)c2 * (d > 1 ? G.dim[1] : 1) + c1) * G.dim[0] + c0;
          for (int e = start[cell]; e < start[cell + 1]; ++e) {
            const int j = items[e];
            if (j == qi) continue;
            const double* xj = pts + (size_t)j * d;
            double g = 0.0;
            for (int q = 0; q < d; ++q) g = fma(xq[q], xj[q], g);
            double d2 = (sqq + sq[j]) - 2.0 * g;
            if (!(d2 > 0.0)) d2 = 0.0;
            double wd = bd[0];
            int wi = bi[0];
#pragma unroll
            for (int s = 0; s < KMAX; ++s)
              if (s == k - 1) {
                wd = bd[s];
                wi = bi[s];
              }
            if (!(d2 < wd || (d2 == wd && j < wi))) continue;
#pragma unroll
            for (int s = KMAX - 1; s > 0; --s) {
              if (s < k) {
                if (bd[s - 1] > d2 || (bd[s - 1] == d2 && bi[s - 1] > j)) {
                  bd[s] = bd[s - 1];
                  bi[s] = bi[s - 1];
                } else if (bd[s] > d2 || (bd[s] == d2 && bi[s] > j)) {
                  bd[s] = d2;
                  bi[s] = j;
                }
              }
            }
            if (bd[0] > d2 || (bd[0] == d2 && bi[0] > j)) {
              bd[0] = d2;
              bi[0] = j;
            }
          }
          if (inner12 && R > 0 && c0 == hi0) break;
        }
      }
    }
    // every point outside the searched cube is at least R cell widths away
    double wd = bd[0];
#pragma unroll
    for (int s = 0; s < KMAX; ++s)
      if (s == k - 1) wd = bd[s];
    const double reach = (double)R * G.h;
    if (wd + slack < reach * reach) break;
  }
  int last = 0;
#pragma unroll
  for (int s = 0; s < KMAX; ++s) {
    if (s < k) nbrs[(size_t)qi * k + s] = bi[s];
    if (s == k - 1) last = bi[s];
  }
  double s2 = 0.0;
  for (int q = 0; q < d; ++q) {
    const double diff = xq[q] - pts[(size_t)last * d + q];
    s2 = fma(diff, diff, s2);
  }
  eps[qi] = sqrt(s2);
}

__global__ void k_bbox(const double* __restrict__ pts, int n, int d, double* __restrict__ out /* 2*d */) {
  __shared__ double smin[3][256], smax[3][256];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int q = 0; q < d; ++q) {
      mn[q] = fmin(mn[q], pts[(size_t)i * d + q]);
      mx[q] = fmax(mx[q], pts[(size_t)i * d + q]);
    }
  for (int q = 0; q < 3; ++q) {
    smin[q][threadIdx.x] = mn[q];
    smax[q][threadIdx.x] = mx[q];
  }
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int q = 0; q < 3; ++q) {
        smin[q][threadIdx.x] = fmin(smin[q][threadIdx.x], smin[q][threadIdx.x + s]);
        smax[q][threadIdx.x] = fmax(smax[q][threadIdx.x], smax[q][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < d; ++q) {
      out[2 * (blockIdx.x * 3 + q)] = smin[q][0];
      out[2 * (blockIdx.x * 3 + q) + 1] = smax[q][0];
    }
}

__global__ void k_eps_check(const double* eps, int n, int* first_bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && !(eps[i] > 0.0)) atomicMin(first_bad, i);
}

__global__ void k_pair_keys(const int* __restrict__ nb, int n, int k,
                            unsigned long long* __restrict__ keys) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * k) return;
  const int i = (int)(e / k);
  const int j = nb[e];
  const unsigned lo = (unsigned)min(i, j), hi = (unsigned)max(i, j);
  keys[e] = ((unsigned long long)lo << 32) | hi;
}

// graph.cpp:99-106 (alpha decay) / Gaussian-median extension; both triangles emitted, zero
// weights (from_triplets drops explicit zeros, sparse.cpp:25) get the sentinel key.
__global__ void k_pair_weights(const unsigned long long* __restrict__ ukeys, int64_t u,
                               const double* __restrict__ pts, int d,
                               const double* __restrict__ eps, int kernel, double param,
                               double sigma2, unsigned long long* __restrict__ keys,
                               double* __restrict__ vals) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= u) return;
  const unsigned long long key = ukeys[e];
  const int i = (int)(key >> 32), j = (int)(key & 0xFFFFFFFFull);
  const double d2 = exact_d2(pts + (size_t)i * d, pts + (size_t)j * d, d);
  double w;
  if (kernel == GS_KERNEL_ALPHA_DECAY) {
    const double dist = sqrt(d2);
    w = 0.5 * (exp(-pow(dist / eps[i], param)) + exp(-pow(dist / eps[j], param)));
  } else {
    w = exp(-(d2 / sigma2));
  }
  const bool keep = w != 0.0;
  keys[2 * e] = keep ? key : ~0ull;
  keys[2 * e + 1] = keep ? (((unsigned long long)(unsigned)j << 32) | (unsigned)i) : ~0ull;
  vals[2 * e] = w;
  vals[2 * e + 1] = w;
}

__global__ void k_count_sentinel(const unsigned long long* keys, int64_t m, int* cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < m && keys[e] == ~0ull) atomicAdd(cnt, 1);
}

// ---- Laplacian (graph.cpp:110-165) -----------------------------------------------------------
__global__ void k_degree(int n, const int* __restrict__ offs, const double* __restrict__ vals,
                         double* __restrict__ degree, int* negative) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double dg = 0.0;
  for (int p = offs[i]; p < offs[i + 1]; ++p) {
    if (!(vals[p] >= 0.0)) atomicExch(negative, 1);
    dg += vals[p];
  }
  degree[i] = dg;
}

__device__ __forceinline__ double lap_diag(int kind, int i, double degree_i, const int* offs,
                                           const int* cols, const double* vals,
                                           const double* inv) {
  double diag = kind == GS_LAPLACIAN_COMBINATORIAL ? degree_i : 1.0;
  for (int p = offs[i]; p < offs[i + 1]; ++p) {
    if (cols[p] == i) {
      if (kind == GS_LAPLACIAN_COMBINATORIAL) diag -= vals[p];
      else diag -= vals[p] * inv[i] * inv[i];
    }
  }
  return diag;
}

__device__ __forceinline__ double lap_off(int kind, int i, int j, double v, const double* inv) {
  if (kind == GS_LAPLACIAN_COMBINATORIAL) return -v;
  // the reference computes the upper entry (row min(i,j)) and mirrors it
  const int lo = min(i, j), hi = max(i, j);
  return -(v * inv[lo] * inv[hi]);
}

__global__ void k_lap_count(int kind, int n, const int* __restrict__ offs, const int* __restrict__ cols,
                            const double* __restrict__ vals, const double* __restrict__ degree,
                            const double* __restrict__ inv, int* __restrict__ count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  for (int p = offs[i]; p < offs[i + 1]; ++p) {
    const int j = cols[p];
    if (j != i && lap_off(kind, i, j, vals[p], inv) != 0.0) ++c;
  }
  if (lap_diag(kind, i, degree[i], offs, cols, vals, inv) != 0.0) ++c;
  count[i] = c;
}

__global__ void k_lap_fill(int kind, int n, const int* __restrict__ offs, const int* __restrict__ cols,
                           const double* __restrict__ vals, const double* __restrict__ degree,
                           const double* __restrict__ inv, const int* __restrict__ loffs,
                           int* __restrict__ lcols, double* __restrict__ lvals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double diag = lap_diag(kind, i, degree[i], offs, cols, vals, inv);
  int o = loffs[i];
  bool placed = diag == 0.0;
  for (int p = offs[i]; p < offs[i + 1]; ++p) {
    const int j = cols[p];
    if (!placed && j >= i) {
      lcols[o] = i;
      lvals[o] = diag;
      ++o;
      placed = true;
    }
    if (j == i) continue;
    const double v = lap_off(kind, i, j, vals[p], inv);
    if (v == 0.0) continue;
    lcols[o] = j;
    lvals[o] = v;
    ++o;
  }
  if (!placed) {
    lcols[o] = i;
    lvals[o] = diag;
  }
}

__global__ void k_inv_sqrt(const double* degree, int n, double* inv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) inv[i] = 1.0 / sqrt(degree[i] > 0.0 ? degree[i] : 1.0);
}

// ---- power iteration (graph.cpp:167-194) with the oracle's blocked reduction order ---------
struct PowerState {
  int it, done, converged, zero;
  double est, norm;
};

// y = L x, one thread per row (CSR-order fma chain, sparse.cpp:70-83); the blocked dot products
// of k_power_spmv then read y, so the product itself is not confined to n / 4096 blocks
__global__ void k_power_rows(int n, const int* __restrict__ offs, const int* __restrict__ cols,
                             const double* __restrict__ vals, const double* __restrict__ x,
                             double* __restrict__ y, const PowerState* st) {
  if (st->done) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int p = offs[i]; p < offs[i + 1]; ++p) acc = fma(vals[p], x[cols[p]], acc);
  y[i] = acc;
}

// per 4096-row chunk: the blocked partial sums of y.y and x.y (lane t folds rows
// c*4096 + j*256 + t in j order, then a tree over lanes -- the oracle's go_detdot order)
__global__ void __launch_bounds__(DET_T) k_power_dots(int n, const double* __restrict__ x,
                                                     const double* __restrict__ y, double* part_yy,
                                                     double* part_xy, const PowerState* st) {
  if (st->done) return;
  double ayy = 0.0, axy = 0.0;
  for (int j = 0; j < DET_J; ++j) {
    const int64_t i = (int64_t)blockIdx.x * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
    if (i < n) {
      const double acc = y[i];  // k_power_rows
      ayy = fma(acc, acc, ayy);
      axy = fma(x[i], acc, axy);
    }
  }
  __shared__ double s1[DET_T], s2[DET_T];
  s1[threadIdx.x] = ayy;
  s2[threadIdx.x] = axy;
  __syncthreads();
  for (int s = DET_T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s1[threadIdx.x] = s1[threadIdx.x] + s1[threadIdx.x + s];
      s2[threadIdx.x] = s2[threadIdx.x] + s2[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part_yy[blockIdx.x] = s1[0];
    part_xy[blockIdx.x] = s2[0];
  }
}

__device__ double fold_partials(const double* part, int64_t nparts, double* sh) {
  double acc = 0.0;
  for (int64_t q = threadIdx.x; q < nparts; q += DET_T) acc = acc + part[q];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = DET_T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(DET_T) k_power_update(const double* part_yy, const double* part_xy,
                                                       int64_t nparts, PowerState* st) {
  if (st->done) return;
  __shared__ double sh[DET_T];
  const double yy = fold_partials(part_yy, nparts, sh);
  const double xy = fold_partials(part_xy, nparts, sh);
  if (threadIdx.x != 0) return;
  const double norm = sqrt(yy);
  if (norm <= 1e-300) {
    st->zero = 1;
    st->done = 1;
    st->it += 1;
    return;
  }
  const double r = xy;
  if (st->it > 0 && fabs(r - st->est) <= 1e-6 * fabs(r)) {
    st->est = r;
    st->converged = 1;
    st->done = 1;
    st->it += 1;
    return;
  }
  st->est = r;
  st->norm = norm;
  st->it += 1;
  if (st->it >= 200) st->done = 2;  // fall through to Gershgorin
}

__global__ void k_power_scale(double* __restrict__ x, const double* __restrict__ y, int n,
                              const PowerState* st) {
  if (st->done == 1) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = y[i] / st->norm;
}

__global__ void __launch_bounds__(DET_T) k_det_dot_partial(const double* __restrict__ x,
                                                          const double* __restrict__ y, int n,
                                                          double* part) {
  double acc = 0.0;
  for (int j = 0; j < DET_J; ++j) {
    const int64_t i = (int64_t)blockIdx.x * DET_CHUNK + (int64_t)j * DET_T + threadIdx.x;
    if (i < n) acc = fma(x[i], y[i], acc);
  }
  __shared__ double sh[DET_T];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = DET_T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void __launch_bounds__(DET_T) k_normalize_start(double* x, int n, const double* part,
                                                          int64_t nparts) {
  __shared__ double sh[DET_T];
  __shared__ double s_z;
  const double z = fold_partials(part, nparts, sh);
  if (threadIdx.x == 0) s_z = z;
  __syncthreads();
  if (!(s_z > 0.0)) return;
  const double nr = sqrt(s_z);
  for (int i = threadIdx.x; i < n; i += DET_T) x[i] = x[i] / nr;
}

// ---- Chebyshev coefficients (heat.cpp:14-70), one device thread, oracle-identical rounding --
__device__ void scaled_bessel_dev(double z, int kmax, int start, double* f, double* out) {
  for (int q = 0; q < start + 2; ++q) f[q] = 0.0;
  f[start + 1] = 0.0;
  f[start] = 1e-30;
  for (int j = start; j >= 1; --j) {
    f[j - 1] = f[j + 1] + (2.0 * j / z) * f[j];
    if (fabs(f[j - 1]) > 1e250) {
      const double inv = 1e-250;
      for (int q = j - 1; q < start + 2; ++q) f[q] *= inv;
    }
  }
  double norm = f[0];
  for (int j = 1; j <= start; ++j) norm += 2.0 * f[j];
  for (int k = 0; k <= kmax; ++k) out[k] = (k <= start) ? f[k] / norm : 0.0;
}

__global__ void k_heat_coeffs(double t, int degree, double* f, double* cur, double* refined,
                              double* b) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (t < 1e-300) {
    for (int k = 0; k <= degree; ++k) b[k] = 0.0;
    b[0] = 2.0;
    return;
  }
  int start = degree + (int)ceil(t) + 40 + (int)(2.0 * sqrt((double)degree + t));
  scaled_bessel_dev(t, degree, start, f, cur);
  for (int round = 0; round < 8; ++round) {
    const int next_start = start + start / 2 + 20;
    scaled_bessel_dev(t, degree, next_start, f, refined);
    double worst = 0.0;
    for (int k = 0; k <= degree; ++k) {
      const double scale = fmax(fabs(refined[k]), 1e-280);
      worst = fmax(worst, fabs(refined[k] - cur[k]) / scale);
    }
    double* tmp = cur;
    cur = refined;
    refined = tmp;
    start = next_start;
    if (worst <= 1e-13) break;
  }
  b[0] = 2.0 * cur[0];
  double sign = -1.0;
  for (int k = 1; k <= degree; ++k) {
    b[k] = 2.0 * sign * cur[k];
    sign = -sign;
  }
}

inline unsigned nblk(int64_t m, int t = kThreads) { return (unsigned)((m + t - 1) / t); }

}  // namespace

// =============================================================================================
int gs_coefficients_impl(gs_ctx* ctx, double t, int degree, double* d_out, double* h_out) {
  if (degree < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "Chebyshev degree must be >= 1");
  if (!(t >= 0.0 && std::isfinite(t)))
    return gs_fail(ctx, ERRC_NON_POSITIVE_TIME, "diffusion time must be finite and >= 0");
  cudaStream_t s = ctx->stream;
  int64_t start = degree + (int64_t)std::ceil(t) + 40 + (int64_t)(2.0 * std::sqrt((double)degree + t));
  int64_t maxstart = start;
  for (int r = 0; r < 8; ++r) maxstart = maxstart + maxstart / 2 + 20;
  if (maxstart > (int64_t)1 << 30) return gs_fail(ctx, ERRC_TOO_LARGE, "diffusion time too large");
  DevBuf<double> f, cur, ref, own;
  GS_CUDA(ctx, f.alloc(maxstart + 2, s));
  GS_CUDA(ctx, cur.alloc(degree + 1, s));
  GS_CUDA(ctx, ref.alloc(degree + 1, s));
  double* dst = d_out;
  if (!dst) {
    GS_CUDA(ctx, own.alloc(degree + 1, s));
    dst = own.get();
  }
  gs_launch_begin(ctx, 1);
  k_heat_coeffs<<<1, 1, 0, s>>>(t, degree, f.get(), cur.get(), ref.get(), dst);
  gs_launch_end(ctx, 1);
  if (h_out) GS_CUDA(ctx, cudaMemcpyAsync(h_out, dst, (degree + 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

extern "C" int gs_heat_coefficients(gs_ctx* ctx, double t, int degree, double* out) {
  return gs_coefficients_impl(ctx, t, degree, nullptr, out);
}

int gs_lambda_max_impl(gs_ctx* ctx, const gs_graph* L, double* out, int* rounds_out) {
  const int n = L->n;
  if (rounds_out) *rounds_out = 0;
  if (n == 0) {
    *out = 0.0;
    return GS_OK;
  }
  cudaStream_t s = ctx->stream;
  // start vector: Rng(0x5eed1a4b) normals in vertex order (graph.cpp:171-174), host-generated
  std::vector<double> x0(n);
  {
    gs_rng* r = gs_rng_create(0x5eed1a4bULL);
    for (int i = 0; i < n; ++i) x0[i] = gs_rng_normal(r);
    gs_rng_destroy(r);
  }
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  DevBuf<double> x, y, pyy, pxy;
  DevBuf<PowerState> st;
  GS_CUDA(ctx, x.alloc(n, s));
  GS_CUDA(ctx, y.alloc(n, s));
  GS_CUDA(ctx, pyy.alloc(nchunks, s));
  GS_CUDA(ctx, pxy.alloc(nchunks, s));
  GS_CUDA(ctx, st.alloc(1, s));
  GS_CUDA(ctx, cudaMemcpyAsync(x.get(), x0.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
  GS_CUDA(ctx, cudaMemsetAsync(st.get(), 0, sizeof(PowerState), s));
  gs_launch_begin(ctx, 1);
  k_det_dot_partial<<<(unsigned)nchunks, DET_T, 0, s>>>(x.get(), x.get(), n, pyy.get());
  k_normalize_start<<<1, DET_T, 0, s>>>(x.get(), n, pyy.get(), nchunks);
  gs_launch_end(ctx, 1);
  for (int it = 0; it < 200; ++it) {
    gs_launch_begin(ctx, 1);
    k_power_rows<<<nblk(n), kThreads, 0, s>>>(n, L->offs, L->cols, L->vals, x.get(), y.get(), st.get());
    k_power_dots<<<(unsigned)nchunks, DET_T, 0, s>>>(n, x.get(), y.get(), pyy.get(), pxy.get(), st.get());
    k_power_update<<<1, DET_T, 0, s>>>(pyy.get(), pxy.get(), nchunks, st.get());
    k_power_scale<<<nblk(n), kThreads, 0, s>>>(x.get(), y.get(), n, st.get());
    gs_launch_end(ctx, 1);
    if ((it & 15) == 15) {
      PowerState h;
      GS_CUDA(ctx, cudaMemcpyAsync(&h, st.get(), sizeof h, cudaMemcpyDeviceToHost, s));
      GS_CUDA(ctx, cudaStreamSynchronize(s));
      if (h.done) break;
    }
  }
  PowerState h;
  GS_CUDA(ctx, cudaMemcpyAsync(&h, st.get(), sizeof h, cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h.zero) {
    *out = 0.0;
    if (rounds_out) *rounds_out = h.it;
    return GS_OK;
  }
  if (!h.converged) {
    if (rounds_out) *rounds_out = -1;
    return gs_graph_gershgorin(ctx, L, out);
  }
  if (rounds_out) *rounds_out = h.it;
  *out = 1.01 * h.est;
  return GS_OK;
}

extern "C" int gs_lambda_max(gs_ctx* ctx, const gs_graph* L, double* out, int* rounds_out) {
  return gs_lambda_max_impl(ctx, L, out, rounds_out);
}

extern "C" int gs_laplacian(gs_ctx* ctx, const gs_graph* A, int kind, gs_graph** L_out,
                            double* lambda_bound, int* rounds_out) {
  *L_out = nullptr;
  if (kind != GS_LAPLACIAN_COMBINATORIAL && kind != GS_LAPLACIAN_NORMALIZED)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "unknown laplacian kind");
  const int n = A->n;
  cudaStream_t s = ctx->stream;
  DevBuf<double> degree, inv;
  DevBuf<int> neg, count, loffs;
  GS_CUDA(ctx, degree.alloc(n + 1, s));
  GS_CUDA(ctx, inv.alloc(n + 1, s));
  GS_CUDA(ctx, neg.alloc(1, s));
  GS_CUDA(ctx, count.alloc(n + 1, s));
  GS_CUDA(ctx, cudaMemsetAsync(neg.get(), 0, sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(count.get(), 0, (n + 1) * sizeof(int), s));
  if (n > 0) {
    gs_launch_begin(ctx, 1);
    k_degree<<<nblk(n), kThreads, 0, s>>>(n, A->offs, A->vals, degree.get(), neg.get());
    k_inv_sqrt<<<nblk(n), kThreads, 0, s>>>(degree.get(), n, inv.get());
    k_lap_count<<<nblk(n), kThreads, 0, s>>>(kind, n, A->offs, A->cols, A->vals, degree.get(),
                                              inv.get(), count.get());
    gs_launch_end(ctx, 1);
  }
  int h_neg = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h_neg, neg.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_neg) return gs_fail(ctx, ERRC_NEGATIVE_WEIGHT, "adjacency entries must be non-negative");
  gs_graph* L = nullptr;
  {
    DevBuf<int> offs_tmp;
    GS_CUDA(ctx, offs_tmp.alloc(n + 1, s));
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, count.get(), offs_tmp.get(), n + 1, s);
    DevBuf<unsigned char> tmp;
    GS_CUDA(ctx, tmp.alloc(tb, s));
    cub::DeviceScan::ExclusiveSum(tmp.get(), tb, count.get(), offs_tmp.get(), n + 1, s);
    int nnz = 0;
    GS_CUDA(ctx, cudaMemcpyAsync(&nnz, offs_tmp.get() + n, sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    GS_TRY(gs_graph_alloc(ctx, n, nnz, &L));
    GS_CUDA(ctx, cudaMemcpyAsync(L->offs, offs_tmp.get(), (n + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s));
    if (n > 0) {
      gs_launch_begin(ctx, 1);
      k_lap_fill<<<nblk(n), kThreads, 0, s>>>(kind, n, A->offs, A->cols, A->vals, degree.get(),
                                               inv.get(), L->offs, L->cols, L->vals);
      gs_launch_end(ctx, 1);
    }
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      gs_graph_destroy(L);
      return gs_cuda_fail(ctx, e, "laplacian");
    }
  }
  if (kind == GS_LAPLACIAN_COMBINATORIAL) {
    const int rc = gs_lambda_max_impl(ctx, L, lambda_bound, rounds_out);
    if (rc) {
      gs_graph_destroy(L);
      return rc;
    }
  } else {
    *lambda_bound = 2.0;
    if (rounds_out) *rounds_out = 0;
  }
  *L_out = L;
  return GS_OK;
}

// ---- kNN -----------------------------------------------------------------------------------
// Grid search for d <= 3 (GS_KNN=brute forces the tiled brute force, GS_KNN=grid the grid).
static bool use_grid_knn(int n, int d) {
  const char* e = getenv("GS_KNN");
  if (e && e[0] == 'b') return false;
  if (e && e[0] == 'g') return d <= 3;
  return d <= 3 && n >= 32768;
}

static int knn_grid(gs_ctx* ctx, const double* dpts, const double* sq, int n, int d, int k, int* dnb,
                    double* deps) {
  cudaStream_t s = ctx->stream;
  const int nb = 148 * 4;
  DevBuf<double> part;
  GS_CUDA(ctx, part.alloc((size_t)nb * 6, s));
  gs_launch_begin(ctx, 1);
  k_bbox<<<nb, 256, 0, s>>>(dpts, n, d, part.get());
  gs_launch_end(ctx, 1);
  std::vector<double> hp((size_t)nb * 6);
  GS_CUDA(ctx, cudaMemcpyAsync(hp.data(), part.get(), hp.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  double max_sq = 0.0;
  {
    DevBuf<double> dmax;  // largest squared norm (for the rounding slack)
    GS_CUDA(ctx, dmax.alloc(1, s));
    std::vector<double> hsq(n);
    GS_CUDA(ctx, cudaMemcpyAsync(hsq.data(), sq, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    for (double v : hsq) max_sq = std::max(max_sq, v);
  }
  Grid G{};
  G.d = d;
  double ext[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < d; ++q) {
    double lo = INFINITY, hi = -INFINITY;
    for (int b = 0; b < nb; ++b) {
      lo = std::min(lo, hp[2 * (b * 3 + q)]);
      hi = std::max(hi, hp[2 * (b * 3 + q) + 1]);
    }
    G.lo[q] = lo;
    ext[q] = hi - lo;
  }
  // cell width: about 4 points per cell if they filled the bounding box (surfaces get more)
  double vol = 1.0;
  int used = 0;
  for (int q = 0; q < d; ++q)
    if (ext[q] > 0.0) {
      vol *= ext[q];
      ++used;
    }
  double h = used ? std::pow(vol * 4.0 / n, 1.0 / used) : 1.0;
  if (!(h > 0.0) || !std::isfinite(h)) h = 1.0;
  long long cells = 1;
  for (;;) {
    cells = 1;
    for (int q = 0; q < d; ++q) {
      G.dim[q] = (int)std::min<double>(ext[q] / h + 1.0, 1 << 20);
      cells *= G.dim[q];
    }
    if (cells <= (long long)4 * n + 64) break;
    h *= 1.25;
  }
  for (int q = d; q < 3; ++q) G.dim[q] = 1;
  G.h = h;
  G.inv_h = 1.0 / h;
  DevBuf<int> cell, counts, start, items;
  GS_CUDA(ctx, cell.alloc(n, s));
  GS_CUDA(ctx, counts.alloc((size_t)cells + 1, s));
  GS_CUDA(ctx, start.alloc((size_t)cells + 1, s));
  GS_CUDA(ctx, items.alloc(n, s));
  GS_CUDA(ctx, cudaMemsetAsync(counts.get(), 0, ((size_t)cells + 1) * sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_grid_count<<<nblk(n), kThreads, 0, s>>>(dpts, n, G, cell.get(), counts.get());
  gs_launch_end(ctx, 1);
  size_t tb = 0;
  GS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tb, counts.get(), start.get(), (int)cells + 1, s));
  DevBuf<unsigned char> tmp;
  GS_CUDA(ctx, tmp.alloc(tb, s));
  GS_CUDA(ctx, cub::DeviceScan::ExclusiveSum(tmp.get(), tb, counts.get(), start.get(), (int)cells + 1, s));
  GS_CUDA(ctx, cudaMemcpyAsync(counts.get(), start.get(), ((size_t)cells + 1) * sizeof(int), cudaMemcpyDeviceToDevice, s));
  gs_launch_begin(ctx, 1);
  k_grid_fill<<<nblk(n), kThreads, 0, s>>>(cell.get(), n, counts.get(), items.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  if (k <= 16)
    k_knn_grid<16><<<(n + 127) / 128, 128, 0, s>>>(dpts, sq, n, G, start.get(), items.get(), max_sq, k, dnb, deps);
  else
    k_knn_grid<32><<<(n + 127) / 128, 128, 0, s>>>(dpts, sq, n, G, start.get(), items.get(), max_sq, k, dnb, deps);
  gs_launch_end(ctx, 1);
  GS_CUDA(ctx, cudaGetLastError());
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// brute force over every candidate for the queries of qlist (the tensor-core path's fallback)
int gs_knn_brute_list(gs_ctx* ctx, const double* dpts, const double* sq, int n, int d, int k,
                      const int* qlist, int nq, int* dnb, double* deps) {
  if (nq <= 0) return GS_OK;
  gs_launch_begin(ctx, 1);
  if (k <= 16) launch_knn_k<16>(dpts, sq, n, d, k, dnb, deps, ctx->stream, qlist, nq);
  else launch_knn_k<32>(dpts, sq, n, d, k, dnb, deps, ctx->stream, qlist, nq);
  gs_launch_end(ctx, 1);
  GS_CUDA(ctx, cudaGetLastError());
  return GS_OK;
}

// tensor-core prefilter for 9 <= d <= 31 (GS_KNN=brute forces the fp64 brute force)
static bool use_tc_knn(int n, int d, int k) {
  const char* e = getenv("GS_KNN");
  if (e && e[0] == 'b') return false;
  if (e && e[0] == 't') return d <= 31 && k <= 24;
  return d >= 9 && d <= 31 && k <= 24 && n >= 4096;
}

static int knn_device(gs_ctx* ctx, const double* dpts, int n, int d, int k, int* dnb, double* deps) {
  cudaStream_t s = ctx->stream;
  DevBuf<double> sq;
  GS_CUDA(ctx, sq.alloc(n, s));
  gs_launch_begin(ctx, 1);
  k_sqnorms<<<nblk(n), kThreads, 0, s>>>(dpts, n, d, sq.get());
  gs_launch_end(ctx, 1);
  if (use_grid_knn(n, d)) return knn_grid(ctx, dpts, sq.get(), n, d, k, dnb, deps);
  if (use_tc_knn(n, d, k)) return gs_knn_tc(ctx, dpts, sq.get(), n, d, k, dnb, deps);
  gs_launch_begin(ctx, 1);
  if (k <= 16) launch_knn_k<16>(dpts, sq.get(), n, d, k, dnb, deps, s);
  else launch_knn_k<32>(dpts, sq.get(), n, d, k, dnb, deps, s);
  gs_launch_end(ctx, 1);
  GS_CUDA(ctx, cudaGetLastError());
  return GS_OK;
}

static int validate_cloud(gs_ctx* ctx, const double* dpts, int n, int d, int k) {
  if (!(n >= 1 && d >= 1)) return gs_fail(ctx, ERRC_DIMENSION_MISMATCH, "point cloud must be non-empty");
  DevBuf<int> bad;
  GS_CUDA(ctx, bad.alloc(1, ctx->stream));
  GS_CUDA(ctx, cudaMemsetAsync(bad.get(), 0, sizeof(int), ctx->stream));
  gs_launch_begin(ctx, 1);
  k_check_finite<<<148 * 8, kThreads, 0, ctx->stream>>>(dpts, (int64_t)n * d, bad.get());
  gs_launch_end(ctx, 1);
  int h = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  if (h) return gs_fail(ctx, ERRC_DIMENSION_MISMATCH, "point cloud has non-finite entries");
  if (k < 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "k must be positive");
  if (k >= n) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "k must be < n");
  if (k > 32) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "k must be <= 32 on the device path");
  if (d > 32) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "dimension must be <= 32 on the device path");
  return GS_OK;
}

extern "C" int gs_knn(gs_ctx* ctx, const double* points, int n, int d, int k, int mem, int* nbrs,
                      double* eps) {
  cudaStream_t s = ctx->stream;
  DevBuf<double> bp;
  const double* dpts = points;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, bp.alloc((size_t)n * d, s));
    GS_CUDA(ctx, cudaMemcpyAsync(bp.get(), points, (size_t)n * d * sizeof(double), cudaMemcpyHostToDevice, s));
    dpts = bp.get();
  }
  GS_TRY(validate_cloud(ctx, dpts, n, d, k));
  DevBuf<int> nb;
  DevBuf<double> ep;
  int* dnb = nbrs;
  double* deps = eps;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, nb.alloc((size_t)n * k, s));
    GS_CUDA(ctx, ep.alloc(n, s));
    dnb = nb.get();
    deps = ep.get();
  }
  GS_TRY(knn_device(ctx, dpts, n, d, k, dnb, deps));
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, cudaMemcpyAsync(nbrs, dnb, (size_t)n * k * sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaMemcpyAsync(eps, deps, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

extern "C" int gs_knn_graph(gs_ctx* ctx, const double* points, int n, int d, int k, int kernel,
                            double param, int mem, gs_graph** out, double* sigma_out) {
  *out = nullptr;
  cudaStream_t s = ctx->stream;
  DevBuf<double> bp;
  const double* dpts = points;
  if (mem != GS_MEM_DEVICE) {
    GS_CUDA(ctx, bp.alloc((size_t)n * d, s));
    GS_CUDA(ctx, cudaMemcpyAsync(bp.get(), points, (size_t)n * d * sizeof(double), cudaMemcpyHostToDevice, s));
    dpts = bp.get();
  }
  GS_TRY(validate_cloud(ctx, dpts, n, d, k));
  if (kernel == GS_KERNEL_ALPHA_DECAY && !(param > 0.0))
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "alpha must be positive");
  if (kernel != GS_KERNEL_ALPHA_DECAY && kernel != GS_KERNEL_GAUSSIAN_MEDIAN)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "unknown edge kernel");
  DevBuf<int> nb, firstbad, nsel, cnt;
  DevBuf<double> eps;
  GS_CUDA(ctx, nb.alloc((size_t)n * k, s));
  GS_CUDA(ctx, eps.alloc(n, s));
  GS_TRY(knn_device(ctx, dpts, n, d, k, nb.get(), eps.get()));
  GS_CUDA(ctx, firstbad.alloc(1, s));
  const int big = 0x7fffffff;
  GS_CUDA(ctx, cudaMemcpyAsync(firstbad.get(), &big, sizeof(int), cudaMemcpyHostToDevice, s));
  gs_launch_begin(ctx, 1);
  k_eps_check<<<nblk(n), kThreads, 0, s>>>(eps.get(), n, firstbad.get());
  gs_launch_end(ctx, 1);
  int h_bad = big;
  GS_CUDA(ctx, cudaMemcpyAsync(&h_bad, firstbad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_bad != big)
    return gs_fail(ctx, ERRC_DUPLICATE_POINTS,
                   "zero k-NN bandwidth at point " + std::to_string(h_bad) + " (duplicate points)");
  // union of directed relations (graph.cpp:91-97)
  const int64_t m = (int64_t)n * k;
  DevBuf<unsigned long long> keys, keys2, ukeys;
  GS_CUDA(ctx, keys.alloc(m, s));
  GS_CUDA(ctx, keys2.alloc(m, s));
  GS_CUDA(ctx, ukeys.alloc(m, s));
  GS_CUDA(ctx, nsel.alloc(1, s));
  gs_launch_begin(ctx, 1);
  k_pair_keys<<<nblk(m), kThreads, 0, s>>>(nb.get(), n, k, keys.get());
  gs_launch_end(ctx, 1);
  {
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.get(), keys2.get(), (int)m, 0, 64, s);
    size_t tb2 = 0;
    cub::DeviceSelect::Unique(nullptr, tb2, keys2.get(), ukeys.get(), nsel.get(), (int)m, s);
    DevBuf<unsigned char> tmp;
    GS_CUDA(ctx, tmp.alloc(tb > tb2 ? tb : tb2, s));
    cub::DeviceRadixSort::SortKeys(tmp.get(), tb, keys.get(), keys2.get(), (int)m, 0, 64, s);
    cub::DeviceSelect::Unique(tmp.get(), tb2, keys2.get(), ukeys.get(), nsel.get(), (int)m, s);
  }
  int u = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&u, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  double sigma2 = 0.0;
  if (kernel == GS_KERNEL_GAUSSIAN_MEDIAN) {
    DevBuf<double> sorted;
    GS_CUDA(ctx, sorted.alloc(n, s));
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, eps.get(), sorted.get(), n, 0, 64, s);
    DevBuf<unsigned char> tmp;
    GS_CUDA(ctx, tmp.alloc(tb, s));
    cub::DeviceRadixSort::SortKeys(tmp.get(), tb, eps.get(), sorted.get(), n, 0, 64, s);
    double mid[2] = {0, 0};
    if (n % 2) {
      GS_CUDA(ctx, cudaMemcpyAsync(&mid[0], sorted.get() + n / 2, sizeof(double), cudaMemcpyDeviceToHost, s));
    } else {
      GS_CUDA(ctx, cudaMemcpyAsync(mid, sorted.get() + n / 2 - 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    const double sigma = (n % 2) ? mid[0] : 0.5 * (mid[0] + mid[1]);
    if (sigma_out) *sigma_out = sigma;
    sigma2 = sigma * sigma;
  }
  const int64_t e2 = 2 * (int64_t)u;
  DevBuf<unsigned long long> ek, ek2;
  DevBuf<double> ev, ev2;
  GS_CUDA(ctx, ek.alloc(e2, s));
  GS_CUDA(ctx, ek2.alloc(e2, s));
  GS_CUDA(ctx, ev.alloc(e2, s));
  GS_CUDA(ctx, ev2.alloc(e2, s));
  GS_CUDA(ctx, cnt.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(cnt.get(), 0, sizeof(int), s));
  if (u > 0) {
    gs_launch_begin(ctx, 1);
    k_pair_weights<<<nblk(u), kThreads, 0, s>>>(ukeys.get(), u, dpts, d, eps.get(), kernel, param,
                                                 sigma2, ek.get(), ev.get());
    k_count_sentinel<<<nblk(e2), kThreads, 0, s>>>(ek.get(), e2, cnt.get());
    gs_launch_end(ctx, 1);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, ek.get(), ek2.get(), ev.get(), ev2.get(), (int)e2, 0, 64, s);
    DevBuf<unsigned char> tmp;
    GS_CUDA(ctx, tmp.alloc(tb, s));
    cub::DeviceRadixSort::SortPairs(tmp.get(), tb, ek.get(), ek2.get(), ev.get(), ev2.get(), (int)e2, 0, 64, s);
  }
  int zeros = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&zeros, cnt.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return gs_csr_from_sorted_entries(ctx, n, e2 - zeros, ek2.get(), ev2.get(), false, out);
}
