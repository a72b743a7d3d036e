// Microbenchmark (tuning tool, not product): smem-staged Chebyshev step vs direct gathers on a
// lattice proxy of the CM-ordered kNN graph (n = W x H vertices, row-major, 13 neighbours from a
// radius-2 stencil, so a block of R rows touches ~3R distinct rows in three stripes).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

constexpr int B = 64;
constexpr int R = 32;  // rows per CTA block

template <bool STAGE>
__global__ void __launch_bounds__(256) k_step(const int* __restrict__ offs, const int* __restrict__ cols,
                                              const unsigned short* __restrict__ slot,
                                              const double* __restrict__ vals,
                                              const int* __restrict__ uoff, const int* __restrict__ urows,
                                              const double* __restrict__ tp, double* __restrict__ t2,
                                              double* __restrict__ acc, int n, double bk) {
  extern __shared__ __align__(16) double sx[];
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (STAGE) {
    const int u0 = uoff[b], u1 = uoff[b + 1];
    for (int u = u0 + warp; u < u1; u += 8) {
      const int r = urows[u];
      const double2 v = __ldg(reinterpret_cast<const double2*>(tp + (size_t)r * B + lane * 2));
      *reinterpret_cast<double2*>(sx + (size_t)(u - u0) * B + lane * 2) = v;
    }
    __syncthreads();
  }
  for (int j = 0; j < R / 8; ++j) {
    const int row = b * R + j * 8 + warp;
    if (row >= n) break;
    const int pb = offs[row], pe = offs[row + 1];
    double y0 = 0, y1 = 0;
    for (int p0 = pb; p0 < pe; p0 += 32) {
      int myc = 0;
      double myv = 0;
      if (p0 + lane < pe) {
        myc = STAGE ? (int)slot[p0 + lane] : cols[p0 + lane];
        myv = vals[p0 + lane];
      }
      const int cnt = min(32, pe - p0);
      for (int u = 0; u < cnt; ++u) {
        const int c = __shfl_sync(0xffffffffu, myc, u);
        const double v = __shfl_sync(0xffffffffu, myv, u);
        double2 x;
        if (STAGE) x = *reinterpret_cast<const double2*>(sx + (size_t)c * B + lane * 2);
        else x = __ldg(reinterpret_cast<const double2*>(tp + (size_t)c * B + lane * 2));
        y0 = fma(v, x.x, y0);
        y1 = fma(v, x.y, y1);
      }
    }
    const size_t idx = (size_t)row * B + lane * 2;
    const double2 a = __ldg(reinterpret_cast<const double2*>(tp + idx));
    const double2 c2 = *reinterpret_cast<const double2*>(t2 + idx);
    const double2 ac = *reinterpret_cast<const double2*>(acc + idx);
    double2 t, o;
    t.x = 2.0 * (y0 - a.x) - c2.x;
    t.y = 2.0 * (y1 - a.y) - c2.y;
    o.x = fma(bk, t.x, ac.x);
    o.y = fma(bk, t.y, ac.y);
    *reinterpret_cast<double2*>(t2 + idx) = t;
    *reinterpret_cast<double2*>(acc + idx) = o;
  }
}

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 700;
  const int n = 200000, H = n / W;
  std::vector<int> offs(n + 1), cols;
  std::vector<double> vals;
  const int dx[] = {0, -1, 1, -2, 2, 0, 0, -1, 1, 0, -1, 1, 0};
  const int dy[] = {0, 0, 0, 0, 0, -1, 1, -1, -1, -2, 1, 1, 2};
  for (int i = 0; i < n; ++i) {
    const int x = i % W, y = i / W;
    std::vector<int> c;
    for (int q = 0; q < 13; ++q) {
      const int xx = x + dx[q], yy = y + dy[q];
      if (xx >= 0 && xx < W && yy >= 0 && yy < H) c.push_back(yy * W + xx);
    }
    std::sort(c.begin(), c.end());
    for (int j : c) {
      cols.push_back(j);
      vals.push_back(0.01);
    }
    offs[i + 1] = (int)cols.size();
  }
  const int nb = (n + R - 1) / R;
  std::vector<int> uoff(nb + 1, 0), urows;
  std::vector<unsigned short> slot(cols.size());
  int maxu = 0;
  for (int b = 0; b < nb; ++b) {
    std::vector<int> u;
    for (int r = b * R; r < std::min(n, (b + 1) * R); ++r)
      for (int p = offs[r]; p < offs[r + 1]; ++p) u.push_back(cols[p]);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    for (int r = b * R; r < std::min(n, (b + 1) * R); ++r)
      for (int p = offs[r]; p < offs[r + 1]; ++p)
        slot[p] = (unsigned short)(std::lower_bound(u.begin(), u.end(), cols[p]) - u.begin());
    urows.insert(urows.end(), u.begin(), u.end());
    uoff[b + 1] = (int)urows.size();
    maxu = std::max(maxu, (int)u.size());
  }
  printf("W=%d nnz=%zu unique rows per %d-row block: mean %.1f max %d\n", W, cols.size(), R,
         (double)urows.size() / nb, maxu);
  int *d_offs, *d_cols, *d_uoff, *d_urows;
  unsigned short* d_slot;
  double *d_vals, *tp, *t2, *acc;
  cudaMalloc(&d_offs, (n + 1) * 4);
  cudaMalloc(&d_cols, cols.size() * 4);
  cudaMalloc(&d_slot, slot.size() * 2);
  cudaMalloc(&d_vals, vals.size() * 8);
  cudaMalloc(&d_uoff, (nb + 1) * 4);
  cudaMalloc(&d_urows, urows.size() * 4);
  cudaMemcpy(d_offs, offs.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_cols, cols.data(), cols.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_slot, slot.data(), slot.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(d_vals, vals.data(), vals.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_uoff, uoff.data(), (nb + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_urows, urows.data(), urows.size() * 4, cudaMemcpyHostToDevice);
  const size_t len = (size_t)n * B;
  cudaMalloc(&tp, len * 8);
  cudaMalloc(&t2, len * 8);
  cudaMalloc(&acc, len * 8);
  cudaMemset(tp, 0, len * 8);
  cudaMemset(t2, 0, len * 8);
  cudaMemset(acc, 0, len * 8);
  cudaEvent_t a, bb;
  cudaEventCreate(&a);
  cudaEventCreate(&bb);
  const size_t smem = (size_t)maxu * B * 8;
  cudaFuncSetAttribute(k_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  auto timeit = [&](const char* name, auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) fn();
    cudaEventRecord(bb);
    cudaEventSynchronize(bb);
    float ms;
    cudaEventElapsedTime(&ms, a, bb);
    const double bytes = cols.size() * 12.0 + 4.0 * n + 5.0 * len * 8;
    printf("%-22s %8.1f us  %7.0f GB/s algorithmic\n", name, 1000 * ms / 20, bytes / (ms / 20 * 1e6));
  };
  timeit("direct gathers", [&] { k_step<false><<<nb, 256>>>(d_offs, d_cols, d_slot, d_vals, d_uoff, d_urows, tp, t2, acc, n, 0.5); });
  timeit("smem staged", [&] { k_step<true><<<nb, 256, smem>>>(d_offs, d_cols, d_slot, d_vals, d_uoff, d_urows, tp, t2, acc, n, 0.5); });
  cudaDeviceSynchronize();
  printf("smem %zu B/CTA; err: %s\n", smem, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
