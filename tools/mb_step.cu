// Microbenchmark (tuning tool, not product): ceilings of the Chebyshev step's two halves on a
// synthetic banded graph shaped like config 1 (n = 200k rows, 13 entries/row within +-W,
// B = 64 doubles per row). Kernels: streams only (3 row reads + 2 row writes), gathers only
// (y = sum v * T[col], 1 write), and both (the real step's traffic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

constexpr int B = 64;

__global__ void k_stream(const double* __restrict__ tp, double* __restrict__ t2, double* __restrict__ acc,
                         int n, double bk) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int q = threadIdx.x & 31;
  if (row >= n) return;
  const size_t idx = (size_t)row * B + q * 2;
  const double2 a = *reinterpret_cast<const double2*>(tp + idx);
  const double2 b = *reinterpret_cast<const double2*>(t2 + idx);
  const double2 c = *reinterpret_cast<const double2*>(acc + idx);
  double2 t, o;
  t.x = 2.0 * (a.x * 0.5 - a.x) - b.x;
  t.y = 2.0 * (a.y * 0.5 - a.y) - b.y;
  o.x = fma(bk, t.x, c.x);
  o.y = fma(bk, t.y, c.y);
  *reinterpret_cast<double2*>(t2 + idx) = t;
  *reinterpret_cast<double2*>(acc + idx) = o;
}

template <bool STREAM>
__global__ void k_gather(const int* __restrict__ offs, const int* __restrict__ cols,
                         const double* __restrict__ vals, const double* __restrict__ tp,
                         double* __restrict__ t2, double* __restrict__ acc, int n, double bk) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int q = threadIdx.x & 31;
  if (row >= n) return;
  const int pb = offs[row], pe = offs[row + 1];
  double y0 = 0, y1 = 0;
  for (int p0 = pb; p0 < pe; p0 += 32) {
    int myc = 0;
    double myv = 0;
    if (p0 + q < pe) {
      myc = cols[p0 + q];
      myv = vals[p0 + q];
    }
    const int cnt = min(32, pe - p0);
    int u = 0;
    for (; u + 4 <= cnt; u += 4) {
      int cc[4];
      double vv[4];
      double2 xx[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        cc[j] = __shfl_sync(0xffffffffu, myc, u + j);
        vv[j] = __shfl_sync(0xffffffffu, myv, u + j);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) xx[j] = __ldg(reinterpret_cast<const double2*>(tp + (size_t)cc[j] * B + q * 2));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        y0 = fma(vv[j], xx[j].x, y0);
        y1 = fma(vv[j], xx[j].y, y1);
      }
    }
    for (; u < cnt; ++u) {
      const int c = __shfl_sync(0xffffffffu, myc, u);
      const double v = __shfl_sync(0xffffffffu, myv, u);
      const double2 x = __ldg(reinterpret_cast<const double2*>(tp + (size_t)c * B + q * 2));
      y0 = fma(v, x.x, y0);
      y1 = fma(v, x.y, y1);
    }
  }
  const size_t idx = (size_t)row * B + q * 2;
  if (STREAM) {
    const double2 a = *reinterpret_cast<const double2*>(tp + idx);
    const double2 b = *reinterpret_cast<const double2*>(t2 + idx);
    const double2 c = *reinterpret_cast<const double2*>(acc + idx);
    double2 t, o;
    t.x = 2.0 * (y0 - a.x) - b.x;
    t.y = 2.0 * (y1 - a.y) - b.y;
    o.x = fma(bk, t.x, c.x);
    o.y = fma(bk, t.y, c.y);
    *reinterpret_cast<double2*>(t2 + idx) = t;
    *reinterpret_cast<double2*>(acc + idx) = o;
  } else {
    *reinterpret_cast<double2*>(t2 + idx) = make_double2(y0, y1);
  }
}

// Persistent variant: grouped layout (GW doubles per row-group), each CTA sweeps a contiguous
// row range of one group in order, so its SM's L1 keeps the sliding neighbour window.
template <int GW, bool STREAM>
__global__ void __launch_bounds__(256) k_persist(const int* __restrict__ offs, const int* __restrict__ cols,
                          const double* __restrict__ vals, const double* __restrict__ tp,
                          double* __restrict__ t2, double* __restrict__ acc, int n, int G,
                          int ctas_per_group, double bk) {
  constexpr int LPR = GW / 2, RPW = 32 / LPR, BR = 8 * RPW;
  const int g = blockIdx.x / ctas_per_group;
  const int c = blockIdx.x % ctas_per_group;
  const int chunk = (n + ctas_per_group - 1) / ctas_per_group;
  const int r0 = c * chunk, r1 = min(n, r0 + chunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane / LPR, q = lane % LPR;
  const unsigned mask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const size_t gb = (size_t)g * n * GW + q * 2;
  for (int rb = r0; rb < r1; rb += BR) {
    const int row = rb + warp * RPW + sub;
    const bool valid = row < r1;
    const int pb = valid ? offs[row] : 0, pe = valid ? offs[row + 1] : 0;
    double y0 = 0, y1 = 0;
    for (int p0 = pb; p0 < pe; p0 += LPR) {
      int myc = 0;
      double myv = 0;
      if (p0 + q < pe) {
        myc = cols[p0 + q];
        myv = vals[p0 + q];
      }
      const int cnt = min(LPR, pe - p0);
      int u = 0;
      for (; u + 4 <= cnt; u += 4) {
        int cc[4];
        double vv[4];
        double2 xx[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          cc[j] = __shfl_sync(mask, myc, u + j, LPR);
          vv[j] = __shfl_sync(mask, myv, u + j, LPR);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) xx[j] = __ldg(reinterpret_cast<const double2*>(tp + gb + (size_t)cc[j] * GW));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          y0 = fma(vv[j], xx[j].x, y0);
          y1 = fma(vv[j], xx[j].y, y1);
        }
      }
      for (; u < cnt; ++u) {
        const int cc = __shfl_sync(mask, myc, u, LPR);
        const double v = __shfl_sync(mask, myv, u, LPR);
        const double2 x = __ldg(reinterpret_cast<const double2*>(tp + gb + (size_t)cc * GW));
        y0 = fma(v, x.x, y0);
        y1 = fma(v, x.y, y1);
      }
    }
    if (!valid) continue;
    const size_t idx = gb + (size_t)row * GW;
    if (STREAM) {
      const double2 a = __ldg(reinterpret_cast<const double2*>(tp + idx));
      const double2 b = __ldcs(reinterpret_cast<const double2*>(t2 + idx));
      const double2 cacc = __ldcs(reinterpret_cast<const double2*>(acc + idx));
      double2 t, o;
      t.x = 2.0 * (y0 - a.x) - b.x;
      t.y = 2.0 * (y1 - a.y) - b.y;
      o.x = fma(bk, t.x, cacc.x);
      o.y = fma(bk, t.y, cacc.y);
      __stcs(reinterpret_cast<double2*>(t2 + idx), t);
      __stcs(reinterpret_cast<double2*>(acc + idx), o);
    } else {
      __stcs(reinterpret_cast<double2*>(t2 + idx), make_double2(y0, y1));
    }
  }
}

int main(int argc, char** argv) {
  const int n = 200000, deg = 13;
  const int W = argc > 1 ? atoi(argv[1]) : 1000;
  std::mt19937 rng(1);
  std::vector<int> offs(n + 1), cols;
  std::vector<double> vals;
  for (int i = 0; i < n; ++i) {
    std::vector<int> c;
    c.push_back(i);
    while ((int)c.size() < deg) {
      int j = i + (int)(rng() % (2 * W + 1)) - W;
      if (j >= 0 && j < n && std::find(c.begin(), c.end(), j) == c.end()) c.push_back(j);
    }
    std::sort(c.begin(), c.end());
    for (int j : c) {
      cols.push_back(j);
      vals.push_back(0.01);
    }
    offs[i + 1] = (int)cols.size();
  }
  int *d_offs, *d_cols;
  double *d_vals, *tp, *t2, *acc;
  cudaMalloc(&d_offs, (n + 1) * 4);
  cudaMalloc(&d_cols, cols.size() * 4);
  cudaMalloc(&d_vals, vals.size() * 8);
  cudaMemcpy(d_offs, offs.data(), (n + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_cols, cols.data(), cols.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_vals, vals.data(), vals.size() * 8, cudaMemcpyHostToDevice);
  const size_t len = (size_t)n * B;
  cudaMalloc(&tp, len * 8);
  cudaMalloc(&t2, len * 8);
  cudaMalloc(&acc, len * 8);
  cudaMemset(tp, 0, len * 8);
  cudaMemset(t2, 0, len * 8);
  cudaMemset(acc, 0, len * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = (n + 7) / 8;
  auto timeit = [&](const char* name, auto fn, double bytes) {
    for (int w = 0; w < 3; ++w) fn();
    cudaEventRecord(a);
    const int reps = 20;
    for (int r = 0; r < reps; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = 1000.0 * ms / reps;
    printf("%-28s W=%5d %8.1f us  %7.0f GB/s (model bytes %.0f MB)\n", name, W, us, bytes / (us * 1e3), bytes / 1e6);
  };
  const double vb = (double)len * 8;
  const double mb = cols.size() * 12.0 + 4.0 * (n + 1);
  timeit("stream (3R+2W)", [&] { k_stream<<<grid, 256>>>(tp, t2, acc, n, 0.5); }, 5 * vb);
  timeit("gather only (+1W)", [&] { k_gather<false><<<grid, 256>>>(d_offs, d_cols, d_vals, tp, t2, acc, n, 0.5); }, 2 * vb + mb);
  timeit("gather+stream (step)", [&] { k_gather<true><<<grid, 256>>>(d_offs, d_cols, d_vals, tp, t2, acc, n, 0.5); }, 5 * vb + mb);
  for (int cps : {2, 4, 8}) {
    const int nct = 144 * cps;  // divisible by 1, 2, 4, 8 groups
    char nm[64];
    snprintf(nm, sizeof nm, "persist GW=16 cps=%d gather", cps);
    timeit(nm, [&] { k_persist<16, false><<<nct, 256>>>(d_offs, d_cols, d_vals, tp, t2, acc, n, 4, nct / 4, 0.5); }, 2 * vb + mb);
    snprintf(nm, sizeof nm, "persist GW=16 cps=%d step", cps);
    timeit(nm, [&] { k_persist<16, true><<<nct, 256>>>(d_offs, d_cols, d_vals, tp, t2, acc, n, 4, nct / 4, 0.5); }, 5 * vb + mb);
    snprintf(nm, sizeof nm, "persist GW=8 cps=%d step", cps);
    timeit(nm, [&] { k_persist<8, true><<<nct, 256>>>(d_offs, d_cols, d_vals, tp, t2, acc, n, 8, nct / 8, 0.5); }, 5 * vb + mb);
    snprintf(nm, sizeof nm, "persist GW=32 cps=%d step", cps);
    timeit(nm, [&] { k_persist<32, true><<<nct, 256>>>(d_offs, d_cols, d_vals, tp, t2, acc, n, 2, nct / 2, 0.5); }, 5 * vb + mb);
    snprintf(nm, sizeof nm, "persist GW=64 cps=%d step", cps);
    timeit(nm, [&] { k_persist<64, true><<<nct, 256>>>(d_offs, d_cols, d_vals, tp, t2, acc, n, 1, nct, 0.5); }, 5 * vb + mb);
  }
  cudaDeviceSynchronize();
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
