// Microbenchmark (tuning tool, not product): the ceiling of config 2's access pattern -- random
// 64-byte row gathers from a table that stays L2-resident (n = 1e6 rows x 8 doubles = 64 MB),
// 26.5 entries per row drawn inside the row's 50,000-row cluster (a kNN graph in R^30 has no
// finer index locality), index stream read coalesced. No fma chain, no T_{k-2} / acc streams,
// no epilogue: only the (col) stream, the gathers and one 64-byte store per row. Reports the time
// of one pass and the L2->SM gather bandwidth, to compare with k_cheb_step<double,8> (324 us).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mb_gather tools/mb_gather.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

constexpr int B = 8;  // doubles per row

// 8 lanes per row (one double each), 4 rows per warp, GB gathers in flight per lane
template <int GB>
__global__ void __launch_bounds__(256) k_gather(const int* __restrict__ offs, const int* __restrict__ cols,
                                                const double* __restrict__ tp, double* __restrict__ out, int n) {
  const int lane = threadIdx.x & 31, q = lane & 7;
  const int row = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 4 + (lane >> 3);
  if (row >= n) return;
  const int pb = offs[row], pe = offs[row + 1];
  const unsigned mask = 0xffu << (lane & 24);
  double y = 0;
  for (int p0 = pb; p0 < pe; p0 += 8) {
    const int myc = p0 + q < pe ? __ldg(cols + p0 + q) : -1;
    const int cnt = min(8, pe - p0);
    for (int u = 0; u < cnt; u += GB) {
      double x[GB];
#pragma unroll
      for (int j = 0; j < GB; ++j) {
        const int c = __shfl_sync(mask, myc, min(u + j, cnt - 1), 8);
        x[j] = __ldg(tp + (size_t)c * B + q);
      }
#pragma unroll
      for (int j = 0; j < GB; ++j)
        if (u + j < cnt) y += x[j];
    }
  }
  out[(size_t)row * B + q] = y;
}

// the same pass with the value stream: (col, val) chunks loaded coalesced and broadcast with three
// shuffles per entry (col, and the two halves of the fp64 value), fma chain -- k_cheb_step's
// narrow-row inner loop without its own-row streams
template <int GB>
__global__ void __launch_bounds__(256) k_gather_val(const int* __restrict__ offs, const int* __restrict__ cols,
                                                    const double* __restrict__ vals, const double* __restrict__ tp,
                                                    double* __restrict__ out, int n) {
  const int lane = threadIdx.x & 31, q = lane & 7;
  const int row = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 4 + (lane >> 3);
  if (row >= n) return;
  const int pb = offs[row], pe = offs[row + 1];
  const unsigned mask = 0xffu << (lane & 24);
  double y = 0;
  for (int p0 = pb; p0 < pe; p0 += 8) {
    const int myc = p0 + q < pe ? __ldg(cols + p0 + q) : -1;
    const double myv = p0 + q < pe ? __ldg(vals + p0 + q) : 0.0;
    const int cnt = min(8, pe - p0);
    for (int u = 0; u < cnt; u += GB) {
      double x[GB], v[GB];
#pragma unroll
      for (int j = 0; j < GB; ++j) {
        const int c = __shfl_sync(mask, myc, min(u + j, cnt - 1), 8);
        v[j] = __shfl_sync(mask, myv, min(u + j, cnt - 1), 8);
        x[j] = __ldg(tp + (size_t)c * B + q);
      }
#pragma unroll
      for (int j = 0; j < GB; ++j)
        if (u + j < cnt) y = fma(v[j], x[j], y);
    }
  }
  out[(size_t)row * B + q] = y;
}

// (col, val) as 16-byte records staged per warp in shared memory by one bulk copy; every lane
// reads its row's record with one 16-byte shared-memory load (a broadcast inside the row's lanes)
struct Rec {
  int col, pad;
  double val;
};
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int GB, int CAP>
__global__ void __launch_bounds__(256) k_gather_rec(const int* __restrict__ offs, const Rec* __restrict__ recs,
                                                    const double* __restrict__ tp, double* __restrict__ out, int n) {
  __shared__ __align__(128) Rec s_rec[8][CAP];
  __shared__ __align__(8) unsigned long long s_bar[8];
  const int lane = threadIdx.x & 31, q = lane & 7, warp = threadIdx.x >> 5;
  const int r0 = (blockIdx.x * 8 + warp) * 4;
  const int row = r0 + (lane >> 3);
  if (r0 >= n) return;
  const int p0 = offs[r0], p1 = offs[min(r0 + 4, n)];
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&s_bar[warp])) : "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    const unsigned bytes = (unsigned)((p1 - p0) * sizeof(Rec));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&s_bar[warp])), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(&s_rec[warp][0])), "l"(recs + p0), "r"(bytes), "r"(smem_u32(&s_bar[warp])) : "memory");
  }
  __syncwarp();
  const int pb = row < n ? offs[row] - p0 : 0, pe = row < n ? offs[row + 1] - p0 : 0;
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}\n" ::"r"(
                   smem_u32(&s_bar[warp])) : "memory");
  double y = 0;
  for (int p = pb; p < pe; p += GB) {
    double x[GB], v[GB];
#pragma unroll
    for (int j = 0; j < GB; ++j) {
      const int4 r = *reinterpret_cast<const int4*>(&s_rec[warp][min(p + j, pe - 1)]);
      v[j] = __hiloint2double(r.w, r.z);
      x[j] = __ldg(tp + (size_t)r.x * B + q);
    }
#pragma unroll
    for (int j = 0; j < GB; ++j)
      if (p + j < pe) y = fma(v[j], x[j], y);
  }
  if (row < n) out[(size_t)row * B + q] = y;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1000000;
  const int cluster = 50000;
  std::mt19937 rng(7);
  std::vector<int> offs(n + 1, 0), cols;
  cols.reserve((size_t)n * 27);
  for (int i = 0; i < n; ++i) {
    const int d = 20 + (int)(rng() % 14);  // 26.5 on average
    const int c0 = i / cluster * cluster;
    for (int j = 0; j < d; ++j) cols.push_back(c0 + (int)(rng() % cluster));
    offs[i + 1] = (int)cols.size();
  }
  const size_t nnz = cols.size();
  int *d_offs, *d_cols;
  double *d_tp, *d_out;
  cudaMalloc(&d_offs, (n + 1) * sizeof(int));
  cudaMalloc(&d_cols, (nnz + 8) * sizeof(int));
  cudaMalloc(&d_tp, (size_t)n * B * sizeof(double));
  cudaMalloc(&d_out, (size_t)n * B * sizeof(double));
  cudaMemcpy(d_offs, offs.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(d_cols, cols.data(), nnz * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemset(d_tp, 0, (size_t)n * B * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name) {
    const int grid = (n + 31) / 32;
    for (int i = 0; i < 3; ++i) kern<<<grid, 256>>>(d_offs, d_cols, d_tp, d_out, n);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) kern<<<grid, 256>>>(d_offs, d_cols, d_tp, d_out, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = 1e3 * ms / reps;
    printf("%s: %.1f us per pass, %zu gathers, %.2f TB/s of 64-byte rows from L2\n", name, us, nnz,
           (double)nnz * 64 / us * 1e-6);
  };
  run(k_gather<4>, "gathers in flight 4");
  run(k_gather<8>, "gathers in flight 8");
  std::vector<double> vals(nnz, 0.5);
  std::vector<Rec> recs(nnz + 8);
  int maxw = 0;
  for (int r = 0; r < n; r += 4) maxw = std::max(maxw, offs[std::min(r + 4, n)] - offs[r]);
  for (size_t p = 0; p < nnz; ++p) recs[p] = Rec{cols[p], 0, 0.5};
  double* d_vals;
  Rec* d_recs;
  cudaMalloc(&d_vals, (nnz + 8) * sizeof(double));
  cudaMalloc(&d_recs, (nnz + 8) * sizeof(Rec));
  cudaMemcpy(d_vals, vals.data(), nnz * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(d_recs, recs.data(), (nnz + 8) * sizeof(Rec), cudaMemcpyHostToDevice);
  auto runv = [&](auto kern, const char* name, auto a2) {
    const int grid = (n + 31) / 32;
    for (int i = 0; i < 3; ++i) kern<<<grid, 256>>>(d_offs, a2, d_tp, d_out, n);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) kern<<<grid, 256>>>(d_offs, a2, d_tp, d_out, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s: %.1f us per pass\n", name, 1e3 * ms / reps);
  };
  {
    const int grid = (n + 31) / 32;
    for (int i = 0; i < 3; ++i) k_gather_val<8><<<grid, 256>>>(d_offs, d_cols, d_vals, d_tp, d_out, n);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) k_gather_val<8><<<grid, 256>>>(d_offs, d_cols, d_vals, d_tp, d_out, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("col + val chunks, 3 shuffles per entry, fma chain (8 in flight): %.1f us per pass\n", 1e3 * ms / 20);
    for (int i = 0; i < 3; ++i) k_gather_val<4><<<grid, 256>>>(d_offs, d_cols, d_vals, d_tp, d_out, n);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) k_gather_val<4><<<grid, 256>>>(d_offs, d_cols, d_vals, d_tp, d_out, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("col + val chunks, 3 shuffles per entry, fma chain (4 in flight): %.1f us per pass\n", 1e3 * ms / 20);
  }
  printf("largest 4-row slice: %d records\n", maxw);
  if (maxw <= 160) {
    runv(k_gather_rec<4, 160>, "16-byte records staged per warp, LDS.128 broadcast (4 in flight)", d_recs);
    runv(k_gather_rec<8, 160>, "16-byte records staged per warp, LDS.128 broadcast (8 in flight)", d_recs);
  }
  printf("cuda status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
