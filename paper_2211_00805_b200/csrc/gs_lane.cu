// gs_lane.cu -- copies of a CSR operator for the staged step kernels of gs_step.cuh: the odd-stride
// copy k_cheb_lane reads, and the 16-byte record copy of the opt-in k_cheb_rec.
//
// Reference path: the copy only re-spaces the entries of L_s (heat.cpp:86-93's scaled copy):
// every row keeps its entries in CSR order (sparse.cpp:15-53), so SparseSymMatrix::multiply's
// per-row sum (sparse.cpp:85-99) runs as the same fma chain.
//
// k_cheb_lane stages the slice of a warp's 32 rows in shared memory and lane i reads entry u of
// its own row, at word start_i + u. Rows of a degree-sorted block share their length d, so the
// lanes' stride is d words: an even d maps them onto 32 / gcd(d, 32) banks (d = 12: 4-way, d = 16:
// 16-way conflicts; config 3: 58% of the shared-memory wavefronts were conflict replays). Here
// every row with an even number of entries is followed by one pad entry (column -1, value 0),
// which makes every row stride odd: equal lengths in a warp are conflict-free. The kernel drops a
// row's pad by looking at its last column.
#include <cub/cub.cuh>

#include "gs_internal.cuh"

namespace {

__global__ void k_lp_len(const int* __restrict__ offs, int n, int* len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  len[i] = i < n ? ((offs[i + 1] - offs[i]) | 1) : 0;
}

template <typename V>
__global__ void k_lp_fill(const int* __restrict__ offs, const int* __restrict__ cols, const V* __restrict__ vals,
                          const int* __restrict__ poffs, int n, int* pcols, V* pvals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = offs[i], e = offs[i + 1];
  int q = poffs[i];
  for (int p = b; p < e; ++p, ++q) {
    pcols[q] = cols[p];
    pvals[q] = vals[p];
  }
  if (q < poffs[i + 1]) {
    pcols[q] = -1;
    pvals[q] = V(0);
  }
}

struct Rec16 {
  int col, pad;
  double val;
};
__global__ void k_recs_fill(const int* __restrict__ cols, const double* __restrict__ vals, long long nnz,
                            long long total, Rec16* out) {
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= total) return;
  Rec16 r{0, 0, 0.0};
  if (p < nnz) {
    r.col = cols[p];
    r.val = vals[p];
  }
  out[p] = r;
}

}  // namespace

// k_cheb_rec's copy of the entries (gs_step.cuh): one 16-byte record per entry, CSR order
int gs_recs_build(gs_ctx* ctx, const int* cols, const double* vals, int64_t nnz, void** out) {
  *out = nullptr;
  const long long total = nnz + kCsrPad;
  Rec16* r = nullptr;
  if (cudaMalloc((void**)&r, (size_t)total * sizeof(Rec16)) != cudaSuccess)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "record copy allocation failed");
  gs_launch_begin(ctx, 1);
  k_recs_fill<<<(unsigned)((total + 255) / 256), 256, 0, ctx->stream>>>(cols, vals, nnz, total, r);
  gs_launch_end(ctx, 1);
  const cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    cudaFree(r);
    return gs_cuda_fail(ctx, e, "record copy");
  }
  *out = r;
  return GS_OK;
}

void gs_lanepad_destroy(gs_lanepad* p) {
  if (!p) return;
  cudaFree(p->offs);
  cudaFree(p->cols);
  cudaFree(p->vals);
  delete p;
}

int gs_lanepad_build(gs_ctx* ctx, const int* offs, const int* cols, const void* vals, int elem_bytes, int n,
                     int64_t nnz, gs_lanepad** out) {
  *out = nullptr;
  if (nnz + n + kCsrPad >= (int64_t)INT32_MAX) return GS_ERR_UNSUPPORTED;  // 32-bit entry positions
  cudaStream_t s = ctx->stream;
  struct Guard {  // frees the partial copy on every early return
    gs_lanepad* p;
    ~Guard() { gs_lanepad_destroy(p); }
  } guard{new gs_lanepad()};
  gs_lanepad* P = guard.p;
  P->elem_bytes = elem_bytes;
  auto fail = [&](const char* what) { return gs_fail(ctx, ERRC_INVALID_ARGUMENT, what); };
  if (cudaMalloc((void**)&P->offs, (size_t)(n + 1) * sizeof(int)) != cudaSuccess) return fail("lane copy allocation failed");
  DevBuf<int> len;
  GS_CUDA(ctx, len.alloc((size_t)n + 1, s));
  const unsigned nb = (unsigned)((n + 1 + 255) / 256);
  gs_launch_begin(ctx, 1);
  k_lp_len<<<nb, 256, 0, s>>>(offs, n, len.get());
  gs_launch_end(ctx, 1);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, len.get(), P->offs, n + 1, s);
  DevBuf<unsigned char> tmp;
  GS_CUDA(ctx, tmp.alloc(tb, s));
  cub::DeviceScan::ExclusiveSum(tmp.get(), tb, len.get(), P->offs, n + 1, s);
  int total = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&total, P->offs + n, sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  P->nnz = total;
  const size_t cnt = (size_t)total + kCsrPad;
  if (cudaMalloc((void**)&P->cols, cnt * sizeof(int)) != cudaSuccess ||
      cudaMalloc((void**)&P->vals, cnt * (size_t)elem_bytes) != cudaSuccess)
    return fail("lane copy allocation failed");
  GS_CUDA(ctx, cudaMemsetAsync(P->cols + total, 0, kCsrPad * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(static_cast<char*>(P->vals) + (size_t)total * elem_bytes, 0,
                               (size_t)kCsrPad * elem_bytes, s));
  if (n > 0) {
    gs_launch_begin(ctx, 1);
    if (elem_bytes == 4)
      k_lp_fill<float><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(offs, cols, static_cast<const float*>(vals),
                                                                   P->offs, n, P->cols, static_cast<float*>(P->vals));
    else
      k_lp_fill<double><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(offs, cols, static_cast<const double*>(vals),
                                                                    P->offs, n, P->cols, static_cast<double*>(P->vals));
    gs_launch_end(ctx, 1);
  }
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  guard.p = nullptr;
  *out = P;
  return GS_OK;
}
