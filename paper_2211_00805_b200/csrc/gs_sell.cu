// gs_sell.cu -- builds the jagged sliced store of a CSR operator for k_cheb_sell (gs_sell.cuh).
//
// Reference path: the store only re-arranges the entries of L_s (heat.cpp:86-93's scaled copy);
// every row keeps its entries in CSR order (sparse.cpp:15-53), so SparseSymMatrix::multiply's
// per-row sum (sparse.cpp:85-99) runs as the same fma chain.
#include <cub/cub.cuh>

#include "gs_internal.cuh"
#include "gs_sell.cuh"

namespace {

// entries slice s takes: every row's length rounded up to whole chunks, the slice to four entries
__global__ void k_sell_sizes(const int* __restrict__ offs, int n, int C, int JV, int nslices, long long* sz) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > nslices) return;
  long long t = 0;
  if (s < nslices) {
    for (int i = 0; i < C; ++i) {
      const int r = s * C + i;
      if (r < n) t += (offs[r + 1] - offs[r] + JV - 1) / JV * JV;
    }
    t = (t + 3) / 4 * 4;
  }
  sz[s] = t;
}

// cost of slice s for the static split of k_cheb_sellw: chunks of its longest row + a constant
__global__ void k_sell_costs(const int* __restrict__ offs, int n, int C, int nslices, long long* cost) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > nslices) return;
  int mx = 0;
  if (s < nslices)
    for (int i = 0; i < C; ++i) {
      const int r = s * C + i;
      if (r < n) mx = max(mx, offs[r + 1] - offs[r]);
    }
  cost[s] = s < nslices ? (mx + 3) / 4 + 4 : 0;
}

// wstart[w] = first slice whose cost prefix reaches w / W of the total (w = 0 .. W)
__global__ void k_sell_split(const long long* __restrict__ cpre, int nslices, int W, int* wstart) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w > W) return;
  if (w == W) {
    wstart[w] = nslices;
    return;
  }
  const long long total = cpre[nslices];
  const long long target = (long long)(((__int128)total * w) / W);
  int lo = 0, hi = nslices;  // first s with cpre[s] >= target
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cpre[mid] >= target) hi = mid;
    else lo = mid + 1;
  }
  wstart[w] = lo;
}

// One warp per slice, lane i = row i of the slice (C <= 32): the same ballot/rank walk as
// sell_load (gs_sell.cuh), writing instead of reading.
template <typename S>
__global__ void k_sell_fill(const int* __restrict__ offs, const int* __restrict__ cols, const S* __restrict__ vals,
                            int n, int C, int JV, int nslices, const long long* __restrict__ soff, int* ocols,
                            S* ovals) {
  const int s = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (s >= nslices) return;  // warp-uniform
  const int lane = threadIdx.x & 31;
  const unsigned ltmask = (1u << lane) - 1u;
  const int r = s * C + lane;
  const bool valid = lane < C && r < n;
  int pb = 0, len = 0;
  if (valid) {
    pb = offs[r];
    len = offs[r + 1] - pb;
  }
  const int maxlen = __reduce_max_sync(0xffffffffu, len);
  const int PV = 16 / (int)sizeof(S) < JV ? 16 / (int)sizeof(S) : JV;
  const long long O = soff[s];
  long long off = 0;
  for (int jc = 0; jc < maxlen; jc += JV) {
    const bool act = valid && jc < len;
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    const int rank = __popc(bal & ltmask), cnt = __popc(bal);
    if (act) {
      const long long base = O + off;
      for (int e = 0; e < JV; ++e) {
        const bool in = jc + e < len;
        ocols[base + rank * JV + e] = in ? cols[pb + jc + e] : -1;
        ovals[base + (long long)(e / PV) * cnt * PV + rank * PV + e % PV] = in ? vals[pb + jc + e] : S(0);
      }
    }
    off += (long long)cnt * JV;
  }
  // the slice's tail (rounding to four entries) stays col = -1 / val = 0 from the memsets
}

template <typename S>
int build_typed(gs_ctx* ctx, const gs_graph* G, const S* vals, int C, int JV, gs_sell* out) {
  cudaStream_t s = ctx->stream;
  const int n = G->n;
  const int nslices = (n + C - 1) / C;
  DevBuf<long long> sz;
  GS_CUDA(ctx, sz.alloc((size_t)nslices + 1, s));
  gs_launch_begin(ctx, 1);
  k_sell_sizes<<<(nslices + 1 + 255) / 256, 256, 0, s>>>(G->offs, n, C, JV, nslices, sz.get());
  gs_launch_end(ctx, 1);
  if (cudaMalloc((void**)&out->soff, ((size_t)nslices + 1) * sizeof(long long)) != cudaSuccess)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "sliced store: offset allocation failed");
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, sz.get(), out->soff, nslices + 1, s);
  DevBuf<unsigned char> tmp;
  GS_CUDA(ctx, tmp.alloc(tb, s));
  cub::DeviceScan::ExclusiveSum(tmp.get(), tb, sz.get(), out->soff, nslices + 1, s);
  long long total = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&total, out->soff + nslices, sizeof total, cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  out->total = total;
  out->nslices = nslices;
  const size_t cnt = (size_t)total + kCsrPad;
  if (cudaMalloc((void**)&out->cols, cnt * sizeof(int)) != cudaSuccess ||
      cudaMalloc((void**)&out->vals, cnt * sizeof(S)) != cudaSuccess)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "sliced store: allocation failed");
  GS_CUDA(ctx, cudaMemsetAsync(out->cols, 0xff, cnt * sizeof(int), s));
  GS_CUDA(ctx, cudaMemsetAsync(out->vals, 0, cnt * sizeof(S), s));
  if (nslices > 0) {
    gs_launch_begin(ctx, 1);
    k_sell_fill<S><<<(unsigned)(((long long)nslices * 32 + 255) / 256), 256, 0, s>>>(
        G->offs, G->cols, vals, n, C, JV, nslices, out->soff, out->cols, static_cast<S*>(out->vals));
    gs_launch_end(ctx, 1);
  }
  // cost prefix for the static warp split
  if (cudaMalloc((void**)&out->cpre, ((size_t)nslices + 1) * sizeof(long long)) != cudaSuccess)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "sliced store: cost allocation failed");
  gs_launch_begin(ctx, 1);
  k_sell_costs<<<(nslices + 1 + 255) / 256, 256, 0, s>>>(G->offs, n, C, nslices, sz.get());
  gs_launch_end(ctx, 1);
  cub::DeviceScan::ExclusiveSum(tmp.get(), tb, sz.get(), out->cpre, nslices + 1, s);
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

}  // namespace

// Static split of the slices over W warps at equal cost (device array of W + 1 ints).
int gs_sell_split(gs_ctx* ctx, const gs_sell* p, int W, int* d_wstart) {
  gs_launch_begin(ctx, 1);
  k_sell_split<<<(W + 1 + 255) / 256, 256, 0, ctx->stream>>>(p->cpre, p->nslices, W, d_wstart);
  gs_launch_end(ctx, 1);
  return GS_OK;
}

void gs_sell_destroy(gs_sell* p) {
  if (!p) return;
  cudaFree(p->soff);
  cudaFree(p->cols);
  cudaFree(p->vals);
  cudaFree(p->cpre);
  delete p;
}

// Sliced store of G for slices of C rows and values of elem_bytes (8: G->vals; 4: vals32).
int gs_sell_build(gs_ctx* ctx, const gs_graph* G, const float* vals32, int C, int elem_bytes, gs_sell** out) {
  *out = nullptr;
  if (C < 1 || C > 32 || (32 % C) != 0 || (elem_bytes != 4 && elem_bytes != 8) || (elem_bytes == 4 && !vals32))
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "sliced store: bad slice height or element size");
  gs_sell* p = new gs_sell();
  p->C = C;
  p->JV = gsk::sell_jv(C);
  p->elem_bytes = elem_bytes;
  const int rc = elem_bytes == 8 ? build_typed<double>(ctx, G, G->vals, C, p->JV, p)
                                 : build_typed<float>(ctx, G, vals32, C, p->JV, p);
  if (rc) {
    gs_sell_destroy(p);
    return rc;
  }
  *out = p;
  return GS_OK;
}
