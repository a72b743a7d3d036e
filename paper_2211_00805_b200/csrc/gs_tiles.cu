// gs_tiles.cu -- neighbour staging plan for the shared-memory Chebyshev step (k_cheb_tile).
//
// For every block of R consecutive rows of the locality-ordered L_s, the set of columns its
// entries reference is a handful of row runs (previous / own / next BFS-level stretches under the
// Cuthill-McKee order). The plan stores those runs (gaps of <= kGap rows are merged so one bulk
// copy moves each run) and, per CSR entry, the 16-bit position ("slot") of its column inside the
// block's staged window. The step kernel then copies each run of T_{k-1} rows into shared memory
// with one TMA bulk copy and gathers from shared memory instead of L1/L2.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "gs_internal.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kGap = 4;

inline unsigned nblk(int64_t m, int t = kThreads) { return (unsigned)((m + t - 1) / t); }

__global__ void k_entry_rows(const int* offs, int n, int* rowof) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int p = offs[r]; p < offs[r + 1]; ++p) rowof[p] = r;
}

__global__ void k_block_keys(const int* rowof, const int* cols, int64_t nnz, int R,
                             unsigned long long* keys) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < nnz) keys[p] = ((unsigned long long)(unsigned)(rowof[p] / R) << 32) | (unsigned)cols[p];
}

__global__ void k_run_heads(const unsigned long long* u, int m, int* head) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int h = 1;
  if (i > 0) {
    const unsigned bprev = (unsigned)(u[i - 1] >> 32), b = (unsigned)(u[i] >> 32);
    const int cprev = (int)(u[i - 1] & 0xFFFFFFFFull), c = (int)(u[i] & 0xFFFFFFFFull);
    h = (b != bprev || c - cprev > kGap + 1) ? 1 : 0;
  }
  head[i] = h;
}

// run ids = inclusive scan of heads - 1; heads/tails record start/end/block
__global__ void k_run_bounds(const unsigned long long* u, const int* rid_incl, int m, int* rstart,
                             int* rend, int* rblock) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int rid = rid_incl[i] - 1;
  const bool head = i == 0 || rid_incl[i - 1] != rid_incl[i];
  const bool tail = i == m - 1 || rid_incl[i + 1] != rid_incl[i];
  const int c = (int)(u[i] & 0xFFFFFFFFull);
  if (head) {
    rstart[rid] = c;
    rblock[rid] = (int)(u[i] >> 32);
  }
  if (tail) rend[rid] = c;
}

__global__ void k_run_len(const int* rstart, const int* rend, int nruns, int* rlen) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nruns) rlen[r] = rend[r] - rstart[r] + 1;
}

__global__ void k_block_first(const int* rblock, int nruns, int* bfirst) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nruns) return;
  if (r == 0 || rblock[r - 1] != rblock[r]) bfirst[rblock[r]] = r;
}

// per block: run range [first, first + count) and slot count; empty blocks get count 0
__global__ void k_block_ranges(const int* bfirst, const int* rblock, const int* gbase,
                               const int* rlen, int nblocks, int nruns, int* bcount,
                               int* bslots) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  const int f = bfirst[b];
  if (f < 0) {
    bcount[b] = 0;
    bslots[b] = 0;
    return;
  }
  int e = f;
  while (e < nruns && rblock[e] == b) ++e;
  bcount[b] = e - f;
  bslots[b] = gbase[e - 1] + rlen[e - 1] - gbase[f];
}

// local slot base of every run (slots of earlier runs of the same block)
__global__ void k_run_lbase(const int* rblock, const int* bfirst, const int* gbase, int nruns,
                            int* lbase) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nruns) lbase[r] = gbase[r] - gbase[bfirst[rblock[r]]];
}

__global__ void k_entry_slots(const int* rowof, const int* cols, int64_t nnz, int R,
                              const int* bfirst, const int* bcount, const int* rstart,
                              const int* rend, const int* lbase, unsigned short* slot) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const int b = rowof[p] / R;
  const int c = cols[p];
  int lo = bfirst[b], hi = lo + bcount[b] - 1;
  while (lo < hi) {  // last run with start <= c
    const int mid = (lo + hi + 1) >> 1;
    if (rstart[mid] <= c) lo = mid;
    else hi = mid - 1;
  }
  slot[p] = (unsigned short)(lbase[lo] + (c - rstart[lo]));
}

}  // namespace

void gs_tiles_release(gs_tileplan& t) {
  cudaFree(t.bfirst);
  cudaFree(t.bcount);
  cudaFree(t.rstart);
  cudaFree(t.rlen);
  cudaFree(t.lbase);
  cudaFree(t.slot);
  t = gs_tileplan();
}

int gs_tiles_build(gs_ctx* ctx, const gs_graph* g, int R, gs_tileplan* out) {
  const int n = g->n;
  const int64_t nnz = g->nnz;
  cudaStream_t s = ctx->stream;
  gs_tileplan t;
  t.R = R;
  t.nblocks = (n + R - 1) / R;
  if (nnz == 0 || n == 0) {
    *out = t;
    return GS_OK;
  }
  DevBuf<int> rowof, head, rid, rstart, rend, rblock, rlen, gbase, bfirst, bslots, nuniq;
  DevBuf<unsigned long long> keys, keys2, uk;
  GS_CUDA(ctx, rowof.alloc(nnz, s));
  GS_CUDA(ctx, keys.alloc(nnz, s));
  GS_CUDA(ctx, keys2.alloc(nnz, s));
  GS_CUDA(ctx, uk.alloc(nnz, s));
  GS_CUDA(ctx, nuniq.alloc(1, s));
  gs_launch_begin(ctx, 1);
  k_entry_rows<<<nblk(n), kThreads, 0, s>>>(g->offs, n, rowof.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_block_keys<<<nblk(nnz), kThreads, 0, s>>>(rowof.get(), g->cols, nnz, R, keys.get());
  gs_launch_end(ctx, 1);
  {
    size_t tb1 = 0, tb2 = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb1, keys.get(), keys2.get(), (int)nnz, 0, 64, s);
    cub::DeviceSelect::Unique(nullptr, tb2, keys2.get(), uk.get(), nuniq.get(), (int)nnz, s);
    DevBuf<unsigned char> tmp;
    GS_CUDA(ctx, tmp.alloc(std::max(tb1, tb2), s));
    cub::DeviceRadixSort::SortKeys(tmp.get(), tb1, keys.get(), keys2.get(), (int)nnz, 0, 64, s);
    cub::DeviceSelect::Unique(tmp.get(), tb2, keys2.get(), uk.get(), nuniq.get(), (int)nnz, s);
  }
  int m = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&m, nuniq.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  GS_CUDA(ctx, head.alloc(m, s));
  GS_CUDA(ctx, rid.alloc(m, s));
  gs_launch_begin(ctx, 1);
  k_run_heads<<<nblk(m), kThreads, 0, s>>>(uk.get(), m, head.get());
  gs_launch_end(ctx, 1);
  {
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, head.get(), rid.get(), m, s);
    DevBuf<unsigned char> tmp;
    GS_CUDA(ctx, tmp.alloc(tb, s));
    cub::DeviceScan::InclusiveSum(tmp.get(), tb, head.get(), rid.get(), m, s);
  }
  int nruns = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&nruns, rid.get() + m - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  GS_CUDA(ctx, rend.alloc(nruns, s));
  GS_CUDA(ctx, rblock.alloc(nruns, s));
  GS_CUDA(ctx, gbase.alloc(nruns, s));
  cudaError_t e = cudaMalloc((void**)&t.rstart, nruns * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc((void**)&t.rlen, nruns * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc((void**)&t.lbase, nruns * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc((void**)&t.bfirst, t.nblocks * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc((void**)&t.bcount, t.nblocks * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc((void**)&t.slot, nnz * sizeof(unsigned short));
  if (e != cudaSuccess) {
    gs_tiles_release(t);
    return gs_cuda_fail(ctx, e, "tile plan allocation");
  }
  GS_CUDA(ctx, bslots.alloc(t.nblocks, s));
  GS_CUDA(ctx, cudaMemsetAsync(t.bfirst, 0xFF, t.nblocks * sizeof(int), s));
  gs_launch_begin(ctx, 1);
  k_run_bounds<<<nblk(m), kThreads, 0, s>>>(uk.get(), rid.get(), m, t.rstart, rend.get(), rblock.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_run_len<<<nblk(nruns), kThreads, 0, s>>>(t.rstart, rend.get(), nruns, t.rlen);
  gs_launch_end(ctx, 1);
  {
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, t.rlen, gbase.get(), nruns, s);
    DevBuf<unsigned char> tmp;
    GS_CUDA(ctx, tmp.alloc(tb, s));
    cub::DeviceScan::ExclusiveSum(tmp.get(), tb, t.rlen, gbase.get(), nruns, s);
  }
  gs_launch_begin(ctx, 1);
  k_block_first<<<nblk(nruns), kThreads, 0, s>>>(rblock.get(), nruns, t.bfirst);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_block_ranges<<<nblk(t.nblocks), kThreads, 0, s>>>(t.bfirst, rblock.get(), gbase.get(), t.rlen,
                                                       t.nblocks, nruns, t.bcount, bslots.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_run_lbase<<<nblk(nruns), kThreads, 0, s>>>(rblock.get(), t.bfirst, gbase.get(), nruns, t.lbase);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_entry_slots<<<nblk(nnz), kThreads, 0, s>>>(rowof.get(), g->cols, nnz, R, t.bfirst, t.bcount,
                                                 t.rstart, rend.get(), t.lbase, t.slot);
  gs_launch_end(ctx, 1);
  std::vector<int> hs(t.nblocks), hc(t.nblocks);
  GS_CUDA(ctx, cudaMemcpyAsync(hs.data(), bslots.get(), t.nblocks * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(hc.data(), t.bcount, t.nblocks * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  t.max_slots = 0;
  t.max_runs = 0;
  int64_t tot = 0;
  for (int b = 0; b < t.nblocks; ++b) {
    t.max_slots = std::max(t.max_slots, hs[b]);
    t.max_runs = std::max(t.max_runs, hc[b]);
    tot += hs[b];
  }
  t.mean_slots = t.nblocks ? (double)tot / t.nblocks : 0.0;
  t.nruns = nruns;
  *out = t;
  return GS_OK;
}
