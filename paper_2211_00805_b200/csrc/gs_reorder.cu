// gs_reorder.cu -- locality ordering of the filter's vertices (device BFS, Cuthill-McKee style).
//
// The reference keeps vertices in input order (SparseSymMatrix rows, sparse.hpp:23-61); a
// randomly ordered point cloud then makes every neighbour gather of the Chebyshev step a random
// 64-byte access. The filter therefore stores L_s with rows renumbered by BFS level (component by
// component, each from a pseudo-peripheral start), so neighbours sit within about two level
// widths of each other and gathers hit L1/L2. The reference's permutation-invariance test
// (tests/test_transport.cpp:287-321) licenses the relabelling; here it is also exact: each
// renumbered row keeps its entries in the ORIGINAL column order, so every per-vertex value is
// bit-identical to the unpermuted recurrence. Inputs are gathered through `order` when packed
// and results scattered back through it when unpacked.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "gs_internal.cuh"

namespace {

constexpr int kThreads = 256;

inline unsigned nblk(int64_t m, int t = kThreads) { return (unsigned)((m + t - 1) / t); }

__global__ void k_fill_int(int* x, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

__global__ void k_first_unvisited(const int* level, int n, int* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && level[i] < 0) atomicMin(out, i);
}

// one BFS level: vertices at level L mark unvisited neighbours L+1 (benign identical writes)
__global__ void k_bfs_expand(const int* __restrict__ offs, const int* __restrict__ cols,
                             int* __restrict__ level, int n, int L, int* any) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || level[i] != L) return;
  bool grew = false;
  for (int p = offs[i]; p < offs[i + 1]; ++p) {
    const int j = cols[p];
    if (level[j] < 0) {
      level[j] = L + 1;
      grew = true;
    }
  }
  if (grew) *any = 1;
}

__global__ void k_tag_component(const int* level, int* comp, int n, int c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && level[i] >= 0 && comp[i] == -1) comp[i] = c;
}

__global__ void k_min_at_level(const int* level, const int* comp, int n, int c, int L, int* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && comp[i] == c && level[i] == L) atomicMin(out, i);
}

__global__ void k_reset_component(int* level, const int* comp, int n, int c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && comp[i] == c) level[i] = -1;
}

__global__ void k_set(int* x, int i, int v) { x[i] = v; }

// vertices without off-diagonal neighbours are their own components; they are ordered last
__global__ void k_mark_isolated(const int* offs, const int* cols, int n, int* level, int* comp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int p = offs[i]; p < offs[i + 1]; ++p)
    if (cols[p] != i) return;
  level[i] = 0;
  comp[i] = -2;
}

__global__ void k_order_keys(const int* level, const int* comp, const long long* base, int n,
                             int ncomp, unsigned long long* keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = comp[i] >= 0 ? comp[i] : ncomp;  // isolated vertices after every component
  const unsigned long long rank = (unsigned long long)(base[c] + level[i]);
  keys[i] = (rank << 32) | (unsigned)i;
}

__global__ void k_order_from_keys(const unsigned long long* keys, int n, int* order, int* newpos) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int old = (int)(keys[r] & 0xFFFFFFFFull);
  order[r] = old;
  newpos[old] = r;
}

__global__ void k_perm_rowlen(const int* offs, const int* order, int n, int* len) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) {
    const int o = order[r];
    len[r] = offs[o + 1] - offs[o];
  }
}

// permuted CSR: row r = old row order[r], entries in their original order, columns renumbered
__global__ void k_perm_fill(const int* __restrict__ offs, const int* __restrict__ cols,
                            const double* __restrict__ vals, const int* __restrict__ order,
                            const int* __restrict__ newpos, const int* __restrict__ noffs, int n,
                            int* __restrict__ ncols, double* __restrict__ nvals) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int o = order[r];
  int q = noffs[r];
  for (int p = offs[o]; p < offs[o + 1]; ++p, ++q) {
    ncols[q] = newpos[cols[p]];
    nvals[q] = vals[p];
  }
}

// global level of each vertex (component base + BFS level; isolated block last)
__global__ void k_global_level(const int* level, const int* comp, const long long* base, int n,
                               int ncomp, int* gl) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = comp[i] >= 0 ? comp[i] : ncomp;
  gl[i] = (int)(base[c] + level[i]);
}

__global__ void k_level_keys(const int* gl, int n, unsigned long long* keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = ((unsigned long long)(unsigned)gl[i] << 32) | (unsigned)i;
}

// Cuthill-McKee key of the vertices of global level G: the smallest position among their
// neighbours on level G-1 (vertices starting a component have none and keep their index order).
__global__ void k_cm_keys(const unsigned long long* bylevel, int start, int cnt,
                          const int* __restrict__ offs, const int* __restrict__ cols,
                          const int* __restrict__ gl, const int* __restrict__ pos, int G,
                          unsigned long long* keys) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int v = (int)(bylevel[start + t] & 0xFFFFFFFFull);
  unsigned best = 0xFFFFFFFFu;
  for (int p = offs[v]; p < offs[v + 1]; ++p) {
    const int u = cols[p];
    if (gl[u] == G - 1) best = min(best, (unsigned)pos[u]);
  }
  keys[t] = ((unsigned long long)best << 32) | (unsigned)v;
}

__global__ void k_cm_assign(const unsigned long long* sorted, int start, int cnt, int* pos) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < cnt) pos[(int)(sorted[t] & 0xFFFFFFFFull)] = start + t;
}

// SELL-C-sigma style: within windows of `sigma` consecutive CM positions, rows are ordered by
// length (longest first), so rows that share a warp (narrow column groups) have similar lengths.
__global__ void k_sigma_keys(const int* pos, const int* offs, int n, int sigma,
                             unsigned long long* keys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = pos[i];
  const unsigned len = (unsigned)min(offs[i + 1] - offs[i], (1 << 20) - 1);
  const unsigned long long win = (unsigned long long)(p / sigma);
  keys[i] = (win << 44) | ((unsigned long long)((1u << 20) - 1u - len) << 24) |
            (unsigned long long)(p % sigma);
}

__global__ void k_sigma_assign(const unsigned long long* sorted_keys, const int* sorted_vertex, int n,
                               int* pos) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) pos[sorted_vertex[r]] = r;
}

__global__ void k_iota(int* x, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = i;
}

__global__ void k_pos_to_order(const int* pos, int n, int* order, int* newpos) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  newpos[i] = pos[i];
  order[pos[i]] = i;
}

}  // namespace

// Computes order[new] = old and newpos[old] = new on the device.
int gs_bfs_order(gs_ctx* ctx, const gs_graph* g, int* d_order, int* d_newpos, int sigma,
                 int* d_order_sig, int* d_newpos_sig) {
  const int n = g->n;
  if (n == 0) return GS_OK;
  cudaStream_t s = ctx->stream;
  DevBuf<int> level, comp, scal, any;
  GS_CUDA(ctx, level.alloc(n, s));
  GS_CUDA(ctx, comp.alloc(n, s));
  GS_CUDA(ctx, scal.alloc(1, s));
  GS_CUDA(ctx, any.alloc(256, s));
  gs_launch_begin(ctx, 1);
  k_fill_int<<<nblk(n), kThreads, 0, s>>>(level.get(), n, -1);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_fill_int<<<nblk(n), kThreads, 0, s>>>(comp.get(), n, -1);
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_mark_isolated<<<nblk(n), kThreads, 0, s>>>(g->offs, g->cols, n, level.get(), comp.get());
  gs_launch_end(ctx, 1);
  const int BIG = 0x7fffffff;
  std::vector<long long> depth;  // levels per component
  int hint_unvisited = 0;
  (void)hint_unvisited;
  auto bfs = [&](int start) -> int {  // returns last level index
    gs_launch_begin(ctx, 1);
    k_set<<<1, 1, 0, s>>>(level.get(), start, 0);
    gs_launch_end(ctx, 1);
    int L = 0;
    const int batch = 64;
    std::vector<int> h(batch);
    for (;;) {
      cudaMemsetAsync(any.get(), 0, batch * sizeof(int), s);
      for (int q = 0; q < batch; ++q) {
        gs_launch_begin(ctx, 1);
        k_bfs_expand<<<nblk(n), kThreads, 0, s>>>(g->offs, g->cols, level.get(), n, L + q, any.get() + q);
        gs_launch_end(ctx, 1);
      }
      cudaMemcpyAsync(h.data(), any.get(), batch * sizeof(int), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      int q = 0;
      while (q < batch && h[q]) ++q;
      if (q < batch) return L + q;  // level L+q expanded nothing: it is the last level
      L += batch;
    }
  };
  for (int c = 0;; ++c) {
    int first = BIG;
    GS_CUDA(ctx, cudaMemcpyAsync(scal.get(), &first, sizeof(int), cudaMemcpyHostToDevice, s));
    gs_launch_begin(ctx, 1);
    k_first_unvisited<<<nblk(n), kThreads, 0, s>>>(level.get(), n, scal.get());
    gs_launch_end(ctx, 1);
    GS_CUDA(ctx, cudaMemcpyAsync(&first, scal.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    if (first == BIG) break;
    int last = bfs(first);
    gs_launch_begin(ctx, 1);
    k_tag_component<<<nblk(n), kThreads, 0, s>>>(level.get(), comp.get(), n, c);
    gs_launch_end(ctx, 1);
    if (last > 0) {  // pseudo-peripheral restart from the lowest-index vertex of the last level
      int p = BIG;
      GS_CUDA(ctx, cudaMemcpyAsync(scal.get(), &p, sizeof(int), cudaMemcpyHostToDevice, s));
      gs_launch_begin(ctx, 1);
      k_min_at_level<<<nblk(n), kThreads, 0, s>>>(level.get(), comp.get(), n, c, last, scal.get());
      gs_launch_end(ctx, 1);
      GS_CUDA(ctx, cudaMemcpyAsync(&p, scal.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
      GS_CUDA(ctx, cudaStreamSynchronize(s));
      gs_launch_begin(ctx, 1);
      k_reset_component<<<nblk(n), kThreads, 0, s>>>(level.get(), comp.get(), n, c);
      gs_launch_end(ctx, 1);
      last = bfs(p);
    }
    depth.push_back(last + 1);
  }
  depth.push_back(1);  // the isolated-vertex block
  std::vector<long long> base(depth.size() + 1, 0);
  for (size_t c = 0; c < depth.size(); ++c) base[c + 1] = base[c] + depth[c];
  const int ncomp = (int)depth.size() - 1;
  DevBuf<long long> dbase;
  DevBuf<unsigned long long> keys, keys2, lk, lk2;
  DevBuf<int> gl, pos;
  GS_CUDA(ctx, dbase.alloc(base.size(), s));
  GS_CUDA(ctx, keys.alloc(n, s));
  GS_CUDA(ctx, keys2.alloc(n, s));
  GS_CUDA(ctx, gl.alloc(n, s));
  GS_CUDA(ctx, pos.alloc(n, s));
  GS_CUDA(ctx, cudaMemcpyAsync(dbase.get(), base.data(), base.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  gs_launch_begin(ctx, 1);
  k_global_level<<<nblk(n), kThreads, 0, s>>>(level.get(), comp.get(), dbase.get(), n, ncomp, gl.get());
  gs_launch_end(ctx, 1);
  gs_launch_begin(ctx, 1);
  k_level_keys<<<nblk(n), kThreads, 0, s>>>(gl.get(), n, keys.get());
  gs_launch_end(ctx, 1);
  {
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.get(), keys2.get(), n, 0, 64, s);
    DevBuf<unsigned char> tmp;
    GS_CUDA(ctx, tmp.alloc(tb, s));
    cub::DeviceRadixSort::SortKeys(tmp.get(), tb, keys.get(), keys2.get(), n, 0, 64, s);
  }
  // level start offsets (host): histogram of global levels
  const int nlev = (int)base.back();
  std::vector<int> hgl(n), cnt(nlev + 1, 0);
  GS_CUDA(ctx, cudaMemcpyAsync(hgl.data(), gl.get(), n * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  for (int i = 0; i < n; ++i) cnt[hgl[i]]++;
  std::vector<int> lstart(nlev + 1, 0);
  for (int G = 0; G < nlev; ++G) lstart[G + 1] = lstart[G] + cnt[G];
  int maxcnt = 1;
  for (int G = 0; G < nlev; ++G) maxcnt = std::max(maxcnt, cnt[G]);
  GS_CUDA(ctx, lk.alloc(maxcnt, s));
  GS_CUDA(ctx, lk2.alloc(maxcnt, s));
  size_t tb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb, lk.get(), lk2.get(), maxcnt, 0, 64, s);
  DevBuf<unsigned char> tmp;
  GS_CUDA(ctx, tmp.alloc(tb, s));
  // levels in order; each level sorted by (min parent position, index)
  for (int G = 0; G < nlev; ++G) {
    const int c = cnt[G];
    if (c == 0) continue;
    gs_launch_begin(ctx, 1);
    k_cm_keys<<<nblk(c), kThreads, 0, s>>>(keys2.get(), lstart[G], c, g->offs, g->cols, gl.get(),
                                            pos.get(), G, lk.get());
    gs_launch_end(ctx, 1);
    size_t tb2 = tb;
    cub::DeviceRadixSort::SortKeys(tmp.get(), tb2, lk.get(), lk2.get(), c, 0, 64, s);
    gs_launch_begin(ctx, 1);
    k_cm_assign<<<nblk(c), kThreads, 0, s>>>(lk2.get(), lstart[G], c, pos.get());
    gs_launch_end(ctx, 1);
  }
  gs_launch_begin(ctx, 1);
  k_pos_to_order<<<nblk(n), kThreads, 0, s>>>(pos.get(), n, d_order, d_newpos);
  gs_launch_end(ctx, 1);
  // second layout: degree-sorted windows of `sigma` CM positions (narrow column groups)
  if (d_order_sig && sigma > 1) {
    GS_TRY(gs_sigma_order(ctx, g, d_newpos, sigma, d_order_sig, d_newpos_sig));
  } else if (d_order_sig) {
    cudaMemcpyAsync(d_order_sig, d_order, n * sizeof(int), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(d_newpos_sig, d_newpos, n * sizeof(int), cudaMemcpyDeviceToDevice, s);
  }
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// Degree-sorted windows of `sigma` positions of an existing order (d_newpos[old] = position):
// inside each window rows go longest first (SELL-C-sigma style), ties in position order.
int gs_sigma_order(gs_ctx* ctx, const gs_graph* g, const int* d_newpos, int sigma, int* d_order_sig,
                   int* d_newpos_sig) {
  const int n = g->n;
  if (n == 0) return GS_OK;
  cudaStream_t s = ctx->stream;
  DevBuf<int> pos;
  GS_CUDA(ctx, pos.alloc(n, s));
  GS_CUDA(ctx, cudaMemcpyAsync(pos.get(), d_newpos, (size_t)n * sizeof(int), cudaMemcpyDeviceToDevice, s));
  {
    DevBuf<unsigned long long> sk, sk2;
    DevBuf<int> vid, vid2;
    GS_CUDA(ctx, sk.alloc(n, s));
    GS_CUDA(ctx, sk2.alloc(n, s));
    GS_CUDA(ctx, vid.alloc(n, s));
    GS_CUDA(ctx, vid2.alloc(n, s));
    gs_launch_begin(ctx, 1);
    k_sigma_keys<<<nblk(n), kThreads, 0, s>>>(pos.get(), g->offs, n, sigma, sk.get());
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_iota<<<nblk(n), kThreads, 0, s>>>(vid.get(), n);
    gs_launch_end(ctx, 1);
    size_t tb3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb3, sk.get(), sk2.get(), vid.get(), vid2.get(), n, 0, 64, s);
    DevBuf<unsigned char> tmp3;
    GS_CUDA(ctx, tmp3.alloc(tb3, s));
    cub::DeviceRadixSort::SortPairs(tmp3.get(), tb3, sk.get(), sk2.get(), vid.get(), vid2.get(), n, 0, 64, s);
    gs_launch_begin(ctx, 1);
    k_sigma_assign<<<nblk(n), kThreads, 0, s>>>(sk2.get(), vid2.get(), n, pos.get());
    gs_launch_end(ctx, 1);
    gs_launch_begin(ctx, 1);
    k_pos_to_order<<<nblk(n), kThreads, 0, s>>>(pos.get(), n, d_order_sig, d_newpos_sig);
    gs_launch_end(ctx, 1);
  }
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

// Renumbered copy of g (rows in `order`, entries in original order).
int gs_permute_graph(gs_ctx* ctx, const gs_graph* g, const int* d_order, const int* d_newpos,
                     gs_graph** out) {
  const int n = g->n;
  cudaStream_t s = ctx->stream;
  gs_graph* p = nullptr;
  GS_TRY(gs_graph_alloc(ctx, n, g->nnz, &p));
  DevBuf<int> len;
  GS_CUDA(ctx, len.alloc(n + 1, s));
  GS_CUDA(ctx, cudaMemsetAsync(len.get(), 0, (n + 1) * sizeof(int), s));
  if (n > 0) {
    gs_launch_begin(ctx, 1);
    k_perm_rowlen<<<nblk(n), kThreads, 0, s>>>(g->offs, d_order, n, len.get());
    gs_launch_end(ctx, 1);
  }
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, len.get(), p->offs, n + 1, s);
  DevBuf<unsigned char> tmp;
  GS_CUDA(ctx, tmp.alloc(tb, s));
  cub::DeviceScan::ExclusiveSum(tmp.get(), tb, len.get(), p->offs, n + 1, s);
  if (n > 0) {
    gs_launch_begin(ctx, 1);
    k_perm_fill<<<nblk(n), kThreads, 0, s>>>(g->offs, g->cols, g->vals, d_order, d_newpos, p->offs,
                                              n, p->cols, p->vals);
    gs_launch_end(ctx, 1);
  }
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    gs_graph_destroy(p);
    return gs_cuda_fail(ctx, e, "permute graph");
  }
  *out = p;
  return GS_OK;
}
