// gs_part.cu -- row partitions of a filter for the multi-GPU row-partitioned path (SURVEY.md
// §8(e) "Row partitioning (config 3)"). The reference has no multi-process path; this splits the
// Chebyshev products of HeatFilter::apply (proj/src/heat.cpp:116-131) by rows, so each product
// needs T_{k-1} at the halo rows only, exchanged once per step (gs_cheb.cu, run_apply_part).
//
// Every rank builds its own partition from the same (replicated, deterministic) filter, so the
// halo and send lists agree without communication: the operator is structurally symmetric
// (sparse.cpp:40-44), hence rank q's halo rows owned by p are exactly p's rows adjacent to q's
// range, and both sides list them in ascending position order.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <memory>

#include "gs_internal.cuh"
#include "geosink_b200.h"

namespace {

constexpr int kT = 256;

inline unsigned blocks_for(int64_t work) { return (unsigned)((work + kT - 1) / kT); }

// bounds[p] = first row whose CSR offset reaches p * nnz / nparts (nnz-balanced ranges)
__global__ void k_bounds(const int* __restrict__ offs, int n, int64_t nnz, int nparts, int* out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > nparts) return;
  if (p == 0 || p == nparts) {
    out[p] = p == 0 ? 0 : n;
    return;
  }
  const int64_t target = nnz * p / nparts;
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((int64_t)offs[mid] >= target) hi = mid;
    else lo = mid + 1;
  }
  out[p] = lo;
}

__device__ __forceinline__ int owner_of(const int* __restrict__ bounds, int nparts, int c) {
  int lo = 0, hi = nparts - 1;  // largest p with bounds[p] <= c
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bounds[mid] <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void k_local_offs(const int* __restrict__ offs, int rb, int nl, int* __restrict__ out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r <= nl) out[r] = offs[rb + r] - offs[rb];
}

// halo candidates: columns outside [rb, re) (INT_MAX otherwise)
__global__ void k_halo_keys(const int* __restrict__ cols, int64_t e0, int64_t m, int rb, int re,
                            int* __restrict__ keys) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int c = cols[e0 + e];
  keys[e] = (c < rb || c >= re) ? c : INT_MAX;
}

__global__ void k_remap(const int* __restrict__ cols, int64_t e0, int64_t m, int rb, int re, int nl,
                        const int* __restrict__ halo, int nh, int* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int c = cols[e0 + e];
  if (c >= rb && c < re) {
    out[e] = c - rb;
    return;
  }
  int lo = 0, hi = nh;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (halo[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  out[e] = nl + lo;
}

// (owner << 32 | local row) for every entry whose column another rank owns (~0 otherwise)
__global__ void k_send_keys(const int* __restrict__ offs, const int* __restrict__ cols, int rb, int re,
                            int nl, const int* __restrict__ bounds, int nparts,
                            unsigned long long* __restrict__ keys) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nl) return;
  const int e0 = offs[rb];
  for (int p = offs[rb + r]; p < offs[rb + r + 1]; ++p) {
    const int c = cols[p];
    keys[p - e0] = (c < rb || c >= re)
                       ? ((unsigned long long)owner_of(bounds, nparts, c) << 32) | (unsigned)r
                       : ~0ull;
  }
}

// boundary rows (reading a halo row): the largest one in the first half, the smallest in the second
__global__ void k_boundary_rows(const int* __restrict__ offs, const int* __restrict__ cols, int nl,
                                int* lo_max, int* hi_min) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nl) return;
  bool b = false;
  for (int p = offs[r]; p < offs[r + 1] && !b; ++p) b = cols[p] >= nl;
  if (!b) return;
  if (r < nl / 2) atomicMax(lo_max, r);
  else atomicMin(hi_min, r);
}

__global__ void k_low32(const unsigned long long* __restrict__ k, int m, int* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = (int)(k[i] & 0xFFFFFFFFull);
}

__global__ void k_float_slice(const float* __restrict__ src, int64_t m, float* __restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < m) dst[e] = src[e];
}

struct NotIntMax {
  __device__ bool operator()(int v) const { return v != INT_MAX; }
};
struct NotAllOnes {
  __device__ bool operator()(unsigned long long v) const { return v != ~0ull; }
};

// sorted unique values of keys[0..m) that pass `pred` -> out (device), count -> *count
template <class K, class Pred>
int select_sort_unique(gs_ctx* ctx, const K* keys, int64_t m, Pred pred, DevBuf<K>& out, int* count) {
  cudaStream_t s = ctx->stream;
  DevBuf<K> sel, sorted;
  DevBuf<int> nsel;
  GS_CUDA(ctx, sel.alloc(m, s));
  GS_CUDA(ctx, nsel.alloc(1, s));
  size_t tb = 0;
  GS_CUDA(ctx, cub::DeviceSelect::If(nullptr, tb, keys, sel.get(), nsel.get(), (int)m, pred, s));
  DevBuf<unsigned char> tmp;
  GS_CUDA(ctx, tmp.alloc(tb, s));
  GS_CUDA(ctx, cub::DeviceSelect::If(tmp.get(), tb, keys, sel.get(), nsel.get(), (int)m, pred, s));
  int k = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&k, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  GS_CUDA(ctx, sorted.alloc(k, s));
  GS_CUDA(ctx, out.alloc(k, s));
  if (k > 0) {
    size_t t1 = 0, t2 = 0;
    GS_CUDA(ctx, cub::DeviceRadixSort::SortKeys(nullptr, t1, sel.get(), sorted.get(), k, 0, (int)sizeof(K) * 8, s));
    GS_CUDA(ctx, cub::DeviceSelect::Unique(nullptr, t2, sorted.get(), out.get(), nsel.get(), k, s));
    GS_CUDA(ctx, tmp.alloc(t1 > t2 ? t1 : t2, s));
    GS_CUDA(ctx, cub::DeviceRadixSort::SortKeys(tmp.get(), t1, sel.get(), sorted.get(), k, 0, (int)sizeof(K) * 8, s));
    GS_CUDA(ctx, cub::DeviceSelect::Unique(tmp.get(), t2, sorted.get(), out.get(), nsel.get(), k, s));
    GS_CUDA(ctx, cudaMemcpyAsync(&k, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
  }
  *count = k;
  return GS_OK;
}

int part_build(gs_ctx* ctx, const gs_filter* f, int nparts, int part, gs_part* P) {
  cudaStream_t s = ctx->stream;
  const gs_layout& L = f->lay[0];
  const gs_graph* g = L.perm;
  const int n = g->n;
  P->f = f;
  P->nparts = nparts;
  P->part = part;
  P->n_global = n;
  // ---- ranges ------------------------------------------------------------------------------
  DevBuf<int> dbounds;
  GS_CUDA(ctx, dbounds.alloc(nparts + 1, s));
  gs_launch_begin(ctx, 1);
  k_bounds<<<blocks_for(nparts + 1), kT, 0, s>>>(g->offs, n, g->nnz, nparts, dbounds.get());
  gs_launch_end(ctx, 1);
  P->bounds.resize(nparts + 1);
  GS_CUDA(ctx, cudaMemcpyAsync(P->bounds.data(), dbounds.get(), (nparts + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  const int rb = P->bounds[part], re = P->bounds[part + 1];
  P->row_begin = rb;
  P->row_end = re;
  P->nl = re - rb;
  int eb = 0, ee = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&eb, g->offs + rb, sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaMemcpyAsync(&ee, g->offs + re, sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  const int64_t m = (int64_t)ee - eb;
  const int nl = P->nl;
  // ---- local CSR: offsets, halo list, renumbered columns, values ------------------------------
  GS_TRY(gs_graph_alloc(ctx, nl, m, &P->local));
  gs_launch_begin(ctx, 1);
  k_local_offs<<<blocks_for(nl + 1), kT, 0, s>>>(g->offs, rb, nl, P->local->offs);
  gs_launch_end(ctx, 1);
  DevBuf<int> hkeys, halo;
  GS_CUDA(ctx, hkeys.alloc(m, s));
  if (m > 0) {
    gs_launch_begin(ctx, 1);
    k_halo_keys<<<blocks_for(m), kT, 0, s>>>(g->cols, eb, m, rb, re, hkeys.get());
    gs_launch_end(ctx, 1);
  }
  GS_TRY(select_sort_unique<int>(ctx, hkeys.get(), m, NotIntMax(), halo, &P->nh));
  if (m > 0) {
    gs_launch_begin(ctx, 1);
    k_remap<<<blocks_for(m), kT, 0, s>>>(g->cols, eb, m, rb, re, nl, halo.get(), P->nh, P->local->cols);
    gs_launch_end(ctx, 1);
    GS_CUDA(ctx, cudaMemcpyAsync(P->local->vals, g->vals + eb, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  {  // interior rows: between the last boundary row of the first half and the first of the second
    DevBuf<int> lh;
    GS_CUDA(ctx, lh.alloc(2, s));
    const int init[2] = {-1, nl};
    GS_CUDA(ctx, cudaMemcpyAsync(lh.get(), init, sizeof init, cudaMemcpyHostToDevice, s));
    if (nl > 0) {
      gs_launch_begin(ctx, 1);
      k_boundary_rows<<<blocks_for(nl), kT, 0, s>>>(P->local->offs, P->local->cols, nl, lh.get(), lh.get() + 1);
      gs_launch_end(ctx, 1);
    }
    int hb[2];
    GS_CUDA(ctx, cudaMemcpyAsync(hb, lh.get(), sizeof hb, cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    P->int_lo = hb[0] + 1;
    P->int_hi = hb[1] < P->int_lo ? P->int_lo : hb[1];
  }
  GS_CUDA(ctx, cudaMalloc((void**)&P->vals32, (size_t)(m + kCsrPad) * sizeof(float)));
  if (m > 0 && L.vals32) {
    gs_launch_begin(ctx, 1);
    k_float_slice<<<blocks_for(m), kT, 0, s>>>(L.vals32 + eb, m, P->vals32);
    gs_launch_end(ctx, 1);
  }
  GS_CUDA(ctx, cudaMalloc((void**)&P->vertices, (size_t)(nl ? nl : 1) * sizeof(int)));
  if (nl > 0)
    GS_CUDA(ctx, cudaMemcpyAsync(P->vertices, L.order + rb, (size_t)nl * sizeof(int), cudaMemcpyDeviceToDevice, s));
  // ---- receive counts per owner (halo is sorted by position, hence by owner) ---------------------
  P->recv_counts.assign(nparts, 0);
  if (P->nh > 0) {
    std::vector<int> hh(P->nh);
    GS_CUDA(ctx, cudaMemcpyAsync(hh.data(), halo.get(), P->nh * sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    for (int c : hh) {
      const int q = (int)(std::upper_bound(P->bounds.begin(), P->bounds.end(), c) - P->bounds.begin()) - 1;
      P->recv_counts[q] += 1;
    }
  }
  // ---- send lists --------------------------------------------------------------------------
  DevBuf<unsigned long long> skeys, sends;
  GS_CUDA(ctx, skeys.alloc(m, s));
  if (nl > 0) {
    gs_launch_begin(ctx, 1);
    k_send_keys<<<blocks_for(nl), kT, 0, s>>>(g->offs, g->cols, rb, re, nl, dbounds.get(), nparts, skeys.get());
    gs_launch_end(ctx, 1);
  }
  GS_TRY(select_sort_unique<unsigned long long>(ctx, skeys.get(), m, NotAllOnes(), sends, &P->ns));
  P->send_counts.assign(nparts, 0);
  GS_CUDA(ctx, cudaMalloc((void**)&P->send_rows, (size_t)(P->ns ? P->ns : 1) * sizeof(int)));
  if (P->ns > 0) {
    std::vector<unsigned long long> hs(P->ns);
    GS_CUDA(ctx, cudaMemcpyAsync(hs.data(), sends.get(), P->ns * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    gs_launch_begin(ctx, 1);
    k_low32<<<blocks_for(P->ns), kT, 0, s>>>(sends.get(), P->ns, P->send_rows);
    gs_launch_end(ctx, 1);
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    for (unsigned long long k : hs) P->send_counts[(int)(k >> 32)] += 1;
  }
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  return GS_OK;
}

}  // namespace

extern "C" int gs_part_create(gs_ctx* ctx, const gs_filter* f, int nparts, int part, gs_part** out) {
  if (!ctx || !f || !out) return GS_ERR_UNSUPPORTED;
  if (nparts < 1 || part < 0 || part >= nparts)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "partition index out of range");
  std::unique_ptr<gs_part> P(new gs_part());
  const int rc = part_build(ctx, f, nparts, part, P.get());
  if (rc) {
    gs_part_destroy(P.release());
    return rc;
  }
  *out = P.release();
  return GS_OK;
}

extern "C" void gs_part_destroy(gs_part* p) {
  if (!p) return;
  gs_graph_destroy(p->local);
  cudaFree(p->vals32);
  gs_lanepad_destroy(p->lanepad[0]);
  gs_lanepad_destroy(p->lanepad[1]);
  cudaFree(p->vertices);
  cudaFree(p->send_rows);
  delete p;
}

extern "C" int gs_part_info(const gs_part* p, int* row_begin, int* row_end, int* n_halo,
                            int64_t* nnz_local, int* n_send) {
  if (!p) return GS_ERR_UNSUPPORTED;
  if (row_begin) *row_begin = p->row_begin;
  if (row_end) *row_end = p->row_end;
  if (n_halo) *n_halo = p->nh;
  if (nnz_local) *nnz_local = p->local ? p->local->nnz : 0;
  if (n_send) *n_send = p->ns;
  return GS_OK;
}

extern "C" int gs_part_interior(const gs_part* p, int* lo, int* hi) {
  if (!p) return GS_ERR_UNSUPPORTED;
  if (lo) *lo = p->int_lo;
  if (hi) *hi = p->int_hi;
  return GS_OK;
}

extern "C" int gs_part_counts(const gs_part* p, int64_t* send_counts, int64_t* recv_counts) {
  if (!p) return GS_ERR_UNSUPPORTED;
  for (int q = 0; q < p->nparts; ++q) {
    if (send_counts) send_counts[q] = p->send_counts[q];
    if (recv_counts) recv_counts[q] = p->recv_counts[q];
  }
  return GS_OK;
}

extern "C" int gs_part_vertices(gs_ctx* ctx, const gs_part* p, int* out, int mem) {
  if (!p || !out) return GS_ERR_UNSUPPORTED;
  return gs_copy_out(ctx, out, p->vertices, (size_t)p->nl * sizeof(int), mem);
}
