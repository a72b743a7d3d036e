// gs_win.cu -- host side of the windowed Chebyshev step (gs_win.cuh): the window layout's vertex
// order (recursive BFS bisection), the per-CTA ring schedule, its device copy and the TMA tensor
// maps of the Chebyshev vectors.
//
// Reference path: the layout only renumbers rows of L_s (heat.cpp:72-96's scaled Laplacian); every
// row keeps its CSR entries in the original column order (gs_permute_graph), so the recurrence
// (heat.cpp:121-130) and its fma chains are unchanged and results stay bit-identical.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "gs_internal.cuh"
#include "gs_win.cuh"

using gsk::WinBlk;

namespace {

// Recursive BFS bisection (graph only): each part is ordered by BFS from a pseudo-peripheral
// vertex (two BFS sweeps; components one after another), split at the median, and both halves
// recurse; parts of at most `leaf` vertices are emitted in their BFS order. Consecutive vertices
// are then compact patches of the graph at every scale, so a CTA's contiguous range is a patch
// and its row blocks reuse each other's neighbour rows (SURVEY §8(d) gather model).
void bisect_order(int n, const int* offs, const int* cols, int leaf, std::vector<int>& order) {
  order.clear();
  order.reserve(n);
  std::vector<int> seq(n), tmp(n), label(n, 0), vis(n, 0), queue(n);
  std::iota(seq.begin(), seq.end(), 0);
  int stamp = 0, next_label = 1;
  struct Part { int b, e, lab; };
  std::vector<Part> stack{{0, n, 0}};
  auto bfs = [&](int src, int lab, int* out) {  // returns count; last vertex at out[count-1]
    ++stamp;
    int h = 0, t = 0;
    queue[t++] = src;
    vis[src] = stamp;
    while (h < t) {
      const int u = queue[h++];
      for (int p = offs[u]; p < offs[u + 1]; ++p) {
        const int v = cols[p];
        if (label[v] == lab && vis[v] != stamp) {
          vis[v] = stamp;
          queue[t++] = v;
        }
      }
    }
    if (out) std::copy(queue.begin(), queue.begin() + t, out);
    return t;
  };
  std::vector<int> placed(n, 0);
  int place_stamp = 0;
  while (!stack.empty()) {
    const Part pt = stack.back();
    stack.pop_back();
    const int sz = pt.e - pt.b;
    if (sz <= leaf) {
      for (int i = pt.b; i < pt.e; ++i) order.push_back(seq[i]);
      continue;
    }
    // BFS order of the part, component by component
    ++place_stamp;
    int w = pt.b;
    for (int i = pt.b; i < pt.e; ++i) {
      const int s0 = seq[i];
      if (placed[s0] == place_stamp) continue;
      int cnt = bfs(s0, pt.lab, nullptr);
      int far = queue[cnt - 1];
      cnt = bfs(far, pt.lab, nullptr);
      far = queue[cnt - 1];
      cnt = bfs(far, pt.lab, &tmp[w]);
      for (int k = 0; k < cnt; ++k) placed[tmp[w + k]] = place_stamp;
      w += cnt;
    }
    std::copy(tmp.begin() + pt.b, tmp.begin() + pt.e, seq.begin() + pt.b);
    const int mid = pt.b + sz / 2;
    const int l1 = next_label++, l2 = next_label++;
    for (int i = pt.b; i < mid; ++i) label[seq[i]] = l1;
    for (int i = mid; i < pt.e; ++i) label[seq[i]] = l2;
    stack.push_back({mid, pt.e, l2});
    stack.push_back({pt.b, mid, l1});
  }
}

struct WinHost {
  int W = 0, lmax = 0, nctas = 0;
  std::vector<WinBlk> blk;
  std::vector<int> cta_blk, loads;
  std::vector<int> poffs;  // padded row starts + padding count (gs_win.cuh WinArgs::poffs)
  std::vector<unsigned short> slot, own;
  int64_t entries = 0, padded = 0;
};

// Ring schedule (see gs_win.cuh). Rows [bounds[c], bounds[c+1]) go to CTA c (weight-balanced:
// padded entries + 2 per row). Positions count the CTA's loads; a load at position p lives in
// ring slot p mod W until the load at p + W overwrites it. A block b loads positions
// [P_b, P_b + L_b) (L_b <= LMAX), so it may reuse a position p only if p >= P_b + LMAX + margin - W
// (its own loads never overwrite what it reads; `margin` keeps reuse away from slots about to be
// refilled, which would stall the producer). Before the producer issues block b it waits until
// block wait(b) is consumed: the last block that reads a slot b's loads overwrite, and at least
// b - kWinStages (the metadata stages). Consumers finish blocks in order, so every block up to
// wait(b) is then done. Returns false if one row alone exceeds LMAX loads or EMAX entries (the
// caller keeps the register-gather kernel then).
bool build_schedule(int n, const int* offs, const int* cols, int row_bytes, int elem_bytes, int rows_max,
                    int nctas, WinHost& out) {
  const int W = elem_bytes == 8 ? gsk::win_ring_slots<double>(row_bytes) : gsk::win_ring_slots<float>(row_bytes);
  // loads per block: min(256, W / 4) (512-byte rows: 92 of 368 slots), raised to the largest
  // row's need (its entries + its own row) up to W / 2
  int maxdeg = 0;
  for (int r = 0; r < n; ++r) maxdeg = std::max(maxdeg, offs[r + 1] - offs[r]);
  const int lcap = std::min(gsk::kWinLmaxCap, (W / 2) & ~3);
  const int LMAX = std::min(lcap, std::max(std::min(256, (W / 4) & ~3), ((maxdeg + 1 + 3) & ~3)));
  static const int margin_div = [] {
    const char* e = getenv("GS_WIN_MARGIN_DIV");
    return e ? atoi(e) : 4;
  }();
  const int margin = margin_div > 0 ? (W / margin_div) & ~3 : 0;
  if (getenv("GS_WIN_VERBOSE") && atoi(getenv("GS_WIN_VERBOSE")) != 0)
    fprintf(stderr, "[gs_win] n=%d max degree %d, W=%d, lmax=%d (cap %d) margin=%d\n", n, maxdeg, W, LMAX, lcap,
            margin);
  const int EMAX = gsk::kWinEmax;
  if (W < LMAX + margin + 4 || nctas < 1) return false;
  out.W = W;
  out.lmax = LMAX;
  out.nctas = nctas;
  out.blk.clear();
  out.loads.clear();
  out.cta_blk.assign(nctas + 1, 0);
  const int64_t nnz = offs[n];
  out.entries = nnz;
  // every row padded to whole quads
  std::vector<int64_t> pstart(n + 1, 0);
  for (int r = 0; r < n; ++r) pstart[r + 1] = pstart[r] + (((int64_t)(offs[r + 1] - offs[r]) + 3) & ~3LL);
  if (pstart[n] >= INT32_MAX) return false;
  out.padded = pstart[n];
  out.poffs.assign((size_t)n + 1 + 8, (int)pstart[n]);
  for (int r = 0; r < n; ++r)
    out.poffs[r] = (int)pstart[r] + (int)((pstart[r + 1] - pstart[r]) - (offs[r + 1] - offs[r]));
  out.slot.assign(pstart[n] + 16, 0);
  out.own.assign((size_t)n + 16, 0);
  // weight-balanced contiguous ranges
  std::vector<int> bounds(nctas + 1, n);
  {
    const int64_t total = pstart[n] + 2 * (int64_t)n;
    int r = 0;
    int64_t acc = 0;
    bounds[0] = 0;
    for (int c = 1; c < nctas; ++c) {
      const int64_t target = total * c / nctas;
      while (r < n && acc + (pstart[r + 1] - pstart[r]) + 2 <= target) {
        acc += (pstart[r + 1] - pstart[r]) + 2;
        ++r;
      }
      bounds[c] = r;
    }
    bounds[nctas] = n;
  }
  std::vector<int64_t> last(n, INT64_MIN / 4);
  std::vector<int> rstamp(n, 0);
  std::vector<int> lastref(W);  // per ring slot: the last block (global index) reading it
  int rs = 0;
  int64_t base = 0;
  std::vector<int> rownew;
  std::vector<int> blkloads;
  for (int c = 0; c < nctas; ++c) {
    const int bfirst = (int)out.blk.size();
    out.cta_blk[c] = bfirst;
    std::fill(lastref.begin(), lastref.end(), -1);
    int64_t P = base;
    int r = bounds[c];
    const int rend = bounds[c + 1];
    while (r < rend) {
      const int bidx = (int)out.blk.size();
      const int64_t Pb = P, lo = Pb + LMAX + margin - W;
      blkloads.clear();
      const int row0 = r;
      int nrows = 0;
      int64_t nent = 0;
      while (r < rend && nrows < rows_max) {
        const int deg = (int)(pstart[r + 1] - pstart[r]);  // padded
        ++rs;
        rownew.clear();
        auto consider = [&](int col) {
          if (last[col] >= lo || rstamp[col] == rs) return;
          rstamp[col] = rs;
          rownew.push_back(col);
        };
        consider(r);
        for (int p = offs[r]; p < offs[r + 1]; ++p) consider(cols[p]);
        const int64_t nl = (int64_t)blkloads.size() + (int64_t)rownew.size();
        if (nrows > 0 && (((nl + 3) & ~3LL) > LMAX || nent + deg > EMAX)) break;
        if (((nl + 3) & ~3LL) > LMAX || deg > EMAX) return false;  // one row alone too big
        for (int col : rownew) {
          last[col] = Pb + (int64_t)blkloads.size();
          blkloads.push_back(col);
        }
        for (int p = offs[r]; p < offs[r + 1]; ++p)
          out.slot[pstart[r] + (p - offs[r])] = (unsigned short)(last[cols[p]] % W);
        out.own[r] = (unsigned short)(last[r] % W);
        nent += deg;
        ++nrows;
        ++r;
      }
      const int nl = (int)((blkloads.size() + 3) & ~(size_t)3);
      while ((int)blkloads.size() < nl) blkloads.push_back(blkloads.back());  // padding: a repeat
      // the producer's wait: the last reader of every slot this block overwrites, and the
      // metadata stage this block reuses
      int wait = std::max(bfirst - 1, bidx - gsk::kWinStages);
      for (int i = 0; i < nl; ++i) wait = std::max(wait, lastref[(Pb + i) % W]);
      // this block's readers: its loads and every reused slot
      for (int i = 0; i < nl; ++i) lastref[(Pb + i) % W] = bidx;
      for (int rr = row0; rr < row0 + nrows; ++rr) {
        lastref[out.own[rr]] = bidx;
        for (int p = offs[rr]; p < offs[rr + 1]; ++p) lastref[out.slot[pstart[rr] + (p - offs[rr])]] = bidx;
      }
      WinBlk b{};
      b.row0 = row0;
      b.nrows = nrows;
      b.lbeg = (int)out.loads.size();
      b.nl = nl;
      b.slot0 = (int)(Pb % W);
      b.e0 = (int)pstart[row0];
      b.e1 = (int)pstart[row0 + nrows];
      b.wait = wait;  // < bfirst: no wait
      out.blk.push_back(b);
      out.loads.insert(out.loads.end(), blkloads.begin(), blkloads.end());
      P += nl;
    }
    base = ((P + W + 3) / 4) * 4;  // nothing loaded by an earlier CTA is ever reusable
  }
  out.cta_blk[nctas] = (int)out.blk.size();
  if (out.loads.empty()) out.loads.assign(4, 0);
  return true;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

}  // namespace

template <typename S>
__global__ void k_win_pad_vals(int n, const int* __restrict__ offs, const S* __restrict__ vals,
                               const int* __restrict__ poffs, S* __restrict__ pvals) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int p0 = offs[r], deg = offs[r + 1] - p0, q0 = poffs[r] & ~3, qe = poffs[r + 1] & ~3;
  for (int i = 0; i < qe - q0; ++i) pvals[q0 + i] = i < deg ? vals[p0 + i] : S(0);
}

// ---- engine-internal entry points (gs_internal.cuh) --------------------------------------------
int gs_win_build(gs_ctx* ctx, gs_filter* f, int row_bytes, int elem_bytes) {
  gs_layout& Ly = f->lay[2];
  const int n = f->scaled->n;
  if (row_bytes <= 0 || row_bytes > 1024 || (row_bytes & 15)) return GS_ERR_UNSUPPORTED;
  const int key = row_bytes * 16 + elem_bytes;
  for (auto* w : Ly.win)
    if (w->row_bytes == key) return w->ok ? GS_OK : GS_ERR_UNSUPPORTED;
  cudaStream_t s = ctx->stream;
  // host copy of the caller-order operator
  std::vector<int> offs(n + 1), cols;
  if (!Ly.perm) {
    // window layout: recursive-bisection order of the scaled operator, renumbered on the device
    GS_CUDA(ctx, cudaMemcpyAsync(offs.data(), f->scaled->offs, (size_t)(n + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    cols.resize(offs[n] > 0 ? offs[n] : 1);
    if (offs[n] > 0)
      GS_CUDA(ctx, cudaMemcpyAsync(cols.data(), f->scaled->cols, (size_t)offs[n] * sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    std::vector<int> order;
    bisect_order(n, offs.data(), cols.data(), 32, order);
    GS_TRY(gs_layout_from_order(ctx, f, 2, order.data()));
  }
  // host copy of the window layout's operator
  const gs_graph* G = Ly.perm;
  GS_CUDA(ctx, cudaMemcpyAsync(offs.data(), G->offs, (size_t)(n + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  cols.resize(offs[n] > 0 ? offs[n] : 1);
  if (offs[n] > 0)
    GS_CUDA(ctx, cudaMemcpyAsync(cols.data(), G->cols, (size_t)offs[n] * sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  const int rows_max = gsk::WinMeta<double>::ROWS_MAX;
  gs_winsched* w = new gs_winsched();
  w->row_bytes = key;
  Ly.win.push_back(w);
  WinHost h;
  const bool verbose = getenv("GS_WIN_VERBOSE") && atoi(getenv("GS_WIN_VERBOSE")) != 0;
  if (n == 0 || !build_schedule(n, offs.data(), cols.data(), row_bytes, elem_bytes, rows_max, sms, h)) {
    w->ok = false;
    if (verbose) fprintf(stderr, "[gs_win] row_bytes=%d elem=%d: no schedule (a row exceeds a block)\n", row_bytes, elem_bytes);
    return GS_ERR_UNSUPPORTED;
  }
  if (verbose)
    fprintf(stderr, "[gs_win] row_bytes=%d elem=%d W=%d lmax=%d blocks=%zu loads=%zu loads/entry=%.3f\n", row_bytes,
            elem_bytes, h.W, h.lmax, h.blk.size(), h.loads.size(), h.entries ? (double)h.loads.size() / h.entries : 0.0);
  w->W = h.W;
  w->nctas = h.nctas;
  w->nblocks = (int)h.blk.size();
  w->nloads = (int64_t)h.loads.size();
  w->loads_per_entry = h.entries ? (double)w->nloads / (double)h.entries : 0.0;
  auto up = [&](void** dst, const void* src, size_t bytes) -> int {
    GS_CUDA(ctx, cudaMalloc(dst, bytes ? bytes : 16));
    if (bytes) GS_CUDA(ctx, cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
    return GS_OK;
  };
  GS_TRY(up((void**)&w->blk, h.blk.data(), h.blk.size() * sizeof(WinBlk)));
  GS_TRY(up((void**)&w->cta_blk, h.cta_blk.data(), h.cta_blk.size() * sizeof(int)));
  GS_TRY(up((void**)&w->loads, h.loads.data(), h.loads.size() * sizeof(int)));
  GS_TRY(up((void**)&w->slot, h.slot.data(), h.slot.size() * sizeof(unsigned short)));
  GS_TRY(up((void**)&w->own, h.own.data(), h.own.size() * sizeof(unsigned short)));
  GS_TRY(up((void**)&w->poffs, h.poffs.data(), h.poffs.size() * sizeof(int)));
  w->padded = h.padded;
  GS_CUDA(ctx, cudaMalloc(&w->pvals, (size_t)(h.padded + 8) * elem_bytes));
  GS_CUDA(ctx, cudaMemsetAsync(w->pvals, 0, (size_t)(h.padded + 8) * elem_bytes, s));
  gs_launch_begin(ctx, 1);
  if (elem_bytes == 8)
    k_win_pad_vals<double><<<(n + 255) / 256, 256, 0, s>>>(n, G->offs, G->vals, w->poffs, (double*)w->pvals);
  else
    k_win_pad_vals<float><<<(n + 255) / 256, 256, 0, s>>>(n, G->offs, Ly.vals32, w->poffs, (float*)w->pvals);
  gs_launch_end(ctx, 1);
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  w->ok = true;
  return GS_OK;
}

const gs_winsched* gs_win_get(const gs_filter* f, int row_bytes, int elem_bytes) {
  for (auto* w : f->lay[2].win)
    if (w->row_bytes == row_bytes * 16 + elem_bytes && w->ok) return w;
  return nullptr;
}

void gs_win_destroy(gs_winsched* w) {
  if (!w) return;
  cudaFree(w->blk);
  cudaFree(w->cta_blk);
  cudaFree(w->loads);
  cudaFree(w->slot);
  cudaFree(w->own);
  cudaFree(w->poffs);
  cudaFree(w->pvals);
  delete w;
}

// 2-D tensor map over `rows` rows of `row_elems` elements (fp64 or 32-bit words), box = one row:
// the source of the tile::gather4 loads.
int gs_win_tensor_map(gs_ctx* ctx, void* tmap, const void* base, int64_t rows, int row_elems, int elem_bytes) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)row_elems, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_elems * (cuuint64_t)elem_bytes};
  cuuint32_t box[2] = {(cuuint32_t)row_elems, 1};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(reinterpret_cast<CUtensorMap*>(tmap),
                        elem_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return GS_OK;
}

// ---- CPU test hooks (no device needed): the order and the schedule on host arrays ---------------
extern "C" int gs_win_bisect_order_host(int n, const int* offs, const int* cols, int leaf, int* order) {
  std::vector<int> o;
  bisect_order(n, offs, cols, leaf, o);
  std::copy(o.begin(), o.end(), order);
  return GS_OK;
}

struct gs_winplan {
  WinHost h;
};

extern "C" int gs_win_plan_host(int n, const int* offs, const int* cols, int row_bytes, int nctas,
                                gs_winplan** out, int64_t* sizes /* W, nctas, blocks, loads, stages, lmax */) {
  *out = nullptr;
  const int rows_max = gsk::WinMeta<double>::ROWS_MAX;
  gs_winplan* p = new gs_winplan();
  if (!build_schedule(n, offs, cols, row_bytes, 8, rows_max, nctas, p->h)) {
    delete p;
    return GS_ERR_UNSUPPORTED;
  }
  sizes[0] = p->h.W;
  sizes[1] = p->h.nctas;
  sizes[2] = (int64_t)p->h.blk.size();
  sizes[3] = (int64_t)p->h.loads.size();
  sizes[4] = gsk::kWinStages;
  sizes[5] = p->h.lmax;
  sizes[6] = p->h.padded;
  *out = p;
  return GS_OK;
}

extern "C" int gs_win_plan_arrays(const gs_winplan* p, int* blk /* 8 per block */, int* cta_blk,
                                  int* loads, int* poffs, unsigned short* slot, unsigned short* own) {
  if (blk) memcpy(blk, p->h.blk.data(), p->h.blk.size() * sizeof(WinBlk));
  if (cta_blk) memcpy(cta_blk, p->h.cta_blk.data(), p->h.cta_blk.size() * sizeof(int));
  if (loads) memcpy(loads, p->h.loads.data(), p->h.loads.size() * sizeof(int));
  if (poffs) memcpy(poffs, p->h.poffs.data(), (p->h.poffs.size() - 8) * sizeof(int));
  if (slot) memcpy(slot, p->h.slot.data(), p->h.padded * sizeof(unsigned short));
  if (own) memcpy(own, p->h.own.data(), (p->h.own.size() - 16) * sizeof(unsigned short));
  return GS_OK;
}

extern "C" void gs_win_plan_destroy(gs_winplan* p) { delete p; }
