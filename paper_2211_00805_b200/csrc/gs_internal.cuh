// gs_internal.cuh -- shared declarations of the B200 Geodesic Sinkhorn engine.
//
// Rounding contract: every translation unit is compiled with -fmad=false; fused operations are
// written as fma() exactly where oracle/geosink_oracle.c writes them, so the device reproduces
// the oracle bit for bit on every + - * / sqrt fma path (log/exp/pow are the only libdevice vs
// glibc differences).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <mutex>
#include <vector>

#include "geosink_b200.h"

// errc numbering (proj/include/geosink/errors.hpp:10-30)
enum gs_errc {
  ERRC_DIMENSION_MISMATCH = 0, ERRC_DUPLICATE_POINTS, ERRC_NEGATIVE_WEIGHT,
  ERRC_NON_POSITIVE_TIME, ERRC_LENGTH_MISMATCH, ERRC_TOO_LARGE, ERRC_INDEX_OUT_OF_RANGE,
  ERRC_SIZE_MISMATCH, ERRC_DEGENERATE_INPUT, ERRC_INVALID_ARGUMENT, ERRC_KERNEL_NOT_POSITIVE,
  ERRC_DISCONNECTED, ERRC_SOLVE_FAILURE, ERRC_NUMERICAL_UNDERFLOW, ERRC_DEGENERATE_PLAN,
  ERRC_IO_ERROR
};

const char* gs_errc_name(int errc);

struct gs_status;

struct gs_event_pair {
  cudaEvent_t a, b;
  int cls;
};

struct gs_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  // timing ring (gs_ctx_set_timing)
  bool timing = false;
  std::vector<gs_event_pair> pending;
  std::vector<gs_event_pair> pool;
  int64_t t_launches[2] = {0, 0};
  double t_ms[2] = {0.0, 0.0};
  int timing_period = 1;         // time every Nth launch of a class (sampling)
  int64_t t_seen[2] = {0, 0};
  bool t_open = false;
  // pinned status mirror for host polling
  gs_status* h_status = nullptr;
  // CUDA-graph capture in progress: launches are counted, not timed
  bool capturing = false;
  // row-partitioned runs: halo exchanges run on a second stream, overlapped with interior rows
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_received = nullptr;
  // queries of the last tensor-core kNN that the brute force re-ran (gs_knn_tc.cu)
  int64_t knn_fallback = 0;
};

struct gs_graph {
  int n = 0;
  int64_t nnz = 0;
  int* offs = nullptr;    // n+1
  int* cols = nullptr;    // nnz
  double* vals = nullptr; // nnz
  int device = 0;
};

// Ring schedule of the windowed step kernel for one row size (gs_win.cu / gs_win.cuh).
struct gs_winsched {
  int row_bytes = 0;
  bool ok = false;
  int W = 0, nctas = 0, nblocks = 0;
  int64_t nloads = 0;
  double loads_per_entry = 0.0;  // neighbour-row loads per CSR entry (the gather model counts 1)
  void* blk = nullptr;           // gsk::WinBlk[nblocks]
  int* cta_blk = nullptr;        // nctas + 1
  int* loads = nullptr;
  unsigned short* slot = nullptr;
  unsigned short* own = nullptr;
  int* poffs = nullptr;    // rows padded to whole quads (gs_win.cuh WinArgs::poffs)
  void* pvals = nullptr;   // padded values (fp64, or fp32 for the 32-bit mode's row size)
  int64_t padded = 0;
};

// Jagged sliced store of a CSR operator for the sliced step kernel (gs_sell.cu / gs_sell.cuh).
struct gs_sell {
  int C = 0, JV = 0, elem_bytes = 0;  // rows per slice, entries per chunk, value size
  int nslices = 0;
  long long total = 0;        // stored entries (padding included)
  long long* soff = nullptr;  // nslices + 1
  int* cols = nullptr;
  void* vals = nullptr;
  long long* cpre = nullptr;  // nslices + 1: prefix of the slice costs (static warp split)
};

// One locality layout of the filter's operator (gs_reorder.cu): renumbered rows + fp32 copy.
// odd-stride copy of a layout's CSR arrays for k_cheb_lane (gs_lane.cu): rows with an even number
// of entries are followed by one pad entry (column -1, value 0)
struct gs_lanepad {
  int* offs = nullptr;  // n + 1
  int* cols = nullptr;  // nnz + kCsrPad
  void* vals = nullptr;
  int elem_bytes = 0;   // 4: vals32, 8: fp64 values
  int64_t nnz = 0;      // stored entries, pads included
};

struct gs_layout {
  gs_graph* perm = nullptr;  // L_s with rows renumbered (entries kept in original column order)
  int* order = nullptr;      // order[new] = old
  int* newpos = nullptr;     // newpos[old] = new
  float* vals32 = nullptr;   // fp32 copy of perm->vals (optional fp32 mode)
  double near_frac = 1.0;    // fraction of entries within 256 rows of their row (L1 locality)
  // 8-row block records (gs_step.cuh k_cheb_blk; built on first use by a wide fp64 run): the
  // entries of rows [8b, 8b + 8) in positions [offs[8b], offs[8b + 8]) re-sorted by (original
  // column, row), key = new column << 3 | row within the block
  int* rec_key = nullptr;
  double* rec_val = nullptr;
  // lay[2] only: ring schedules of the windowed step kernel, one per row size (built on first use)
  std::vector<gs_winsched*> win;
  // sliced stores of `perm`, one per (slice height, value size); built on first use
  std::vector<gs_sell*> sell;
  // odd-stride copies of `perm` for k_cheb_lane, one per value size; built on first use
  std::vector<gs_lanepad*> lanepad;
  // `perm`'s entries as 16-byte records {col, -, val} for k_cheb_rec (fp64); built on first use
  void* recs = nullptr;
};

struct gs_filter {
  gs_graph* scaled = nullptr;   // L_s in the caller's vertex order (heat.hpp:47)
  // lay[0]: Cuthill-McKee order (wide batches, one warp per row);
  // lay[1]: CM with degree-sorted windows (narrow batches, several rows per warp);
  // lay[2]: recursive-bisection order for the windowed step kernel (built on first use)
  gs_layout lay[3];
  double t = 0, t_eff = 0, scale = 1;
  int degree = 0, kind = 0;
  int sigma = 0;  // window of lay[1]'s degree sort (0: a caller-supplied order, no such structure)
  std::vector<double> coeffs;  // host mirror (heat.hpp:37)
  // serialises the structures built on first use (window schedules, sliced stores, odd-stride and
  // record copies, block records) when several host threads run on one filter
  std::mutex build_mu;
  double* d_coeffs = nullptr;
};

// One rank's row partition of a filter (gs_part.cu; SURVEY.md §8(e) "row partitioning"): a
// contiguous nnz-balanced range [row_begin, row_end) of the filter's Cuthill-McKee order (lay[0]).
// Local rows keep their CSR entries in the original order with columns renumbered: [0, nl) local
// rows, [nl, nl + nh) halo rows sorted by (owner rank, position). Rows this rank sends to rank q
// (its rows adjacent to q's range, ascending) are send_rows[send_offs[q] .. send_offs[q + 1]).
struct gs_part {
  const gs_filter* f = nullptr;
  int nparts = 1, part = 0;
  int n_global = 0, row_begin = 0, row_end = 0, nl = 0, nh = 0, ns = 0;
  int int_lo = 0, int_hi = 0;  // local rows [int_lo, int_hi) read no halo row (interior)
  gs_graph* local = nullptr;
  float* vals32 = nullptr;
  gs_lanepad* lanepad[2] = {nullptr, nullptr};  // odd-stride copies of `local` (vals32 / fp64), on first use
  int* vertices = nullptr;   // nl: original vertex id of each local row
  int* send_rows = nullptr;  // ns local row indices
  std::vector<int> bounds;   // nparts + 1 positions
  std::vector<int64_t> send_counts, recv_counts;  // rows per rank
};

// ---- error plumbing ----------------------------------------------------------------------
int gs_fail(gs_ctx* ctx, int errc, const std::string& what);  // returns errc + 1
int gs_cuda_fail(gs_ctx* ctx, cudaError_t e, const char* where);

#define GS_CUDA(ctx, expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return gs_cuda_fail(ctx, _e, #expr); \
  } while (0)

#define GS_TRY(expr)          \
  do {                        \
    int _rc = (expr);         \
    if (_rc != 0) return _rc; \
  } while (0)

// ---- once-per-device setup (function attributes are set per device) ---------------------------
// runs `setup` the first time this site is reached on the current device; `seen` is the site's
// static record. Serialised: contexts on several host threads launch the same kernels, and a
// launch must not overtake another thread's cudaFuncSetAttribute.
inline std::mutex& gs_once_mutex() {
  static std::mutex mu;
  return mu;
}
template <typename F>
inline void gs_once_per_device(std::vector<char>& seen, F&& setup) {
  std::lock_guard<std::mutex> lock(gs_once_mutex());
  int dev = 0;
  cudaGetDevice(&dev);
  if ((int)seen.size() <= dev) seen.resize(dev + 1, 0);
  if (seen[dev]) return;
  setup();
  seen[dev] = 1;
}

// ---- launch accounting / timing ------------------------------------------------------------
void gs_launch_begin(gs_ctx* ctx, int cls);
void gs_launch_end(gs_ctx* ctx, int cls);

// ---- device scratch ------------------------------------------------------------------------
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  cudaError_t alloc(size_t count, cudaStream_t stream) {
    release();
    s = stream;
    n = count;
    return cudaMallocAsync((void**)&p, (count ? count : 1) * sizeof(T), stream);
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

// ---- shared device helpers ----------------------------------------------------------------
constexpr int kCsrPad = 8;  // elements allocated past nnz in CSR column / value arrays
#define GS_FLOOR 1e-300
#define GS_CEIL 1e300
#define DET_T 256
#define DET_J 16
#define DET_CHUNK (DET_T * DET_J)

// Global status word layout shared by kernels and the host poll.
struct gs_status {
  int error;      // 0 or errc + 1
  int fail_pair;  // Disconnected pair
  int fail_sweep; // sweep of the failure
  int n_active;   // active columns after the last control step
  int done;       // barycenter converged / finished
  int pad[3];
};

// ---- internal entry points shared across translation units -----------------------------------
int gs_graph_alloc(gs_ctx* ctx, int n, int64_t nnz, gs_graph** out);
int gs_copy_in(gs_ctx* ctx, void* dst, const void* src, size_t bytes, int mem);
int gs_copy_out(gs_ctx* ctx, void* dst, const void* src, size_t bytes, int mem);
int gs_lambda_max_impl(gs_ctx* ctx, const gs_graph* L, double* out, int* rounds_out);
int gs_coefficients_impl(gs_ctx* ctx, double t, int degree, double* d_out, double* h_out);
int gs_sigma_order(gs_ctx* ctx, const gs_graph* g, const int* d_newpos, int sigma, int* d_order_sig,
                   int* d_newpos_sig);
int gs_bfs_order(gs_ctx* ctx, const gs_graph* g, int* d_order, int* d_newpos, int sigma,
                 int* d_order_sig, int* d_newpos_sig);
int gs_permute_graph(gs_ctx* ctx, const gs_graph* g, const int* d_order, const int* d_newpos,
                     gs_graph** out);
// grouped-layout fp64 SpMM y = G x through the step kernel (gs_cheb.cu): B columns in
// gs_group_width(B)-wide groups, each an n x GW row-major block
int gs_group_width(int B);
int gs_spmm_grouped(gs_ctx* ctx, const gs_graph* g, const double* x, double* y, int B);
int gs_check_transport_inputs(gs_ctx* ctx, int n, const double* dmu, const double* dnu, const double* da,
                              int P, int max_iter, double tol);
// windowed step kernel (gs_win.cu): build / look up the ring schedule of lay[2] for a row size
// (GS_ERR_UNSUPPORTED when a row alone exceeds a block), free one, encode a gather tensor map
int gs_win_build(gs_ctx* ctx, gs_filter* f, int row_bytes, int elem_bytes);
const gs_winsched* gs_win_get(const gs_filter* f, int row_bytes, int elem_bytes);
void gs_win_destroy(gs_winsched* w);
int gs_win_tensor_map(gs_ctx* ctx, void* tmap, const void* base, int64_t rows, int row_elems, int elem_bytes);
// sliced store (gs_sell.cu) of G for slices of C rows, values of elem_bytes (4: vals32)
int gs_sell_build(gs_ctx* ctx, const gs_graph* G, const float* vals32, int C, int elem_bytes, gs_sell** out);
void gs_sell_destroy(gs_sell* p);
int gs_sell_split(gs_ctx* ctx, const gs_sell* p, int W, int* d_wstart);
// odd-stride CSR copy (gs_lane.cu); GS_ERR_UNSUPPORTED when the padded positions leave 32 bits
int gs_lanepad_build(gs_ctx* ctx, const int* offs, const int* cols, const void* vals, int elem_bytes, int n,
                     int64_t nnz, gs_lanepad** out);
void gs_lanepad_destroy(gs_lanepad* p);
// 16-byte record copy {col, -, val} of a CSR operator's entries (nnz + kCsrPad records)
int gs_recs_build(gs_ctx* ctx, const int* cols, const double* vals, int64_t nnz, void** out);
// layout l of f from a host order (order[new] = old): newpos, renumbered operator, fp32 copy
int gs_layout_from_order(gs_ctx* ctx, gs_filter* f, int l, const int* h_order);
// kNN (gs_graph.cu / gs_knn_tc.cu): brute force over a query list; tensor-core prefilter + exact
// fp64 re-rank (indices and eps identical to the brute force)
int gs_knn_brute_list(gs_ctx* ctx, const double* dpts, const double* sq, int n, int d, int k,
                      const int* qlist, int nq, int* dnb, double* deps);
int gs_knn_tc(gs_ctx* ctx, const double* dpts, const double* sq, int n, int d, int k, int* dnb,
              double* deps);
int gs_csr_from_sorted_entries(gs_ctx* ctx, int n, int64_t m, const unsigned long long* d_keys,
                               const double* d_vals, bool check_dups, gs_graph** out);
