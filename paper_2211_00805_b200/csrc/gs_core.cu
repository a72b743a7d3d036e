// gs_core.cu -- context, error plumbing, device CSR objects and from_triplets.
//
// SparseSymMatrix (proj/include/geosink/sparse.hpp:23-61) becomes a device-resident CSR
// (int32 offsets/indices, fp64 values, both triangles, rows sorted by column). from_triplets
// (proj/src/sparse.cpp:15-53) runs on the device: mirror -> radix sort of (row<<32|col) keys
// (stable, so duplicates keep input order) -> run heads -> duplicate-agreement check -> CSR.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstring>

#include "gs_internal.cuh"

static const char* kErrcName[] = {
    "DimensionMismatch", "DuplicatePoints", "NegativeWeight", "NonPositiveTime",
    "LengthMismatch", "TooLarge", "IndexOutOfRange", "SizeMismatch", "DegenerateInput",
    "InvalidArgument", "KernelNotPositive", "Disconnected", "SolveFailure",
    "NumericalUnderflow", "DegeneratePlan", "IoError"};

const char* gs_errc_name(int errc) {
  return (errc >= 0 && errc < 16) ? kErrcName[errc] : "UnknownError";
}

int gs_fail(gs_ctx* ctx, int errc, const std::string& what) {
  if (ctx) ctx->err = std::string(gs_errc_name(errc)) + ": " + what;
  return errc + 1;
}

int gs_cuda_fail(gs_ctx* ctx, cudaError_t e, const char* where) {
  if (ctx) ctx->err = std::string("CudaError: ") + cudaGetErrorString(e) + " at " + where;
  return GS_ERR_CUDA;
}

// ---- context -------------------------------------------------------------------------------
extern "C" int gs_ctx_create(int device, gs_ctx** out) {
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) return GS_ERR_CUDA;
  if (device < 0 || device >= count) return GS_ERR_CUDA;
  if (cudaSetDevice(device) != cudaSuccess) return GS_ERR_CUDA;
  gs_ctx* ctx = new gs_ctx();
  ctx->device = device;
  if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return GS_ERR_CUDA;
  }
  ctx->stream = ctx->own_stream;
  // Workspaces are stream-ordered allocations (cudaMallocAsync) made per call; by default the
  // pool returns freed memory to the driver at every synchronisation, so each call would map its
  // (up to GB-sized) buffers again. Keep it in the pool (GS_POOL_KEEP=0 restores the default).
  {
    const char* e = getenv("GS_POOL_KEEP");
    if (!(e && atoi(e) == 0)) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
    }
  }
  if (cudaMallocHost((void**)&ctx->h_status, 4 * sizeof(gs_status)) != cudaSuccess) {
    cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return GS_ERR_CUDA;
  }
  *out = ctx;
  return GS_OK;
}

extern "C" void gs_ctx_destroy(gs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto& p : ctx->pool) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->ev_packed) cudaEventDestroy(ctx->ev_packed);
  if (ctx->ev_received) cudaEventDestroy(ctx->ev_received);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

extern "C" const char* gs_last_error(const gs_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

extern "C" int gs_ctx_synchronize(gs_ctx* ctx) {
  GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GS_OK;
}

extern "C" int gs_ctx_set_stream(gs_ctx* ctx, void* stream) {
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return GS_OK;
}

extern "C" void* gs_ctx_stream(gs_ctx* ctx) { return (void*)ctx->stream; }

extern "C" int64_t gs_ctx_launch_count(const gs_ctx* ctx) { return ctx->launches; }

static void drain_timing(gs_ctx* ctx, size_t keep) {
  while (ctx->pending.size() > keep) {
    gs_event_pair p = ctx->pending.front();
    ctx->pending.erase(ctx->pending.begin());
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    ctx->t_ms[p.cls] += ms;
    ctx->t_launches[p.cls] += 1;
    ctx->pool.push_back(p);
  }
}

extern "C" int gs_ctx_set_timing(gs_ctx* ctx, int enable) {
  drain_timing(ctx, 0);
  ctx->timing = enable != 0;
  ctx->timing_period = enable > 1 ? enable : 1;  // enable = N > 1: sample every Nth launch
  ctx->t_launches[0] = ctx->t_launches[1] = 0;
  ctx->t_ms[0] = ctx->t_ms[1] = 0.0;
  ctx->t_seen[0] = ctx->t_seen[1] = 0;
  return GS_OK;
}

extern "C" int gs_ctx_timing(gs_ctx* ctx, int cls, int64_t* launches, double* total_ms) {
  drain_timing(ctx, 0);
  if (cls < 0 || cls > 1) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "timing class");
  *launches = ctx->t_launches[cls];
  *total_ms = ctx->t_ms[cls];
  return GS_OK;
}


void gs_launch_begin(gs_ctx* ctx, int cls) {
  ctx->launches++;
  ctx->t_open = false;
  if (!ctx->timing || ctx->capturing) return;
  if ((ctx->t_seen[cls]++ % ctx->timing_period) != 0) return;
  ctx->t_open = true;
  if (ctx->pending.size() >= 8192) drain_timing(ctx, 4096);
  gs_event_pair p;
  if (!ctx->pool.empty()) {
    p = ctx->pool.back();
    ctx->pool.pop_back();
  } else {
    cudaEventCreate(&p.a);
    cudaEventCreate(&p.b);
  }
  p.cls = cls;
  cudaEventRecord(p.a, ctx->stream);
  ctx->pending.push_back(p);
}

void gs_launch_end(gs_ctx* ctx, int cls) {
  (void)cls;
  if (!ctx->timing || ctx->capturing || !ctx->t_open || ctx->pending.empty()) return;
  ctx->t_open = false;
  cudaEventRecord(ctx->pending.back().b, ctx->stream);
}

// ---- copies --------------------------------------------------------------------------------
int gs_copy_in(gs_ctx* ctx, void* dst, const void* src, size_t bytes, int mem) {
  if (!bytes) return GS_OK;
  GS_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes,
                               mem == GS_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                    : cudaMemcpyHostToDevice,
                               ctx->stream));
  return GS_OK;
}

int gs_copy_out(gs_ctx* ctx, void* dst, const void* src, size_t bytes, int mem) {
  if (!bytes) return GS_OK;
  GS_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes,
                               mem == GS_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                    : cudaMemcpyDeviceToHost,
                               ctx->stream));
  if (mem != GS_MEM_DEVICE) GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return GS_OK;
}

// ---- graph objects ---------------------------------------------------------------------------
int gs_graph_alloc(gs_ctx* ctx, int n, int64_t nnz, gs_graph** out) {
  gs_graph* g = new gs_graph();
  g->n = n;
  g->nnz = nnz;
  g->device = ctx->device;
  cudaError_t e = cudaMalloc((void**)&g->offs, ((size_t)n + 1) * sizeof(int));
  // kCsrPad: vectorised CSR loads (gs_step.cuh) read aligned blocks up to 3 entries past a row
  if (e == cudaSuccess) e = cudaMalloc((void**)&g->cols, (size_t)(nnz + kCsrPad) * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc((void**)&g->vals, (size_t)(nnz + kCsrPad) * sizeof(double));
  if (e != cudaSuccess) {
    gs_graph_destroy(g);
    return gs_cuda_fail(ctx, e, "gs_graph_alloc");
  }
  *out = g;
  return GS_OK;
}

extern "C" void gs_graph_destroy(gs_graph* g) {
  if (!g) return;
  cudaFree(g->offs);
  cudaFree(g->cols);
  cudaFree(g->vals);
  delete g;
}

extern "C" int gs_graph_info(const gs_graph* g, int* n, int64_t* nnz) {
  if (n) *n = g->n;
  if (nnz) *nnz = g->nnz;
  return GS_OK;
}

extern "C" int gs_graph_from_csr(gs_ctx* ctx, int n, int64_t nnz, const int* offs,
                                 const int* cols, const double* vals, int mem, gs_graph** out) {
  *out = nullptr;
  if (n < 0 || nnz < 0) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "negative dimension");
  if (nnz > INT32_MAX) return gs_fail(ctx, ERRC_TOO_LARGE, "nnz exceeds int32 offsets");
  gs_graph* g = nullptr;
  GS_TRY(gs_graph_alloc(ctx, n, nnz, &g));
  int rc = gs_copy_in(ctx, g->offs, offs, ((size_t)n + 1) * sizeof(int), mem);
  if (!rc) rc = gs_copy_in(ctx, g->cols, cols, (size_t)nnz * sizeof(int), mem);
  if (!rc) rc = gs_copy_in(ctx, g->vals, vals, (size_t)nnz * sizeof(double), mem);
  if (!rc && mem != GS_MEM_DEVICE) rc = gs_ctx_synchronize(ctx);
  if (rc) {
    gs_graph_destroy(g);
    return rc;
  }
  *out = g;
  return GS_OK;
}

extern "C" int gs_graph_download(gs_ctx* ctx, const gs_graph* g, int* offs, int* cols,
                                 double* vals, int mem) {
  if (offs) GS_TRY(gs_copy_out(ctx, offs, g->offs, ((size_t)g->n + 1) * sizeof(int), mem));
  if (cols) GS_TRY(gs_copy_out(ctx, cols, g->cols, (size_t)g->nnz * sizeof(int), mem));
  if (vals) GS_TRY(gs_copy_out(ctx, vals, g->vals, (size_t)g->nnz * sizeof(double), mem));
  return gs_ctx_synchronize(ctx);
}

// ---- from_triplets (sparse.cpp:15-53) ----------------------------------------------------------
// First failing triplet in input order decides the error, as the reference's sequential loop.
__global__ void k_triplet_check(int n, int64_t m, const int* rows, const int* cols,
                                const double* vals, unsigned long long* first_bad,
                                int* emit_count) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const int r = rows[e], c = cols[e];
  const double v = vals[e];
  int code = -1;
  if (!(r >= 0 && r < n && c >= 0 && c < n)) code = 0;       // IndexOutOfRange
  else if (!isfinite(v)) code = 1;                            // InvalidArgument
  if (code >= 0) atomicMin(first_bad, ((unsigned long long)e << 1) | (unsigned long long)code);
  emit_count[e] = (code >= 0 || v == 0.0) ? 0 : (r != c ? 2 : 1);
}

__global__ void k_triplet_emit(int64_t m, const int* rows, const int* cols, const double* vals,
                               const int* pos, unsigned long long* keys, double* kv) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const double v = vals[e];
  if (v == 0.0 || !isfinite(v)) return;
  const int r = rows[e], c = cols[e];
  const int p = pos[e];
  keys[p] = ((unsigned long long)(unsigned)r << 32) | (unsigned)c;
  kv[p] = v;
  if (r != c) {
    keys[p + 1] = ((unsigned long long)(unsigned)c << 32) | (unsigned)r;
    kv[p + 1] = v;
  }
}

__global__ void k_run_heads(int64_t m, const unsigned long long* keys, const double* vals,
                            unsigned char* head, int* conflict) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const bool h = (e == 0) || keys[e] != keys[e - 1];
  head[e] = h ? 1 : 0;
  if (!h && vals[e] != vals[e - 1]) atomicExch(conflict, 1);
}

__global__ void k_split_keys(int64_t m, const unsigned long long* keys, int* cols) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m) return;
  cols[e] = (int)(unsigned)(keys[e] & 0xFFFFFFFFull);
}

// offs[r] = first entry of row r in the sorted unique key array (rows with no entries repeat).
__global__ void k_row_offsets(int n, int64_t m, const unsigned long long* keys, int* offs) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e > m) return;
  const int64_t lo = (e == 0) ? -1 : (int64_t)(keys[e - 1] >> 32);
  const int64_t hi = (e == m) ? (int64_t)n : (int64_t)(keys[e] >> 32);
  for (int64_t r = lo + 1; r <= hi; ++r) offs[r] = (int)e;
}

static inline unsigned nblk(int64_t m, int t = 256) { return (unsigned)((m + t - 1) / t); }

int gs_csr_from_sorted_entries(gs_ctx* ctx, int n, int64_t m, const unsigned long long* d_keys,
                               const double* d_vals, bool check_dups, gs_graph** out) {
  cudaStream_t s = ctx->stream;
  DevBuf<unsigned char> head;
  DevBuf<int> conflict, nsel;
  GS_CUDA(ctx, head.alloc(m, s));
  GS_CUDA(ctx, conflict.alloc(1, s));
  GS_CUDA(ctx, nsel.alloc(1, s));
  GS_CUDA(ctx, cudaMemsetAsync(conflict.get(), 0, sizeof(int), s));
  if (m > 0) {
    gs_launch_begin(ctx, 1);
    k_run_heads<<<nblk(m), 256, 0, s>>>(m, d_keys, d_vals, head.get(), conflict.get());
    gs_launch_end(ctx, 1);
  }
  int h_conflict = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h_conflict, conflict.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  DevBuf<unsigned long long> ukeys;
  DevBuf<double> uvals;
  GS_CUDA(ctx, ukeys.alloc(m, s));
  GS_CUDA(ctx, uvals.alloc(m, s));
  int64_t u = 0;
  if (m > 0) {
    size_t tmp_bytes = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp_bytes, d_keys, head.get(), ukeys.get(), nsel.get(),
                               (int)m, s);
    DevBuf<unsigned char> tmp;
    GS_CUDA(ctx, tmp.alloc(tmp_bytes, s));
    cub::DeviceSelect::Flagged(tmp.get(), tmp_bytes, d_keys, head.get(), ukeys.get(), nsel.get(),
                               (int)m, s);
    cub::DeviceSelect::Flagged(tmp.get(), tmp_bytes, d_vals, head.get(), uvals.get(), nsel.get(),
                               (int)m, s);
    int h_u = 0;
    GS_CUDA(ctx, cudaMemcpyAsync(&h_u, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    GS_CUDA(ctx, cudaStreamSynchronize(s));
    u = h_u;
  } else {
    GS_CUDA(ctx, cudaStreamSynchronize(s));
  }
  if (check_dups && h_conflict)
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "conflicting duplicate entries break symmetry");
  gs_graph* g = nullptr;
  GS_TRY(gs_graph_alloc(ctx, n, u, &g));
  if (u > 0) {
    gs_launch_begin(ctx, 1);
    k_split_keys<<<nblk(u), 256, 0, s>>>(u, ukeys.get(), g->cols);
    gs_launch_end(ctx, 1);
    cudaMemcpyAsync(g->vals, uvals.get(), (size_t)u * sizeof(double), cudaMemcpyDeviceToDevice, s);
  }
  gs_launch_begin(ctx, 1);
  k_row_offsets<<<nblk(u + 1), 256, 0, s>>>(n, u, ukeys.get(), g->offs);
  gs_launch_end(ctx, 1);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    gs_graph_destroy(g);
    return gs_cuda_fail(ctx, e, "csr assembly");
  }
  *out = g;
  return GS_OK;
}

extern "C" int gs_graph_from_triplets(gs_ctx* ctx, int n, int64_t m, const int* rows,
                                      const int* cols, const double* vals, int mem,
                                      gs_graph** out) {
  *out = nullptr;
  if (n < 0) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "negative dimension");
  cudaStream_t s = ctx->stream;
  DevBuf<int> d_rows, d_cols, cnt, pos;
  DevBuf<double> d_vals;
  DevBuf<unsigned long long> bad;
  GS_CUDA(ctx, d_rows.alloc(m, s));
  GS_CUDA(ctx, d_cols.alloc(m, s));
  GS_CUDA(ctx, d_vals.alloc(m, s));
  GS_CUDA(ctx, cnt.alloc(m + 1, s));
  GS_CUDA(ctx, pos.alloc(m + 1, s));
  GS_CUDA(ctx, bad.alloc(1, s));
  GS_TRY(gs_copy_in(ctx, d_rows.get(), rows, (size_t)m * sizeof(int), mem));
  GS_TRY(gs_copy_in(ctx, d_cols.get(), cols, (size_t)m * sizeof(int), mem));
  GS_TRY(gs_copy_in(ctx, d_vals.get(), vals, (size_t)m * sizeof(double), mem));
  GS_CUDA(ctx, cudaMemsetAsync(bad.get(), 0xFF, sizeof(unsigned long long), s));
  GS_CUDA(ctx, cudaMemsetAsync(cnt.get(), 0, (m + 1) * sizeof(int), s));
  if (m > 0) {
    gs_launch_begin(ctx, 1);
    k_triplet_check<<<nblk(m), 256, 0, s>>>(n, m, d_rows.get(), d_cols.get(), d_vals.get(),
                                            bad.get(), cnt.get());
    gs_launch_end(ctx, 1);
  }
  unsigned long long h_bad = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h_bad, bad.get(), sizeof(h_bad), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  if (h_bad != ~0ull) {
    if ((h_bad & 1ull) == 0) return gs_fail(ctx, ERRC_INDEX_OUT_OF_RANGE, "triplet index out of range");
    return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "non-finite matrix entry");
  }
  // exclusive scan of emit counts -> positions; total at pos[m]
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.get(), pos.get(), (int)(m + 1), s);
  DevBuf<unsigned char> tmp;
  GS_CUDA(ctx, tmp.alloc(tmp_bytes, s));
  cub::DeviceScan::ExclusiveSum(tmp.get(), tmp_bytes, cnt.get(), pos.get(), (int)(m + 1), s);
  int total = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&total, pos.get() + m, sizeof(int), cudaMemcpyDeviceToHost, s));
  GS_CUDA(ctx, cudaStreamSynchronize(s));
  DevBuf<unsigned long long> keys, keys2;
  DevBuf<double> kv, kv2;
  GS_CUDA(ctx, keys.alloc(total, s));
  GS_CUDA(ctx, keys2.alloc(total, s));
  GS_CUDA(ctx, kv.alloc(total, s));
  GS_CUDA(ctx, kv2.alloc(total, s));
  if (m > 0) {
    gs_launch_begin(ctx, 1);
    k_triplet_emit<<<nblk(m), 256, 0, s>>>(m, d_rows.get(), d_cols.get(), d_vals.get(), pos.get(),
                                           keys.get(), kv.get());
    gs_launch_end(ctx, 1);
  }
  if (total > 0) {
    size_t sb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sb, keys.get(), keys2.get(), kv.get(), kv2.get(),
                                    total, 0, 64, s);
    DevBuf<unsigned char> st;
    GS_CUDA(ctx, st.alloc(sb, s));
    cub::DeviceRadixSort::SortPairs(st.get(), sb, keys.get(), keys2.get(), kv.get(), kv2.get(),
                                    total, 0, 64, s);
  }
  return gs_csr_from_sorted_entries(ctx, n, total, keys2.get(), kv2.get(), true, out);
}

// ---- Gershgorin bound (sparse.cpp:107-116) ------------------------------------------------------
__global__ void k_gershgorin(int n, const int* offs, const double* vals, unsigned long long* best) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double row = 0.0;
  for (int p = offs[i]; p < offs[i + 1]; ++p) row = row + fabs(vals[p]);
  // non-negative doubles order like their bit patterns; max is order-free
  atomicMax(best, (unsigned long long)__double_as_longlong(row));
}

extern "C" int gs_graph_gershgorin(gs_ctx* ctx, const gs_graph* g, double* out) {
  DevBuf<unsigned long long> best;
  GS_CUDA(ctx, best.alloc(1, ctx->stream));
  GS_CUDA(ctx, cudaMemsetAsync(best.get(), 0, sizeof(unsigned long long), ctx->stream));
  if (g->n > 0) {
    gs_launch_begin(ctx, 1);
    k_gershgorin<<<nblk(g->n), 256, 0, ctx->stream>>>(g->n, g->offs, g->vals, best.get());
    gs_launch_end(ctx, 1);
  }
  unsigned long long h = 0;
  GS_CUDA(ctx, cudaMemcpyAsync(&h, best.get(), sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  GS_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  double v;
  memcpy(&v, &h, sizeof v);
  *out = v;
  return GS_OK;
}

extern "C" int64_t gs_ctx_knn_fallback(const gs_ctx* ctx) { return ctx ? ctx->knn_fallback : 0; }
