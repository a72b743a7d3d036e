/*
 * geosink_b200.h -- C ABI of the B200-native Geodesic Sinkhorn engine (libgeosink_b200.so).
 *
 * This is the drop-in boundary for the reference library's hot path (`geosink`, a static C++
 * library with no FFI of its own). Each entry point replaces one reference
 * routine, cited as proj/<file>:<line> under /root/reference; the C++ drop-in layer
 * (include/geosink/*.hpp) and the Python mirror (paper_2211_00805_b200/) are thin callers of
 * these functions. Plain pointers and sizes only; no exceptions cross this boundary.
 *
 * Status codes: 0 = ok; 1..16 = reference errc + 1 (proj/include/geosink/errors.hpp:10-30,
 * e.g. 11 = KernelNotPositive, 12 = Disconnected); GS_ERR_CUDA / GS_ERR_NCCL for device and
 * collective failures. gs_last_error() returns "<ErrcName>: <message>" exactly as the
 * reference's geosink::Error::what() would (errors.hpp:54-57).
 *
 * Memory: every array argument lives on the host (GS_MEM_HOST) or on the context's device
 * (GS_MEM_DEVICE), selected per call with `mem`. Vertex signals are `width` contiguous
 * n-vectors (vector p at p*n), the layout of the reference's std::vector<Distribution> inputs.
 * Graphs and filters are device-resident handles owned by the caller.
 *
 * Threading: a context owns one device and one CUDA stream; calls on one context are
 * serialised and stream-ordered. Separate contexts are independent.
 */
#ifndef GEOSINK_B200_H
#define GEOSINK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_OK 0
#define GS_ERR_CUDA 100
#define GS_ERR_NCCL 101
#define GS_ERR_UNSUPPORTED 102

#define GS_MEM_HOST 0
#define GS_MEM_DEVICE 1

/* LaplacianKind (graph.hpp:10) */
#define GS_LAPLACIAN_COMBINATORIAL 0
#define GS_LAPLACIAN_NORMALIZED 1

/* kNN edge kernels: the reference's alpha decay (graph.hpp:26-33) and the BASELINE
 * Gaussian exp(-d^2/sigma^2) with sigma = median k-NN bandwidth (extension) */
#define GS_KERNEL_ALPHA_DECAY 0
#define GS_KERNEL_GAUSSIAN_MEDIAN 1

/* gs_sinkhorn flags */
#define GS_FLAG_SINGLE 1             /* sinkhorn_single messages (transport.cpp:132-134) */
#define GS_FLAG_NO_STAGNATION_ABORT 2 /* bench-only deviation: never raise Disconnected */
#define GS_FLAG_FP32 4                /* optional fp32 mode (vectors and L_s in fp32) */

typedef struct gs_ctx gs_ctx;
typedef struct gs_graph gs_graph;   /* SparseSymMatrix on device (sparse.hpp:23-61) */
typedef struct gs_filter gs_filter; /* HeatFilter on device (heat.hpp:25-54) */

/* ---- context ------------------------------------------------------------------------- */
int gs_ctx_create(int device, gs_ctx** out);
void gs_ctx_destroy(gs_ctx* ctx);
const char* gs_last_error(const gs_ctx* ctx);
int gs_ctx_synchronize(gs_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores the own stream. */
int gs_ctx_set_stream(gs_ctx* ctx, void* stream);
void* gs_ctx_stream(gs_ctx* ctx);
/* Per-kernel-class device timing with CUDA events around launches (bench evidence):
 * enable = 1 times every launch, N > 1 every Nth launch of each class, 0 turns timing off. */
int gs_ctx_set_timing(gs_ctx* ctx, int enable);
/* class: 0 = Chebyshev step kernels, 1 = epilogue/finalise kernels. Returns launches, ms. */
int gs_ctx_timing(gs_ctx* ctx, int kernel_class, int64_t* launches, double* total_ms);
/* Number of engine kernel launches issued on this context so far. */
int64_t gs_ctx_launch_count(const gs_ctx* ctx);
/* Queries of the last kNN in R^d (9 <= d <= 31) whose tensor-core candidate set could not be
 * proven to contain the k nearest and were re-run by the fp64 brute force (diagnostics). */
int64_t gs_ctx_knn_fallback(const gs_ctx* ctx);

/* ---- SparseSymMatrix (sparse.hpp:23-61, sparse.cpp:15-116) --------------------------- */
/* from_triplets (sparse.cpp:15-53): mirror, sort, merge agreeing duplicates, drop zeros. */
int gs_graph_from_triplets(gs_ctx* ctx, int n, int64_t m, const int* rows, const int* cols,
                           const double* vals, int mem, gs_graph** out);
/* Upload an already valid symmetric CSR (both triangles, rows sorted by column). */
int gs_graph_from_csr(gs_ctx* ctx, int n, int64_t nnz, const int* row_offsets,
                      const int* col_indices, const double* values, int mem, gs_graph** out);
void gs_graph_destroy(gs_graph* g);
int gs_graph_info(const gs_graph* g, int* n, int64_t* nnz);
int gs_graph_download(gs_ctx* ctx, const gs_graph* g, int* row_offsets, int* col_indices,
                      double* values, int mem);
/* y = A x (sparse.cpp:70-99); x, y are `width` contiguous n-vectors. */
int gs_graph_multiply(gs_ctx* ctx, const gs_graph* g, const double* x, double* y, int width,
                      int mem);
int gs_graph_gershgorin(gs_ctx* ctx, const gs_graph* g, double* out); /* sparse.cpp:107-116 */

/* ---- graph construction (graph.hpp:26-42, graph.cpp:30-194) -------------------------- */
/* select_knn (graph.cpp:30-71): points row-major n x d; nbrs n x k; eps n. */
int gs_knn(gs_ctx* ctx, const double* points, int n, int d, int k, int mem, int* nbrs,
           double* eps);
/* knn_alpha_decay_graph (graph.cpp:75-108) / Gaussian-median extension; sigma_out optional */
int gs_knn_graph(gs_ctx* ctx, const double* points, int n, int d, int k, int kernel,
                 double param, int mem, gs_graph** out, double* sigma_out);
/* laplacian (graph.cpp:110-165); lambda via estimate_lambda_max for the combinatorial kind;
 * rounds_out (optional): power rounds used, -1 = Gershgorin fallback. */
int gs_laplacian(gs_ctx* ctx, const gs_graph* A, int kind, gs_graph** L_out,
                 double* lambda_bound, int* rounds_out);
int gs_lambda_max(gs_ctx* ctx, const gs_graph* L, double* out, int* rounds_out);

/* ---- heat operator (heat.hpp:19-54, heat.cpp:14-131) --------------------------------- */
int gs_heat_coefficients(gs_ctx* ctx, double t, int degree, double* out /* degree+1 */);
int gs_filter_create(gs_ctx* ctx, const gs_graph* L, int kind, double lambda_bound, double t,
                     int degree, gs_filter** out);
void gs_filter_destroy(gs_filter* f);
int gs_filter_info(const gs_filter* f, int* n, double* t, double* t_eff, double* scale,
                   int* degree, int* kind);
int gs_filter_coefficients(const gs_filter* f, double* out /* degree+1 */);
const gs_graph* gs_filter_scaled(const gs_filter* f);
/* The filter's internal vertex order (order[new] = old, n entries; locality renumbering). */
int gs_filter_order(gs_ctx* ctx, const gs_filter* f, int* order, int mem);
/* Replace the locality order of layout 0 (wide column groups) or 1 (narrow ones) with a
 * caller-supplied permutation (order[new] = old). Results are unchanged (each row keeps its
 * entries in the original column order); only the memory locality of the gathers changes.
 * Not a permutation of 0..n-1 -> invalid_argument (layout reset to the identity). No reference
 * counterpart (the reference has no locality renumbering). */
int gs_filter_set_order(gs_ctx* ctx, gs_filter* f, int layout, const int* order, int mem);

/* ---- windowed step kernel: host-side plan (engine internals, exposed for CPU tests) -------
 * The wide-row Chebyshev step (gs_win.cuh) runs on a recursive-bisection vertex order and a
 * per-CTA shared-memory ring schedule. These host functions compute both from a CSR pattern on
 * host arrays so the schedule's invariants can be checked without a device. sizes[7] = ring
 * slots W, CTAs, blocks, loads, stages, max loads per block, padded entries; blk holds 8 ints
 * per block (row0, nrows, lbeg, nl, slot0, e0, e1, 0) with e0/e1 in the quad-padded CSR whose
 * row starts are poffs[r] & ~3 (poffs[r] & 3 = padding entries of row r); slot is indexed by
 * padded entry. GS_ERR_UNSUPPORTED: a row alone exceeds a block. */
typedef struct gs_winplan gs_winplan;
int gs_win_bisect_order_host(int n, const int* offs, const int* cols, int leaf, int* order);
int gs_win_plan_host(int n, const int* offs, const int* cols, int row_bytes, int nctas,
                     gs_winplan** out, int64_t* sizes);
int gs_win_plan_arrays(const gs_winplan* p, int* blk, int* cta_blk, int* loads, int* poffs,
                       unsigned short* slot, unsigned short* own);
void gs_win_plan_destroy(gs_winplan* p);

/* ---- dense baselines (the kNN benchmark's dense_sinkhorn_w1 / _w2 rows) ---- */
/* dense_sinkhorn (transport.cpp:271-311): cost r x c row-major, mu (r), nu (c); outputs v (r),
 * w (c), cost, kl, iterations, converged, marginal_error. mem applies to every array. */
int gs_dense_sinkhorn(gs_ctx* ctx, const double* cost, int r, int c, const double* mu,
                      const double* nu, double lambda, int max_iter, double tol, int mem,
                      double* out_v, double* out_w, double* out_cost, double* out_kl,
                      int* out_iters, int* out_conv, double* out_err);
/* knn_benchmark's dense methods (bench.cpp:311-331): host arrays. X n x d row-major; group g is
 * X rows group_idx[group_off[g] .. group_off[g+1]); pair p transports group pair_a[p] onto
 * pair_b[p] with uniform marginals and cost squared_distances (bench.cpp:32-39; squared = 1) or
 * its square root. Outputs per pair; the first failing pair (kernel underflow) in fail_pair. */
int gs_dense_sinkhorn_groups(gs_ctx* ctx, const double* X, int n, int d, const int* group_idx,
                             const int* group_off, int ngroups, const int* pair_a,
                             const int* pair_b, int P, int squared, double lambda, int max_iter,
                             double tol, double* out_cost, double* out_kl, int* out_iters,
                             int* out_conv, double* out_err, int* fail_pair);
/* p_K(L_s) X for `width` contiguous n-vectors (heat.cpp:98-131). */
int gs_filter_apply(gs_ctx* ctx, const gs_filter* f, const double* X, double* Y, int width,
                    int mem);
/* Same with flags (GS_FLAG_FP32 selects the fp32 mode). */
int gs_filter_apply_ex(gs_ctx* ctx, const gs_filter* f, const double* X, double* Y, int width,
                       int mem, int flags);

/* ---- transport (transport.hpp:58-69, transport.cpp:108-255) -------------------------- */
/* P pairs against one filter (geodesic_sinkhorn_batch; P = 1 + GS_FLAG_SINGLE is
 * geodesic_sinkhorn). mus, nus, out_v, out_w: P contiguous n-vectors; a: n. On Disconnected
 * fail_pair / fail_sweep (optional) name the pair and sweep. */
int gs_sinkhorn(gs_ctx* ctx, const gs_filter* f, const double* a, const double* mus,
                const double* nus, int P, int max_iter, double tol, int flags, int mem,
                double* out_v, double* out_w, double* out_cost, double* out_kl, int* out_iters,
                int* out_conv, double* out_err, int* fail_pair, int* fail_sweep);

/* plan_row (transport.cpp:314-324), batched: out row q = max(v[rows[q]] * H e_rows[q] .* a .* w, 0);
 * a, v, w: n; rows: nrows; out: nrows contiguous n-vectors. */
int gs_plan_rows(gs_ctx* ctx, const gs_filter* f, const double* a, const double* v,
                 const double* w, const int* rows, int nrows, int mem, double* out);

/* ---- graph text format (sparse.cpp:137-174) ------------------------------------------ */
/* Status 16 (errc::io_error + 1) on file errors; "IoError" semantics of the reference. */
int gs_graph_save(gs_ctx* ctx, const gs_graph* g, const char* path);
int gs_graph_load(gs_ctx* ctx, const char* path, gs_graph** out);

/* ---- collective hooks (multi-process runs) ---------------------------- */
/* allreduce: reduces `count` doubles of the device buffer in place across ranks (op 0 = sum,
 * 1 = max) on `stream`. alltoallv: rank r sends send_bytes[q] bytes (consecutive slices of
 * sendbuf, rank order) to every rank q and receives recv_bytes[q] bytes from q into consecutive
 * slices of recvbuf; device buffers, on `stream`. Return 0 on success. The engine never links a
 * collective library itself: the caller's runtime (torch.distributed over NCCL, MPI, ...) does
 * the transfer. */
typedef int (*gs_allreduce_fn)(void* user, double* device_buf, int64_t count, int op,
                               void* stream);
typedef int (*gs_alltoallv_fn)(void* user, const void* sendbuf, const int64_t* send_bytes,
                               void* recvbuf, const int64_t* recv_bytes, int nranks, void* stream);
#define GS_COMM_GRAPH_SAFE 1 /* hooks only enqueue stream-ordered device work: CUDA-graph capture
                                * of whole sweeps stays on (the engine's NCCL communicator) */
typedef struct {
  gs_allreduce_fn allreduce;
  void* user;
  gs_alltoallv_fn alltoallv; /* row-partitioned runs only; may be NULL otherwise */
  int flags;                 /* GS_COMM_GRAPH_SAFE or 0 (host-callback hooks) */
} gs_comm;

/* ---- in-engine NCCL communicator (NVLink / NVSwitch data plane) --------------------------
 * One process per GPU. Rank 0 calls gs_nccl_unique_id and broadcasts the 128 bytes through the
 * caller's bootstrap (torch.distributed, MPI, a file); every rank then calls
 * gs_nccl_comm_create on its own context. The returned gs_comm's hooks call ncclAllReduce and,
 * for halo exchanges, one ncclGroupStart/End of ncclSend/ncclRecv with the ranks that have bytes
 * to exchange (the partition's neighbours only), on the engine's stream; it carries
 * GS_COMM_GRAPH_SAFE, so barycenter sweeps stay CUDA-graph captured with the collective inside.
 * NCCL is loaded at run time (libnccl.so.2, the one already in the process when there is one);
 * GS_ERR_NCCL when it is missing or a call fails. */
#define GS_NCCL_UNIQUE_ID_BYTES 128
int gs_nccl_unique_id(void* id_out);
int gs_nccl_comm_create(gs_ctx* ctx, const void* id, int nranks, int rank, gs_comm** out);
void gs_nccl_comm_destroy(gs_comm* comm);
/* Host-side invocations of the communicator's hooks so far (a replayed sweep graph re-runs its
 * captured collectives without invoking them again). */
int64_t gs_nccl_comm_calls(const gs_comm* comm);

/* ---- row partitions (row-partitioned multi-GPU applies) ----------------- */
/* The reference is single-process (OpenMP rows, heat.cpp:116-131 over sparse.cpp:85-99); this
 * splits the same products by rows. Part `part` of `nparts` owns a contiguous nnz-balanced range
 * of the filter's locality order plus the halo rows its products read; every rank builds its part
 * from its own replica of the filter. Per-part vectors are n_local = row_end - row_begin values
 * in the order gs_part_vertices lists (original vertex ids). */
typedef struct gs_part gs_part;
int gs_part_create(gs_ctx* ctx, const gs_filter* f, int nparts, int part, gs_part** out);
void gs_part_destroy(gs_part* p);
int gs_part_info(const gs_part* p, int* row_begin, int* row_end, int* n_halo, int64_t* nnz_local,
                 int* n_send);
/* local rows [lo, hi) read no halo row: computed while the exchange is in flight */
int gs_part_interior(const gs_part* p, int* lo, int* hi);
/* rows sent to / received from each rank per exchange (nparts entries each, optional) */
int gs_part_counts(const gs_part* p, int64_t* send_counts, int64_t* recv_counts);
int gs_part_vertices(gs_ctx* ctx, const gs_part* p, int* out, int mem);
/* HeatFilter::apply on this part's rows (heat.cpp:116-131): X, Y are `width` contiguous
 * n_local-vectors; one halo exchange per Chebyshev step through comm->alltoallv (nparts > 1).
 * flags: GS_FLAG_FP32. Results equal gs_filter_apply's rows bit for bit. */
int gs_part_filter_apply(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const double* X,
                         double* Y, int width, int flags, int mem);
/* geodesic_sinkhorn_batch on this part's rows (transport.cpp:144-239): a, mus, nus, out_v, out_w
 * hold n_local values per vector; per-column reductions (positivity min/max, L1 error, cost/KL
 * sums, validation sums) are allreduced so every rank takes the same decisions and returns the
 * same scalars. Arguments otherwise as gs_sinkhorn. */
int gs_part_sinkhorn(gs_ctx* ctx, const gs_part* p, const gs_comm* comm, const double* a,
                     const double* mus, const double* nus, int P, int max_iter, double tol,
                     int flags, int mem, double* out_v, double* out_w, double* out_cost,
                     double* out_kl, int* out_iters, int* out_conv, double* out_err,
                     int* fail_pair, int* fail_sweep);

/* ---- barycenter (barycenter.hpp:36-42, barycenter.cpp:45-107) ------------------------ */
/* `comm` (optional, allreduce only) makes a member-sharded barycenter: NULL = single rank. */

/* members, out_V, out_W: m contiguous n-vectors; alphas: m or NULL (uniform). With a comm,
 * the caller passes its local members and their alphas (global weights). */
int gs_barycenter(gs_ctx* ctx, const gs_filter* f, const double* a, const double* members,
                  int m, const double* alphas, int max_iter, double tol, int mem,
                  const gs_comm* comm, double* out_bary, double* out_V, double* out_W,
                  int* out_iters, int* out_conv, double* out_err);
/* Same with flags (GS_FLAG_FP32 selects the fp32 mode). */
int gs_barycenter_ex(gs_ctx* ctx, const gs_filter* f, const double* a, const double* members,
                     int m, const double* alphas, int max_iter, double tol, int mem,
                     const gs_comm* comm, int flags, double* out_bary, double* out_V,
                     double* out_W, int* out_iters, int* out_conv, double* out_err);

/* ---- EulerHeat (heat.hpp:60-84, heat.cpp:133-219) ------------------- */
/* The implicit-Euler competitor: `steps` solves of (I + (t/steps) L) x = b, each the reference's
 * lockstep conjugate gradient over the batch (Solver::lockstep_cg; tolerance 1e-10 relative
 * residual, at most 10 n iterations -> status 13 = SolveFailure). */
typedef struct gs_euler gs_euler;
/* EulerHeat::Solver (heat.hpp:62): automatic = direct for n <= 4000, lockstep CG above */
#define GS_EULER_AUTOMATIC 0
#define GS_EULER_DIRECT 1     /* dense Cholesky of I + hL on the device (the reference: sparse
                               * LDLT; same solution up to rounding), n <= 16384 */
#define GS_EULER_LOCKSTEP_CG 2
int gs_euler_create(gs_ctx* ctx, const gs_graph* L, double t, int steps, gs_euler** out);
int gs_euler_create_ex(gs_ctx* ctx, const gs_graph* L, double t, int steps, int solver,
                       gs_euler** out);
void gs_euler_destroy(gs_euler* e);
const gs_graph* gs_euler_system(const gs_euler* e); /* I + (t/steps) L, caller's vertex order */
/* X, Y: `width` contiguous n-vectors; iters_out (optional): CG iterations of the last solve */
int gs_euler_apply(gs_ctx* ctx, const gs_euler* e, const double* X, double* Y, int width, int mem,
                   int* iters_out);

/* euler_sinkhorn[_batch] (transport.cpp:257-269): sinkhorn_many over EulerHeat. Arguments as
 * gs_sinkhorn; converged pairs leave the lockstep-CG batch after every sweep, as in the
 * reference's compaction (the CG couples the columns of a batch). */
int gs_euler_sinkhorn(gs_ctx* ctx, const gs_euler* e, const double* a, const double* mus,
                      const double* nus, int P, int max_iter, double tol, int flags, int mem,
                      double* out_v, double* out_w, double* out_cost, double* out_kl,
                      int* out_iters, int* out_conv, double* out_err, int* fail_pair,
                      int* fail_sweep);

/* ---- seeded RNG (rng.hpp:13-68), host-side ---------------------------------------------- */
typedef struct gs_rng gs_rng;
gs_rng* gs_rng_create(uint64_t seed);
void gs_rng_destroy(gs_rng* r);
uint64_t gs_rng_bits(gs_rng* r);
double gs_rng_uniform(gs_rng* r);
double gs_rng_uniform_range(gs_rng* r, double lo, double hi);
double gs_rng_normal(gs_rng* r);
uint64_t gs_rng_below(gs_rng* r, uint64_t n);
uint64_t gs_rng_seed_mix(uint64_t a, uint64_t b);
/* repeating draw pattern: kind 0 = lo + (hi-lo)*uniform, 1 = hi*normal (+lo), 2 = below(hi) */
void gs_rng_fill_pattern(gs_rng* r, double* out, int64_t count, const int* kind,
                         const double* lo, const double* hi, int npat);

#ifdef __cplusplus
}
#endif
#endif
