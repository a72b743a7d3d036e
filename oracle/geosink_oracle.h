/*
 * geosink_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity oracle for the B200 engine. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product path
 * (libgeosink_b200.so) never links or calls it.
 *
 * Every routine restates one reference routine (file:line into /root/reference/proj) in plain
 * C11 + OpenMP with the rounding made explicit: the file is compiled with -ffp-contract=off and
 * every fused multiply-add is written as fma(), so the CUDA kernels (compiled with -fmad=false
 * and the same explicit fma()) reproduce it bit for bit wherever only + - * / sqrt fma occur.
 *
 * Parity pinning: the reference cannot be compiled here (Eigen3 is absent);
 * its header-only RNG (include/geosink/rng.hpp) is compiled into oracle/_ref and checked
 * against go_rng_* below; the numerics are pinned against the reference tests' closed forms
 * and independent scipy oracles (tests/golden/).
 *
 * Status codes: 0 = ok, otherwise (errc + 1) with errc numbered as in
 * reference include/geosink/errors.hpp:10-30. go_last_error() returns the message.
 */
#ifndef GEOSINK_ORACLE_H
#define GEOSINK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int n;
  int64_t nnz;
  int* row_offsets;  /* n+1 */
  int* col_indices;  /* nnz */
  double* values;    /* nnz */
} go_csr;

const char* go_last_error(void);

/* rng.hpp:13-68 */
void go_rng_bits(uint64_t seed, int64_t count, uint64_t* out);
void go_rng_uniform(uint64_t seed, int64_t count, double* out);
void go_rng_normal(uint64_t seed, int64_t count, double* out);
void go_rng_below(uint64_t seed, uint64_t bound, int64_t count, uint64_t* out);
uint64_t go_rng_seed_mix(uint64_t a, uint64_t b);
/* stateful handle: one Rng object drawn across calls */
void* go_rng_new(uint64_t seed);
void go_rng_free(void* r);
uint64_t go_rng_next_bits(void* r);
double go_rng_next_uniform(void* r);
double go_rng_next_normal(void* r);
uint64_t go_rng_next_below(void* r, uint64_t n);
void go_rng_fill_pattern(void* r, double* out, int64_t count, const int* kind, const double* lo,
                         const double* hi, int npat);

/* sparse.cpp:15-53 */
int go_csr_from_triplets(int n, int64_t m, const int* rows, const int* cols, const double* vals,
                         go_csr* out);
int go_csr_from_arrays(int n, int64_t nnz, const int* offs, const int* cols, const double* vals,
                       go_csr* out);
void go_csr_free(go_csr* m);
/* sparse.cpp:70-99 ; x, y row-major n x width */
int go_spmm(const go_csr* m, const double* x, double* y, int width);
/* sparse.cpp:107-116 */
double go_gershgorin(const go_csr* m);

/* deterministic blocked sums shared bit-for-bit with the device */
double go_detdot(const double* x, const double* y, int64_t n);

/* graph.cpp:30-71 ; points row-major n x d ; nbrs n x k ascending (d2, idx) */
int go_knn(const double* pts, int n, int d, int k, int* nbrs, double* eps);
int go_knn_rows(const double* pts, int n, int d, int k, const int* rows, int nrows, int* nbrs,
                double* eps);
/* graph.cpp:75-108 (kernel 0 = alpha decay, param = alpha) and the BASELINE Gaussian
 * extension (kernel 1: w = exp(-d^2 / sigma^2), sigma = median of eps_k); sigma_out optional */
int go_knn_graph(const double* pts, int n, int d, int k, int kernel, double param, go_csr* out,
                 double* sigma_out);
/* graph.cpp:110-165 ; kind 0 combinatorial, 1 normalized ; lambda via graph.cpp:167-194 */
int go_laplacian(const go_csr* A, int kind, go_csr* L, double* lambda_bound, int* rounds_out);
/* graph.cpp:167-194 ; rounds_out = power rounds used, -1 when the Gershgorin fallback fired */
int go_lambda_max(const go_csr* L, double* out, int* rounds_out);

/* heat.cpp:14-70 */
int go_heat_coefficients(double t, int degree, double* out);
/* heat.cpp:72-96 ; fills scaled (caller frees), coeffs (degree+1), scale, t_eff */
int go_filter_prepare(const go_csr* L, int kind, double lambda_bound, double t, int degree,
                      go_csr* scaled, double* coeffs, double* scale, double* t_eff);
/* heat.cpp:116-131 ; X, Y row-major n x width */
int go_filter_apply(const go_csr* scaled, const double* coeffs, int degree, const double* X,
                    double* Y, int width);

/* heat.cpp:133-162: the implicit-Euler system I + (t/steps) L (upper-triangle entries scaled by
 * h = t/steps, +1 on the diagonal, a missing diagonal becomes 1; mirrored by from_triplets) */
int go_euler_system(const go_csr* L, double t, int steps, go_csr* out);
/* heat.cpp:166-219: `steps` lockstep-CG solves (Solver::lockstep_cg) of the batch X (row-major
 * n x width) into Y; column sums in the blocked order of go_detdot (Eigen's order is unpinned);
 * iters_out (optional) = CG iterations of the last solve */
int go_euler_apply(const go_csr* system, int steps, const double* X, double* Y, int width,
                   int* iters_out);

/* transport.cpp:108-255. mus/nus: P contiguous n-vectors. single_style selects the
 * sinkhorn_single messages. flags bit0: no stagnation abort (bench-only deviation).
 * fail_info[0] = failing pair (Disconnected) or -1, fail_info[1] = sweep of the failure. */
int go_sinkhorn_batch(const go_csr* scaled, const double* coeffs, int degree, double t,
                      const double* a, const double* mus, const double* nus, int P, int max_iter,
                      double tol, int flags, int single_style, double* out_v, double* out_w,
                      double* out_cost, double* out_kl, int* out_iters, int* out_conv,
                      double* out_err, int* fail_info);

/* transport.cpp:257-269: the same batch over EulerHeat (system from go_euler_system) */
int go_euler_sinkhorn_batch(const go_csr* system, int steps, double t, const double* a,
                            const double* mus, const double* nus, int P, int max_iter, double tol,
                            int flags, int single_style, double* out_v, double* out_w,
                            double* out_cost, double* out_kl, int* out_iters, int* out_conv,
                            double* out_err, int* fail_info);

/* barycenter.cpp:45-99. members: m contiguous n-vectors; alphas (m) or NULL for uniform.
 * out_V/out_W: m contiguous n-vectors. */
int go_barycenter(const go_csr* scaled, const double* coeffs, int degree, const double* a,
                  const double* members, int m, const double* alphas, int max_iter, double tol,
                  double* out_bary, double* out_V, double* out_W, int* out_iters, int* out_conv,
                  double* out_err);

/* bench.cpp:32-39 (out nx x ny row-major) and transport.cpp:271-311 (C r x c row-major) */
int go_squared_distances(const double* X, int nx, const double* Y, int ny, int d, double* out);
int go_dense_sinkhorn(const double* C, int r, int c, const double* mu, const double* nu,
                      double lambda, int max_iter, double tol, double* v, double* w,
                      double* cost, double* kl, int* iters, int* conv, double* err);

#ifdef __cplusplus
}
#endif
#endif
