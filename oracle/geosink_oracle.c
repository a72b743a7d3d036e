/*
 * geosink_oracle.c -- CPU restatement of the reference Chebyshev-Sinkhorn path.
 *
 * TEST INFRASTRUCTURE ONLY: the parity checker and the CPU baseline. Never linked into or
 * called by the product library. See geosink_oracle.h for the rounding contract
 * (-ffp-contract=off, explicit fma()) and the citation convention: every function names the
 * reference routine it follows as proj/<file>:<lines>.
 */
#include "geosink_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* errc numbering: proj/include/geosink/errors.hpp:10-30 (status = errc + 1) */
enum {
  E_DIMENSION_MISMATCH = 0, E_DUPLICATE_POINTS, E_NEGATIVE_WEIGHT, E_NON_POSITIVE_TIME,
  E_LENGTH_MISMATCH, E_TOO_LARGE, E_INDEX_OUT_OF_RANGE, E_SIZE_MISMATCH, E_DEGENERATE_INPUT,
  E_INVALID_ARGUMENT, E_KERNEL_NOT_POSITIVE, E_DISCONNECTED, E_SOLVE_FAILURE,
  E_NUMERICAL_UNDERFLOW, E_DEGENERATE_PLAN, E_IO_ERROR
};
static const char* kErrcName[] = {
    "DimensionMismatch", "DuplicatePoints", "NegativeWeight", "NonPositiveTime",
    "LengthMismatch", "TooLarge", "IndexOutOfRange", "SizeMismatch", "DegenerateInput",
    "InvalidArgument", "KernelNotPositive", "Disconnected", "SolveFailure",
    "NumericalUnderflow", "DegeneratePlan", "IoError"};

static _Thread_local char g_msg[512];

const char* go_last_error(void) { return g_msg; }

static int fail(int code, const char* fmt, ...) {
  char body[400];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(body, sizeof body, fmt, ap);
  va_end(ap);
  snprintf(g_msg, sizeof g_msg, "%s: %s", kErrcName[code], body);
  return code + 1;
}

#define REQUIRE(cond, code, ...) \
  do {                           \
    if (!(cond)) return fail(code, __VA_ARGS__); \
  } while (0)

/* ------------------------------------------------------------------------------------------
 * Rng: proj/include/geosink/rng.hpp:13-68 (mt19937_64 raw stream, 53-bit uniform, Marsaglia
 * polar normal with one cached spare, rejection `below`, splitmix seed_mix).
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
  int have_spare;
  double spare;
} go_rng;

static void rng_init(go_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->have_spare = 0;
  r->spare = 0.0;
}

static uint64_t rng_next(go_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

static double rng_uniform(go_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static double rng_normal(go_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u, v, s;
  do {
    u = 2.0 * rng_uniform(r) - 1.0;
    v = 2.0 * rng_uniform(r) - 1.0;
    s = u * u + v * v;
  } while (s >= 1.0 || s == 0.0);
  const double m = sqrt(-2.0 * log(s) / s);
  r->spare = v * m;
  r->have_spare = 1;
  return u * m;
}

static uint64_t rng_below(go_rng* r, uint64_t n) {
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = rng_next(r);
  } while (x >= limit);
  return x % n;
}

uint64_t go_rng_seed_mix(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void go_rng_bits(uint64_t seed, int64_t count, uint64_t* out) {
  go_rng r;
  rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng_next(&r);
}
void go_rng_uniform(uint64_t seed, int64_t count, double* out) {
  go_rng r;
  rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng_uniform(&r);
}
void go_rng_normal(uint64_t seed, int64_t count, double* out) {
  go_rng r;
  rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng_normal(&r);
}
void go_rng_below(uint64_t seed, uint64_t bound, int64_t count, uint64_t* out) {
  go_rng r;
  rng_init(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng_below(&r, bound);
}

/* Stateful handle (the reference arm's input generators draw from one Rng across calls, as the
 * reference's own generators do with a geosink::Rng object). */
void* go_rng_new(uint64_t seed) {
  go_rng* r = (go_rng*)malloc(sizeof(go_rng));
  if (r) rng_init(r, seed);
  return r;
}
void go_rng_free(void* r) { free(r); }
uint64_t go_rng_next_bits(void* r) { return rng_next((go_rng*)r); }
double go_rng_next_uniform(void* r) { return rng_uniform((go_rng*)r); }
double go_rng_next_normal(void* r) { return rng_normal((go_rng*)r); }
uint64_t go_rng_next_below(void* r, uint64_t n) { return rng_below((go_rng*)r, n); }
/* repeating draw pattern, kind[e % npat]: 0 -> lo + (hi - lo) U, 1 -> hi N (+ lo), 2 -> below(hi) */
void go_rng_fill_pattern(void* h, double* out, int64_t count, const int* kind, const double* lo,
                         const double* hi, int npat) {
  go_rng* r = (go_rng*)h;
  for (int64_t e = 0; e < count; ++e) {
    const int q = (int)(e % npat);
    switch (kind[q]) {
      case 0: out[e] = lo[q] + (hi[q] - lo[q]) * rng_uniform(r); break;
      case 1: out[e] = lo[q] == 0.0 ? hi[q] * rng_normal(r) : lo[q] + hi[q] * rng_normal(r); break;
      default: out[e] = (double)rng_below(r, (uint64_t)hi[q]); break;
    }
  }
}

/* ------------------------------------------------------------------------------------------
 * Sorting helper: LSD radix sort of (key, value) records by 64-bit key.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  uint64_t key;
  double val;
} kv_t;

static void radix_sort_kv(kv_t* a, int64_t m) {
  if (m <= 1) return;
  kv_t* tmp = (kv_t*)malloc((size_t)m * sizeof(kv_t));
  int64_t* cnt = (int64_t*)malloc(65536 * sizeof(int64_t));
  kv_t *src = a, *dst = tmp;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 16 * pass;
    memset(cnt, 0, 65536 * sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) cnt[(src[i].key >> shift) & 0xFFFF]++;
    int64_t s = 0;
    for (int b = 0; b < 65536; ++b) {
      int64_t c = cnt[b];
      cnt[b] = s;
      s += c;
    }
    for (int64_t i = 0; i < m; ++i) dst[cnt[(src[i].key >> shift) & 0xFFFF]++] = src[i];
    kv_t* t = src;
    src = dst;
    dst = t;
  }
  /* 4 passes: result is back in `a` */
  free(tmp);
  free(cnt);
}

/* ------------------------------------------------------------------------------------------
 * SparseSymMatrix: proj/src/sparse.cpp
 * ---------------------------------------------------------------------------------------- */
void go_csr_free(go_csr* m) {
  if (!m) return;
  free(m->row_offsets);
  free(m->col_indices);
  free(m->values);
  m->row_offsets = NULL;
  m->col_indices = NULL;
  m->values = NULL;
  m->n = 0;
  m->nnz = 0;
}

/* sparse.cpp:15-53 -- mirror, sort by (row, col), merge agreeing duplicates, drop zeros */
int go_csr_from_triplets(int n, int64_t m, const int* rows, const int* cols, const double* vals,
                         go_csr* out) {
  REQUIRE(n >= 0, E_INVALID_ARGUMENT, "negative dimension");
  kv_t* all = (kv_t*)malloc((size_t)(2 * m + 1) * sizeof(kv_t));
  int64_t cnt = 0;
  for (int64_t e = 0; e < m; ++e) {
    const int r = rows[e], c = cols[e];
    if (!(r >= 0 && r < n && c >= 0 && c < n)) {
      free(all);
      return fail(E_INDEX_OUT_OF_RANGE, "triplet index out of range");
    }
    if (!isfinite(vals[e])) {
      free(all);
      return fail(E_INVALID_ARGUMENT, "non-finite matrix entry");
    }
    if (vals[e] == 0.0) continue;
    all[cnt].key = ((uint64_t)(uint32_t)r << 32) | (uint32_t)c;
    all[cnt].val = vals[e];
    ++cnt;
    if (r != c) {
      all[cnt].key = ((uint64_t)(uint32_t)c << 32) | (uint32_t)r;
      all[cnt].val = vals[e];
      ++cnt;
    }
  }
  radix_sort_kv(all, cnt);
  out->n = n;
  out->row_offsets = (int*)calloc((size_t)n + 1, sizeof(int));
  out->col_indices = (int*)malloc((size_t)(cnt + 1) * sizeof(int));
  out->values = (double*)malloc((size_t)(cnt + 1) * sizeof(double));
  int64_t k = 0;
  uint64_t prev = UINT64_MAX;
  for (int64_t e = 0; e < cnt; ++e) {
    if (all[e].key == prev) {
      if (all[e].val != out->values[k - 1]) {
        free(all);
        go_csr_free(out);
        return fail(E_INVALID_ARGUMENT, "conflicting duplicate entries break symmetry");
      }
      continue;
    }
    prev = all[e].key;
    out->col_indices[k] = (int)(uint32_t)(all[e].key & 0xFFFFFFFFu);
    out->values[k] = all[e].val;
    out->row_offsets[(all[e].key >> 32) + 1]++;
    ++k;
  }
  for (int r = 0; r < n; ++r) out->row_offsets[r + 1] += out->row_offsets[r];
  out->nnz = k;
  free(all);
  return 0;
}

int go_csr_from_arrays(int n, int64_t nnz, const int* offs, const int* cols, const double* vals,
                       go_csr* out) {
  out->n = n;
  out->nnz = nnz;
  out->row_offsets = (int*)malloc((size_t)(n + 1) * sizeof(int));
  out->col_indices = (int*)malloc((size_t)(nnz + 1) * sizeof(int));
  out->values = (double*)malloc((size_t)(nnz + 1) * sizeof(double));
  memcpy(out->row_offsets, offs, (size_t)(n + 1) * sizeof(int));
  memcpy(out->col_indices, cols, (size_t)nnz * sizeof(int));
  memcpy(out->values, vals, (size_t)nnz * sizeof(double));
  return 0;
}

/* sparse.cpp:70-99 -- y_i = sum_p vals[p] * x[cols[p]] in CSR order, fma chain from +0.0 */
int go_spmm(const go_csr* m, const double* x, double* y, int width) {
  const int n = m->n;
  const int* offs = m->row_offsets;
  const int* cols = m->col_indices;
  const double* vals = m->values;
  if (width == 1) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int p = offs[i]; p < offs[i + 1]; ++p) acc = fma(vals[p], x[cols[p]], acc);
      y[i] = acc;
    }
    return 0;
  }
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    double* out = y + (size_t)i * width;
    for (int c = 0; c < width; ++c) out[c] = 0.0;
    for (int p = offs[i]; p < offs[i + 1]; ++p) {
      const double v = vals[p];
      const double* xr = x + (size_t)cols[p] * width;
      for (int c = 0; c < width; ++c) out[c] = fma(v, xr[c], out[c]);
    }
  }
  return 0;
}

/* sparse.cpp:107-116 */
double go_gershgorin(const go_csr* m) {
  double bound = 0.0;
  for (int i = 0; i < m->n; ++i) {
    double row = 0.0;
    for (int p = m->row_offsets[i]; p < m->row_offsets[i + 1]; ++p) row += fabs(m->values[p]);
    bound = fmax(bound, row);
  }
  return bound;
}

/* ------------------------------------------------------------------------------------------
 * Deterministic blocked dot product (the device's reduction order):
 * chunks of 4096 = 256 lanes x 16; lane t folds elements c*4096 + j*256 + t (j ascending)
 * with fma from +0.0; 256 lanes fold as a binary tree (v[t] += v[t+s], s = 128..1); chunk
 * partials fold the same way (lane t sums partials t, t+256, ... ascending, then the tree).
 * ---------------------------------------------------------------------------------------- */
#define DET_T 256
#define DET_J 16
#define DET_CHUNK (DET_T * DET_J)

static double tree256(double* v) {
  for (int s = DET_T / 2; s > 0; s >>= 1)
    for (int t = 0; t < s; ++t) v[t] = v[t] + v[t + s];
  return v[0];
}

double go_detdot(const double* x, const double* y, int64_t n) {
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  if (nchunks == 0) return 0.0;
  double* partial = (double*)malloc((size_t)nchunks * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nchunks; ++c) {
    double v[DET_T];
    for (int t = 0; t < DET_T; ++t) {
      double acc = 0.0;
      for (int j = 0; j < DET_J; ++j) {
        const int64_t idx = c * DET_CHUNK + (int64_t)j * DET_T + t;
        if (idx < n) acc = fma(x[idx], y[idx], acc);
      }
      v[t] = acc;
    }
    partial[c] = tree256(v);
  }
  double v[DET_T];
  for (int t = 0; t < DET_T; ++t) {
    double acc = 0.0;
    for (int64_t q = t; q < nchunks; q += DET_T) acc = acc + partial[q];
    v[t] = acc;
  }
  free(partial);
  return tree256(v);
}

/* go_detdot on column c of two row-major n x B matrices (element i at i*B + c) */
static double detdot_col(const double* x, const double* y, int64_t n, int B, int col) {
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  if (nchunks == 0) return 0.0;
  double* partial = (double*)malloc((size_t)nchunks * sizeof(double));
  for (int64_t c = 0; c < nchunks; ++c) {
    double v[DET_T];
    for (int t = 0; t < DET_T; ++t) {
      double acc = 0.0;
      for (int j = 0; j < DET_J; ++j) {
        const int64_t idx = c * DET_CHUNK + (int64_t)j * DET_T + t;
        if (idx < n) acc = fma(x[idx * B + col], y[idx * B + col], acc);
      }
      v[t] = acc;
    }
    partial[c] = tree256(v);
  }
  double v[DET_T];
  for (int t = 0; t < DET_T; ++t) {
    double acc = 0.0;
    for (int64_t q = t; q < nchunks; q += DET_T) acc = acc + partial[q];
    v[t] = acc;
  }
  free(partial);
  return tree256(v);
}

/* ------------------------------------------------------------------------------------------
 * kNN selection: proj/src/graph.cpp:30-71. d2 = max(0, (|xi|^2 + |xj|^2) - 2 <xi,xj>) with the
 * norms and the inner product as fma chains in dimension order; the k smallest (d2, idx) pairs
 * (ties to the lower index) in ascending order; eps = exact distance to the k-th neighbour.
 * ---------------------------------------------------------------------------------------- */
static double sqnorm_row(const double* p, int d) {
  double s = 0.0;
  for (int q = 0; q < d; ++q) s = fma(p[q], p[q], s);
  return s;
}

static double exact_d2(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int q = 0; q < d; ++q) {
    const double diff = a[q] - b[q];
    s = fma(diff, diff, s);
  }
  return s;
}

static void knn_one(const double* pts, const double* sq, int n, int d, int k, int i, int* nb,
                    double* eps_i) {
  double bd[64];
  int bi[64];
  int cnt = 0;
  const double* xi = pts + (size_t)i * d;
  for (int j = 0; j < n; ++j) {
    if (j == i) continue;
    const double* xj = pts + (size_t)j * d;
    double g = 0.0;
    for (int q = 0; q < d; ++q) g = fma(xi[q], xj[q], g);
    double d2 = (sq[i] + sq[j]) - 2.0 * g;
    if (!(d2 > 0.0)) d2 = 0.0; /* std::max(0.0, .) */
    if (cnt == k) {
      if (!(d2 < bd[k - 1] || (d2 == bd[k - 1] && j < bi[k - 1]))) continue;
      --cnt;
    }
    int pos = cnt;
    while (pos > 0 && (d2 < bd[pos - 1] || (d2 == bd[pos - 1] && j < bi[pos - 1]))) {
      bd[pos] = bd[pos - 1];
      bi[pos] = bi[pos - 1];
      --pos;
    }
    bd[pos] = d2;
    bi[pos] = j;
    ++cnt;
  }
  for (int q = 0; q < cnt; ++q) nb[q] = bi[q];
  *eps_i = sqrt(exact_d2(xi, pts + (size_t)bi[cnt - 1] * d, d));
}

int go_knn_rows(const double* pts, int n, int d, int k, const int* rows, int nrows, int* nbrs,
                double* eps) {
  REQUIRE(k >= 1 && k <= 64 && k < n, E_INVALID_ARGUMENT, "bad k");
  double* sq = (double*)malloc((size_t)n * sizeof(double));
  for (int i = 0; i < n; ++i) sq[i] = sqnorm_row(pts + (size_t)i * d, d);
#pragma omp parallel for schedule(dynamic, 16)
  for (int r = 0; r < nrows; ++r) knn_one(pts, sq, n, d, k, rows[r], nbrs + (size_t)r * k, eps + r);
  free(sq);
  return 0;
}

int go_knn(const double* pts, int n, int d, int k, int* nbrs, double* eps) {
  REQUIRE(k >= 1 && k <= 64 && k < n, E_INVALID_ARGUMENT, "bad k");
  double* sq = (double*)malloc((size_t)n * sizeof(double));
  for (int i = 0; i < n; ++i) sq[i] = sqnorm_row(pts + (size_t)i * d, d);
#pragma omp parallel for schedule(dynamic, 16)
  for (int i = 0; i < n; ++i) knn_one(pts, sq, n, d, k, i, nbrs + (size_t)i * k, eps + i);
  free(sq);
  return 0;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* median of the k-NN bandwidths (BASELINE Gaussian kernel; even n: mean of the two middles) */
static double median_of(const double* v, int n) {
  double* s = (double*)malloc((size_t)n * sizeof(double));
  memcpy(s, v, (size_t)n * sizeof(double));
  qsort(s, (size_t)n, sizeof(double), cmp_double);
  const double med = (n % 2) ? s[n / 2] : 0.5 * (s[n / 2 - 1] + s[n / 2]);
  free(s);
  return med;
}

/* graph.cpp:75-108 (+ the Gaussian-median extension, kernel == 1) */
int go_knn_graph(const double* pts, int n, int d, int k, int kernel, double param, go_csr* out,
                 double* sigma_out) {
  REQUIRE(n >= 1 && d >= 1, E_DIMENSION_MISMATCH, "point cloud must be non-empty");
  for (int64_t e = 0; e < (int64_t)n * d; ++e)
    REQUIRE(isfinite(pts[e]), E_DIMENSION_MISMATCH, "point cloud has non-finite entries");
  REQUIRE(k >= 1, E_INVALID_ARGUMENT, "k must be positive");
  REQUIRE(k < n, E_INVALID_ARGUMENT, "k must be < n");
  REQUIRE(k <= 64, E_INVALID_ARGUMENT, "k must be <= 64");
  if (kernel == 0) REQUIRE(param > 0.0, E_INVALID_ARGUMENT, "alpha must be positive");

  int* nbrs = (int*)malloc((size_t)n * k * sizeof(int));
  double* eps = (double*)malloc((size_t)n * sizeof(double));
  go_knn(pts, n, d, k, nbrs, eps);
  for (int i = 0; i < n; ++i)
    if (!(eps[i] > 0.0)) {
      free(nbrs);
      free(eps);
      return fail(E_DUPLICATE_POINTS, "zero k-NN bandwidth at point %d (duplicate points)", i);
    }
  /* union of directed relations, one undirected entry per pair (graph.cpp:91-97) */
  const int64_t m = (int64_t)n * k;
  kv_t* pairs = (kv_t*)malloc((size_t)m * sizeof(kv_t));
  for (int i = 0; i < n; ++i)
    for (int q = 0; q < k; ++q) {
      const int j = nbrs[(size_t)i * k + q];
      const int lo = i < j ? i : j, hi = i < j ? j : i;
      pairs[(size_t)i * k + q].key = ((uint64_t)lo << 32) | (uint32_t)hi;
      pairs[(size_t)i * k + q].val = 0.0;
    }
  radix_sort_kv(pairs, m);
  int64_t u = 0;
  for (int64_t e = 0; e < m; ++e)
    if (u == 0 || pairs[e].key != pairs[u - 1].key) pairs[u++] = pairs[e];

  double sigma2 = 0.0;
  if (kernel == 1) {
    const double sigma = median_of(eps, n);
    if (sigma_out) *sigma_out = sigma;
    sigma2 = sigma * sigma;
  }
  int* ti = (int*)malloc((size_t)u * sizeof(int));
  int* tj = (int*)malloc((size_t)u * sizeof(int));
  double* tv = (double*)malloc((size_t)u * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < u; ++e) {
    const int i = (int)(pairs[e].key >> 32), j = (int)(pairs[e].key & 0xFFFFFFFFu);
    const double d2 = exact_d2(pts + (size_t)i * d, pts + (size_t)j * d, d);
    double w;
    if (kernel == 0) {
      const double dist = sqrt(d2);
      w = 0.5 * (exp(-pow(dist / eps[i], param)) + exp(-pow(dist / eps[j], param)));
    } else {
      w = exp(-(d2 / sigma2));
    }
    ti[e] = i;
    tj[e] = j;
    tv[e] = w;
  }
  const int rc = go_csr_from_triplets(n, u, ti, tj, tv, out);
  free(ti);
  free(tj);
  free(tv);
  free(pairs);
  free(nbrs);
  free(eps);
  return rc;
}

/* ------------------------------------------------------------------------------------------
 * Laplacian and lambda_max: proj/src/graph.cpp:110-194
 * ---------------------------------------------------------------------------------------- */
int go_lambda_max(const go_csr* L, double* out, int* rounds_out) {
  const int n = L->n;
  if (rounds_out) *rounds_out = 0;
  if (n == 0) {
    *out = 0.0;
    return 0;
  }
  double* x = (double*)malloc((size_t)n * sizeof(double));
  double* y = (double*)malloc((size_t)n * sizeof(double));
  go_rng_normal(0x5eed1a4bULL, n, x);
  {
    const double z = go_detdot(x, x, n);
    if (z > 0.0) {
      const double nr = sqrt(z);
      for (int i = 0; i < n; ++i) x[i] = x[i] / nr;
    }
  }
  double estimate = 0.0;
  int converged = 0, it;
  for (it = 0; it < 200; ++it) {
    go_spmm(L, x, y, 1);
    const double norm = sqrt(go_detdot(y, y, n));
    if (norm <= 1e-300) {
      free(x);
      free(y);
      *out = 0.0;
      if (rounds_out) *rounds_out = it + 1;
      return 0;
    }
    const double rayleigh = go_detdot(x, y, n);
    if (it > 0 && fabs(rayleigh - estimate) <= 1e-6 * fabs(rayleigh)) {
      estimate = rayleigh;
      converged = 1;
      break;
    }
    estimate = rayleigh;
    for (int i = 0; i < n; ++i) x[i] = y[i] / norm;
  }
  free(x);
  free(y);
  if (!converged) {
    if (rounds_out) *rounds_out = -1;
    *out = go_gershgorin(L);
    return 0;
  }
  if (rounds_out) *rounds_out = it + 1;
  *out = 1.01 * estimate;
  return 0;
}

int go_laplacian(const go_csr* A, int kind, go_csr* L, double* lambda_bound, int* rounds_out) {
  const int n = A->n;
  const int* offs = A->row_offsets;
  const int* cols = A->col_indices;
  const double* vals = A->values;
  double* degree = (double*)calloc((size_t)n + 1, sizeof(double));
  for (int i = 0; i < n; ++i)
    for (int p = offs[i]; p < offs[i + 1]; ++p) {
      if (!(vals[p] >= 0.0)) {
        free(degree);
        return fail(E_NEGATIVE_WEIGHT, "adjacency entries must be non-negative");
      }
      degree[i] += vals[p];
    }
  const int64_t cap = A->nnz / 2 + n + 1;
  int* ti = (int*)malloc((size_t)cap * sizeof(int));
  int* tj = (int*)malloc((size_t)cap * sizeof(int));
  double* tv = (double*)malloc((size_t)cap * sizeof(double));
  int64_t c = 0;
  int rc;
  if (kind == 0) {
    for (int i = 0; i < n; ++i) {
      double diag = degree[i];
      for (int p = offs[i]; p < offs[i + 1]; ++p) {
        const int j = cols[p];
        if (j == i) diag -= vals[p];
        else if (j > i) { ti[c] = i; tj[c] = j; tv[c] = -vals[p]; ++c; }
      }
      ti[c] = i; tj[c] = i; tv[c] = diag; ++c;
    }
    rc = go_csr_from_triplets(n, c, ti, tj, tv, L);
    if (rc == 0) go_lambda_max(L, lambda_bound, rounds_out);
  } else {
    double* inv_sqrt = (double*)malloc((size_t)n * sizeof(double) + 8);
    for (int i = 0; i < n; ++i) inv_sqrt[i] = 1.0 / sqrt(degree[i] > 0.0 ? degree[i] : 1.0);
    for (int i = 0; i < n; ++i) {
      double diag = 1.0;
      for (int p = offs[i]; p < offs[i + 1]; ++p) {
        const int j = cols[p];
        const double w = vals[p] * inv_sqrt[i] * inv_sqrt[j];
        if (j == i) diag -= w;
        else if (j > i) { ti[c] = i; tj[c] = j; tv[c] = -w; ++c; }
      }
      ti[c] = i; tj[c] = i; tv[c] = diag; ++c;
    }
    free(inv_sqrt);
    rc = go_csr_from_triplets(n, c, ti, tj, tv, L);
    *lambda_bound = 2.0;
    if (rounds_out) *rounds_out = 0;
  }
  free(ti);
  free(tj);
  free(tv);
  free(degree);
  return rc;
}

/* ------------------------------------------------------------------------------------------
 * Chebyshev heat coefficients: proj/src/heat.cpp:14-70
 * ---------------------------------------------------------------------------------------- */
static void scaled_bessel_i(double z, int kmax, int start, double* out /* kmax+1 */) {
  double* f = (double*)calloc((size_t)start + 2, sizeof(double));
  f[start + 1] = 0.0;
  f[start] = 1e-30;
  for (int j = start; j >= 1; --j) {
    f[j - 1] = f[j + 1] + (2.0 * j / z) * f[j];
    if (fabs(f[j - 1]) > 1e250) {
      const double inv = 1e-250;
      for (int q = j - 1; q < start + 2; ++q) f[q] *= inv;
    }
  }
  double norm = f[0];
  for (int j = 1; j <= start; ++j) norm += 2.0 * f[j];
  for (int k = 0; k <= kmax; ++k) out[k] = (k <= start) ? f[k] / norm : 0.0;
  free(f);
}

int go_heat_coefficients(double t, int degree, double* b) {
  REQUIRE(degree >= 1, E_INVALID_ARGUMENT, "Chebyshev degree must be >= 1");
  REQUIRE(t >= 0.0 && isfinite(t), E_NON_POSITIVE_TIME, "diffusion time must be finite and >= 0");
  if (t < 1e-300) {
    for (int k = 0; k <= degree; ++k) b[k] = 0.0;
    b[0] = 2.0;
    return 0;
  }
  int start = degree + (int)ceil(t) + 40 + (int)(2.0 * sqrt((double)degree + t));
  double* cur = (double*)malloc((size_t)(degree + 1) * sizeof(double));
  double* refined = (double*)malloc((size_t)(degree + 1) * sizeof(double));
  scaled_bessel_i(t, degree, start, cur);
  for (int round = 0; round < 8; ++round) {
    const int next_start = start + start / 2 + 20;
    scaled_bessel_i(t, degree, next_start, refined);
    double worst = 0.0;
    for (int k = 0; k <= degree; ++k) {
      const double scale = fmax(fabs(refined[k]), 1e-280);
      worst = fmax(worst, fabs(refined[k] - cur[k]) / scale);
    }
    double* tmp = cur;
    cur = refined;
    refined = tmp;
    start = next_start;
    if (worst <= 1e-13) break;
  }
  b[0] = 2.0 * cur[0];
  double sign = -1.0;
  for (int k = 1; k <= degree; ++k) {
    b[k] = 2.0 * sign * cur[k];
    sign = -sign;
  }
  free(cur);
  free(refined);
  return 0;
}

/* heat.cpp:72-96 */
int go_filter_prepare(const go_csr* L, int kind, double lambda_bound, double t, int degree,
                      go_csr* scaled, double* coeffs, double* scale_out, double* t_eff_out) {
  REQUIRE(t > 0.0 && isfinite(t), E_NON_POSITIVE_TIME, "diffusion time must be > 0");
  REQUIRE(degree >= 1, E_INVALID_ARGUMENT, "Chebyshev degree must be >= 1");
  double scale;
  if (kind == 1) {
    scale = 1.0;
  } else {
    REQUIRE(lambda_bound >= 0.0 && isfinite(lambda_bound), E_INVALID_ARGUMENT,
            "bad lambda_max_bound");
    scale = lambda_bound > 1e-300 ? 2.0 / lambda_bound : 1.0;
  }
  const double t_eff = t / scale;
  const int n = L->n;
  int* ti = (int*)malloc((size_t)(L->nnz + 1) * sizeof(int));
  int* tj = (int*)malloc((size_t)(L->nnz + 1) * sizeof(int));
  double* tv = (double*)malloc((size_t)(L->nnz + 1) * sizeof(double));
  int64_t c = 0;
  for (int i = 0; i < n; ++i)
    for (int p = L->row_offsets[i]; p < L->row_offsets[i + 1]; ++p)
      if (L->col_indices[p] >= i) {
        ti[c] = i;
        tj[c] = L->col_indices[p];
        tv[c] = L->values[p] * scale;
        ++c;
      }
  int rc = go_csr_from_triplets(n, c, ti, tj, tv, scaled);
  free(ti);
  free(tj);
  free(tv);
  if (rc) return rc;
  rc = go_heat_coefficients(t_eff, degree, coeffs);
  if (scale_out) *scale_out = scale;
  if (t_eff_out) *t_eff_out = t_eff;
  return rc;
}

/* heat.cpp:116-131 -- T0 = f; acc = (b0/2) f; T1 = L_s f - f; acc += b1 T1;
 * T_k = 2 (L_s T_{k-1} - T_{k-1}) - T_{k-2}; acc += b_k T_k  (acc += as fma) */
int go_filter_apply(const go_csr* S, const double* b, int degree, const double* X, double* Y,
                    int width) {
  const int64_t len = (int64_t)S->n * width;
  double* prev = (double*)malloc((size_t)(len + 1) * sizeof(double));
  double* cur = (double*)malloc((size_t)(len + 1) * sizeof(double));
  double* tmp = (double*)malloc((size_t)(len + 1) * sizeof(double));
  memcpy(prev, X, (size_t)len * sizeof(double));
  const double b0h = b[0] / 2.0;
  for (int64_t e = 0; e < len; ++e) Y[e] = b0h * X[e];
  go_spmm(S, prev, cur, width);
  for (int64_t e = 0; e < len; ++e) {
    cur[e] = cur[e] - prev[e];
    Y[e] = fma(b[1], cur[e], Y[e]);
  }
  for (int k = 2; k <= degree; ++k) {
    go_spmm(S, cur, tmp, width);
    const double bk = b[k];
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < len; ++e) {
      tmp[e] = 2.0 * (tmp[e] - cur[e]) - prev[e];
      Y[e] = fma(bk, tmp[e], Y[e]);
    }
    double* t = prev;
    prev = cur;
    cur = tmp;
    tmp = t;
  }
  free(prev);
  free(cur);
  free(tmp);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Geodesic Sinkhorn: proj/src/transport.cpp:13-255
 * ---------------------------------------------------------------------------------------- */
#define K_FLOOR 1e-300

/* Distribution::validate (transport.cpp:96-102). The sum uses the blocked tree order of the
 * device (Eigen's sum() is a vectorised blocked reduction too; a plain sequential sum of 1e5
 * equal weights already drifts past the 1e-12 check). */
static double blocked_sum(const double* x, int64_t n) {
  const int64_t nchunks = (n + DET_CHUNK - 1) / DET_CHUNK;
  double total = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) {
    double v[DET_T];
    for (int t = 0; t < DET_T; ++t) {
      double acc = 0.0;
      for (int j = 0; j < DET_J; ++j) {
        const int64_t idx = c * DET_CHUNK + (int64_t)j * DET_T + t;
        if (idx < n) acc = acc + x[idx];
      }
      v[t] = acc;
    }
    total = total + tree256(v);
  }
  return total;
}

static int validate_distribution(const double* w, int n) {
  REQUIRE(n >= 1, E_LENGTH_MISMATCH, "empty distribution");
  for (int i = 0; i < n; ++i) {
    REQUIRE(isfinite(w[i]), E_INVALID_ARGUMENT, "non-finite weights");
    REQUIRE(w[i] >= 0.0, E_INVALID_ARGUMENT, "negative weights");
  }
  REQUIRE(fabs(blocked_sum(w, n) - 1.0) <= 1e-12, E_INVALID_ARGUMENT, "distribution must sum to 1");
  return 0;
}

/* transport.cpp:30-38 (filter_checked) on the n x B row-major block `in`; a-weighted */
/* the heat operator of sinkhorn_many (transport.cpp:144, template <class Op>): the Chebyshev
 * filter or EulerHeat, applied to a row-major n x B block */
typedef struct {
  const go_csr* S;  /* filter: scaled Laplacian; Euler: the system I + (t/steps) L */
  const double* b;  /* filter coefficients (NULL for Euler) */
  int degree;       /* filter degree, or Euler steps */
} heat_op;

static int op_apply(const heat_op* op, const double* x, double* y, int B) {
  if (op->b) return go_filter_apply(op->S, op->b, op->degree, x, y, B);
  return go_euler_apply(op->S, op->degree, x, y, B, NULL);
}

static int apply_weighted(const heat_op* op, const double* a, const double* in, double* tmp,
                          double* out, int n, int B, const char* msg) {
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < B; ++c) tmp[(size_t)i * B + c] = a[i] * in[(size_t)i * B + c];
  const int rc = op_apply(op, tmp, out, B);
  if (rc) return rc;
  for (int c = 0; c < B; ++c) {
    double mx = 0.0, mn = INFINITY;
    for (int i = 0; i < n; ++i) {
      mx = fmax(mx, fabs(tmp[(size_t)i * B + c]));
      mn = fmin(mn, out[(size_t)i * B + c]);
    }
    const double threshold = 1e-12 * mx;
    REQUIRE(mn >= -threshold, E_KERNEL_NOT_POSITIVE, "%s", msg);
  }
  return 0;
}

/* transport.cpp:41-54 */
static double weighted_log_sum(const double* a, const double* mu, const double* s, int n) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i)
    if (mu[i] > 0.0) acc += a[i] * mu[i] * log(s[i]);
  return acc;
}

static int sinkhorn_many(const heat_op* op, double t, const double* a, const double* mus,
                         const double* nus, int P, int max_iter, double tol, int flags,
                         int single_style, double* out_v, double* out_w, double* out_cost,
                         double* out_kl, int* out_iters, int* out_conv, double* out_err,
                         int* fail_info) {
  const int n = op->S->n;
  if (fail_info) {
    fail_info[0] = -1;
    fail_info[1] = 0;
  }
  const char* knp = "heat approximation produced negative mass; increase the degree or diffusion time";
  for (int p = 0; p < P; ++p) {
    int rc = validate_distribution(mus + (size_t)p * n, n);
    if (!rc) rc = validate_distribution(nus + (size_t)p * n, n);
    if (rc) return rc;
    for (int i = 0; i < n; ++i)
      REQUIRE(a[i] > 0.0, E_INVALID_ARGUMENT, "vertex weights must be positive");
    REQUIRE(tol > 0.0, E_INVALID_ARGUMENT, "tolerance must be positive");
    REQUIRE(max_iter >= 1, E_INVALID_ARGUMENT, "max_iter must be >= 1");
  }
  if (P <= 0) return P == 0 ? 0 : fail(E_SIZE_MISMATCH, "pair lists differ in length");
  const double lambda = 4.0 * t;
  int* active = (int*)malloc((size_t)P * sizeof(int));
  int* stagnant = (int*)calloc((size_t)P, sizeof(int));
  int na = P;
  for (int p = 0; p < P; ++p) {
    active[p] = p;
    out_iters[p] = 0;
    out_conv[p] = 0;
    out_err[p] = INFINITY;
  }
  const size_t sz = (size_t)n * P + 1;
  double* M = (double*)malloc(sz * sizeof(double));
  double* N = (double*)malloc(sz * sizeof(double));
  double* V = (double*)calloc(sz, sizeof(double));
  double* W = (double*)malloc(sz * sizeof(double));
  double* phi = (double*)malloc(sz * sizeof(double));
  double* psi = (double*)malloc(sz * sizeof(double));
  double* tmp = (double*)malloc(sz * sizeof(double));
  double* scratch = (double*)malloc(sz * sizeof(double));
  for (int i = 0; i < n; ++i)
    for (int p = 0; p < P; ++p) {
      M[(size_t)i * P + p] = mus[(size_t)p * n + i];
      N[(size_t)i * P + p] = nus[(size_t)p * n + i];
      W[(size_t)i * P + p] = 1.0;
    }
  int rc = apply_weighted(op, a, W, tmp, phi, n, na, knp);
  for (int it = 1; rc == 0 && it <= max_iter && na > 0; ++it) {
    const int B = na;
    for (size_t e = 0; e < (size_t)n * B; ++e) V[e] = M[e] / fmax(phi[e], K_FLOOR);
    rc = apply_weighted(op, a, V, tmp, psi, n, B, knp);
    if (rc) break;
    for (size_t e = 0; e < (size_t)n * B; ++e) W[e] = N[e] / fmax(psi[e], K_FLOOR);
    rc = apply_weighted(op, a, W, tmp, phi, n, B, knp);
    if (rc) break;
    /* transport.cpp:184-226: per-column L1 errors, finalisation, stagnation, compaction */
    int* keep = (int*)malloc((size_t)B * sizeof(int));
    int nk = 0;
    for (int c = 0; c < B; ++c) {
      double err = 0.0;
      for (int i = 0; i < n; ++i) err += fabs(V[(size_t)i * B + c] * phi[(size_t)i * B + c] - M[(size_t)i * B + c]);
      const int pair = active[c];
      out_iters[pair] = it;
      out_err[pair] = err;
      const int done = err <= tol;
      if (done) out_conv[pair] = 1;
      if (done || it == max_iter) {
        for (int i = 0; i < n; ++i) {
          out_v[(size_t)pair * n + i] = V[(size_t)i * B + c];
          out_w[(size_t)pair * n + i] = W[(size_t)i * B + c];
        }
      }
      if (!done) {
        stagnant[pair] = err > 0.5 ? stagnant[pair] + 1 : 0;
        if (!(flags & 1) && !(stagnant[pair] < 50)) {
          if (fail_info) {
            fail_info[0] = pair;
            fail_info[1] = it;
          }
          rc = single_style
                   ? fail(E_DISCONNECTED, "marginal error stagnated above 0.5; are mu and nu in the same graph component?")
                   : fail(E_DISCONNECTED, "marginal error stagnated above 0.5 for pair %d", pair);
          break;
        }
        keep[nk++] = c;
      }
    }
    if (rc == 0 && nk != B) {
      int* still = (int*)malloc((size_t)(nk + 1) * sizeof(int));
      double* arrs[5] = {V, W, M, N, phi};
      for (int q = 0; q < 5; ++q) {
        double* A = arrs[q];
        for (int i = 0; i < n; ++i)
          for (int c = 0; c < nk; ++c) scratch[(size_t)i * nk + c] = A[(size_t)i * B + keep[c]];
        memcpy(A, scratch, (size_t)n * nk * sizeof(double));
      }
      for (int c = 0; c < nk; ++c) still[c] = active[keep[c]];
      memcpy(active, still, (size_t)nk * sizeof(int));
      free(still);
      na = nk;
    }
    free(keep);
  }
  if (rc == 0) {
    for (int p = 0; p < P; ++p) {
      const double* mu = mus + (size_t)p * n;
      const double* nu = nus + (size_t)p * n;
      const double* v = out_v + (size_t)p * n;
      const double* w = out_w + (size_t)p * n;
      out_cost[p] = lambda * (weighted_log_sum(a, mu, v, n) + weighted_log_sum(a, nu, w, n));
      double k1 = 0.0, k2 = 0.0;
      for (int i = 0; i < n; ++i)
        if (mu[i] > 0.0) k1 += mu[i] * log(v[i]);
      for (int i = 0; i < n; ++i)
        if (nu[i] > 0.0) k2 += nu[i] * log(fmax(a[i] * w[i], K_FLOOR));
      out_kl[p] = k1 + k2 - 1.0;
    }
  }
  free(active);
  free(stagnant);
  free(M);
  free(N);
  free(V);
  free(W);
  free(phi);
  free(psi);
  free(tmp);
  free(scratch);
  return rc;
}


int go_sinkhorn_batch(const go_csr* S, const double* b, int degree, double t, const double* a,
                      const double* mus, const double* nus, int P, int max_iter, double tol,
                      int flags, int single_style, double* out_v, double* out_w,
                      double* out_cost, double* out_kl, int* out_iters, int* out_conv,
                      double* out_err, int* fail_info) {
  const heat_op op = {S, b, degree};
  return sinkhorn_many(&op, t, a, mus, nus, P, max_iter, tol, flags, single_style, out_v, out_w,
                       out_cost, out_kl, out_iters, out_conv, out_err, fail_info);
}

/* transport.cpp:257-269: euler_sinkhorn[_batch] = sinkhorn_single / sinkhorn_many over EulerHeat */
int go_euler_sinkhorn_batch(const go_csr* system, int steps, double t, const double* a,
                            const double* mus, const double* nus, int P, int max_iter, double tol,
                            int flags, int single_style, double* out_v, double* out_w,
                            double* out_cost, double* out_kl, int* out_iters, int* out_conv,
                            double* out_err, int* fail_info) {
  const heat_op op = {system, NULL, steps};
  return sinkhorn_many(&op, t, a, mus, nus, P, max_iter, tol, flags, single_style, out_v, out_w,
                       out_cost, out_kl, out_iters, out_conv, out_err, fail_info);
}

/* ------------------------------------------------------------------------------------------
 * Barycenter: proj/src/barycenter.cpp:45-99
 * ---------------------------------------------------------------------------------------- */
int go_barycenter(const go_csr* S, const double* b, int degree, const double* a,
                  const double* members, int m, const double* alphas_in, int max_iter, double tol,
                  double* out_bary, double* out_V, double* out_W, int* out_iters, int* out_conv,
                  double* out_err) {
  const int n = S->n;
  REQUIRE(m >= 1, E_INVALID_ARGUMENT, "family must be non-empty");
  for (int c = 0; c < m; ++c) {
    const int rc = validate_distribution(members + (size_t)c * n, n);
    if (rc) return rc;
  }
  double* alphas = (double*)malloc((size_t)m * sizeof(double));
  for (int c = 0; c < m; ++c) alphas[c] = alphas_in ? alphas_in[c] : 1.0 / (double)m;
  double asum = 0.0;
  for (int c = 0; c < m; ++c) {
    if (!(alphas[c] >= 0.0)) {
      free(alphas);
      return fail(E_INVALID_ARGUMENT, "alphas must be non-negative");
    }
    asum += alphas[c];
  }
  if (!(fabs(asum - 1.0) <= 1e-9)) {
    free(alphas);
    return fail(E_INVALID_ARGUMENT, "alphas must sum to 1");
  }
  for (int i = 0; i < n; ++i)
    if (!(a[i] > 0.0)) {
      free(alphas);
      return fail(E_INVALID_ARGUMENT, "vertex weights must be positive");
    }
  if (!(tol > 0.0 && max_iter >= 1)) {
    free(alphas);
    return fail(E_INVALID_ARGUMENT, "bad parameters");
  }
  const char* knp = "heat filter produced negative mass; increase the Chebyshev degree or diffusion time";
  const size_t sz = (size_t)n * m + 1;
  double* Mb = (double*)malloc(sz * sizeof(double));
  double* V = (double*)calloc(sz, sizeof(double));
  double* W = (double*)malloc(sz * sizeof(double));
  double* phi = (double*)malloc(sz * sizeof(double));
  double* psi = (double*)malloc(sz * sizeof(double));
  double* tmp = (double*)malloc(sz * sizeof(double));
  double* bary = (double*)malloc(((size_t)n + 1) * sizeof(double));
  double* lb = (double*)malloc(((size_t)n + 1) * sizeof(double));
  for (int i = 0; i < n; ++i) {
    bary[i] = 1.0 / n;
    for (int c = 0; c < m; ++c) {
      Mb[(size_t)i * m + c] = members[(size_t)c * n + i];
      W[(size_t)i * m + c] = 1.0;
    }
  }
  *out_iters = 0;
  *out_conv = 0;
  *out_err = INFINITY;
  const heat_op op = {S, b, degree};
  int rc = apply_weighted(&op, a, W, tmp, phi, n, m, knp);
  for (int it = 1; rc == 0 && it <= max_iter; ++it) {
    for (size_t e = 0; e < (size_t)n * m; ++e) V[e] = Mb[e] / fmax(phi[e], K_FLOOR);
    rc = apply_weighted(&op, a, V, tmp, psi, n, m, knp);
    if (rc) break;
    /* barycenter.cpp:75-82: log-domain geometric mean, member order, floor/ceil clamp */
    double mx = -INFINITY;
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int c = 0; c < m; ++c) {
        const double ps = fmin(fmax(psi[(size_t)i * m + c], K_FLOOR), 1e300);
        acc = fma(alphas[c], log(ps), acc);
      }
      lb[i] = acc;
      mx = fmax(mx, acc);
    }
    double mass = 0.0;
    for (int i = 0; i < n; ++i) {
      bary[i] = exp(lb[i] - mx);
      mass += bary[i];
    }
    if (!(mass > 0.0)) {
      rc = fail(E_KERNEL_NOT_POSITIVE, "barycenter iterate collapsed to zero");
      break;
    }
    for (int i = 0; i < n; ++i) bary[i] = bary[i] / mass;
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < m; ++c)
        W[(size_t)i * m + c] = bary[i] / fmax(psi[(size_t)i * m + c], K_FLOOR);
    rc = apply_weighted(&op, a, W, tmp, phi, n, m, knp);
    if (rc) break;
    double err = 0.0;
    for (int c = 0; c < m; ++c) {
      double e = 0.0;
      for (int i = 0; i < n; ++i) e += fabs(V[(size_t)i * m + c] * phi[(size_t)i * m + c] - Mb[(size_t)i * m + c]);
      err = fmax(err, e);
    }
    *out_err = err;
    *out_iters = it;
    if (err <= tol) {
      *out_conv = 1;
      break;
    }
  }
  if (rc == 0) {
    /* barycenter.cpp:94-95 then Distribution::from_weights (transport.cpp:86-94) */
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += bary[i];
    for (int i = 0; i < n; ++i) bary[i] = bary[i] / s;
    for (int pass = 0; pass < 2; ++pass) {
      double tot = 0.0;
      for (int i = 0; i < n; ++i) tot += bary[i];
      for (int i = 0; i < n; ++i) bary[i] = bary[i] / tot;
    }
    memcpy(out_bary, bary, (size_t)n * sizeof(double));
    for (int c = 0; c < m; ++c)
      for (int i = 0; i < n; ++i) {
        out_V[(size_t)c * n + i] = V[(size_t)i * m + c];
        out_W[(size_t)c * n + i] = W[(size_t)i * m + c];
      }
  }
  free(alphas);
  free(Mb);
  free(V);
  free(W);
  free(phi);
  free(psi);
  free(tmp);
  free(bary);
  free(lb);
  return rc;
}

/* ------------------------------------------------------------------------------------------
 * EulerHeat: proj/src/heat.cpp:133-219 (competitor / test oracle).
 * ---------------------------------------------------------------------------------------- */
/* heat.cpp:133-162 */
int go_euler_system(const go_csr* L, double t, int steps, go_csr* out) {
  REQUIRE(t > 0.0 && isfinite(t), E_NON_POSITIVE_TIME, "diffusion time must be > 0");
  REQUIRE(steps >= 1, E_INVALID_ARGUMENT, "substep count must be >= 1");
  const int n = L->n;
  const double h = t / steps;
  int* rows = (int*)malloc((size_t)(L->nnz + n + 1) * sizeof(int));
  int* cols = (int*)malloc((size_t)(L->nnz + n + 1) * sizeof(int));
  double* vals = (double*)malloc((size_t)(L->nnz + n + 1) * sizeof(double));
  int64_t m = 0;
  for (int i = 0; i < n; ++i) {
    int has_diag = 0;
    for (int p = L->row_offsets[i]; p < L->row_offsets[i + 1]; ++p) {
      const int j = L->col_indices[p];
      if (j < i) continue;
      double v = h * L->values[p];
      if (j == i) {
        v = v + 1.0;
        has_diag = 1;
      }
      rows[m] = i;
      cols[m] = j;
      vals[m] = v;
      ++m;
    }
    if (!has_diag) {
      rows[m] = i;
      cols[m] = i;
      vals[m] = 1.0;
      ++m;
    }
  }
  const int rc = go_csr_from_triplets(n, m, rows, cols, vals, out);
  free(rows);
  free(cols);
  free(vals);
  return rc;
}

/* heat.cpp:166-201: every column runs its own CG in lockstep (Solver::lockstep_cg) */
static int euler_solve(const go_csr* A, double* x, int n, int B, int* iters) {
  const size_t len = (size_t)n * B;
  double* b = (double*)malloc(len * sizeof(double));
  double* r = (double*)malloc(len * sizeof(double));
  double* p = (double*)malloc(len * sizeof(double));
  double* ap = (double*)malloc(len * sizeof(double));
  double* rs = (double*)malloc((size_t)B * sizeof(double));
  double* bn = (double*)malloc((size_t)B * sizeof(double));
  double* alpha = (double*)malloc((size_t)B * sizeof(double));
  double* beta = (double*)malloc((size_t)B * sizeof(double));
  int rc = 0;
  memcpy(b, x, len * sizeof(double));
  go_spmm(A, x, ap, B);
  for (size_t e = 0; e < len; ++e) r[e] = b[e] - ap[e];
  memcpy(p, r, len * sizeof(double));
  for (int c = 0; c < B; ++c) {
    rs[c] = detdot_col(r, r, n, B, c);
    bn[c] = fmax(detdot_col(b, b, n, B, c), 1e-300);
  }
  const double tol2 = 1e-10 * 1e-10;
  const long max_iter = 10L * n;
  long it = 0;
  for (;;) {
    int any = 0;
    for (int c = 0; c < B; ++c) any |= rs[c] > tol2 * bn[c];
    if (!any) break;
    if (!(it < max_iter)) {
      rc = fail(E_SOLVE_FAILURE, "conjugate gradient exceeded 10 n iterations");
      break;
    }
    ++it;
    go_spmm(A, p, ap, B);
    for (int c = 0; c < B; ++c) {
      const double pap = detdot_col(p, ap, n, B, c);
      alpha[c] = pap > 0.0 ? rs[c] / pap : 0.0;
    }
    for (size_t e = 0; e < len; ++e) {
      const int c = (int)(e % (size_t)B);
      x[e] = x[e] + p[e] * alpha[c];
      r[e] = r[e] - ap[e] * alpha[c];
    }
    for (int c = 0; c < B; ++c) {
      const double rn = detdot_col(r, r, n, B, c);
      beta[c] = rs[c] > 0.0 ? rn / rs[c] : 0.0;
      rs[c] = rn;
    }
    for (size_t e = 0; e < len; ++e) p[e] = r[e] + p[e] * beta[(int)(e % (size_t)B)];
  }
  if (iters) *iters = (int)it;
  free(b);
  free(r);
  free(p);
  free(ap);
  free(rs);
  free(bn);
  free(alpha);
  free(beta);
  return rc;
}

/* heat.cpp:203-214 */
int go_euler_apply(const go_csr* system, int steps, const double* X, double* Y, int width,
                   int* iters_out) {
  const int n = system->n;
  memcpy(Y, X, (size_t)n * width * sizeof(double));
  for (int s = 0; s < steps; ++s) {
    const int rc = euler_solve(system, Y, n, width, iters_out);
    if (rc) return rc;
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Dense baselines of the kNN benchmark: squared_distances (bench.cpp:32-39) and dense_sinkhorn
 * (transport.cpp:271-311). Eigen's GEMM / GEMV summation orders are unpinned; the restatement
 * fixes them as sequential fma chains in index order (dot products over the coordinates,
 * phi_i over j, psi_j over i, the cost's inner sums over j and outer sum over i) and the
 * marginal error as a sequential sum over i -- the device uses the same orders.
 * ---------------------------------------------------------------------------------------- */
int go_squared_distances(const double* X, int nx, const double* Y, int ny, int d, double* out) {
  REQUIRE(nx >= 0 && ny >= 0 && d >= 1, E_INVALID_ARGUMENT, "bad point set shapes");
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nx; ++i) {
    double xn = 0.0;
    for (int k = 0; k < d; ++k) xn = fma(X[(size_t)i * d + k], X[(size_t)i * d + k], xn);
    for (int j = 0; j < ny; ++j) {
      double yn = 0.0, dot = 0.0;
      for (int k = 0; k < d; ++k) {
        yn = fma(Y[(size_t)j * d + k], Y[(size_t)j * d + k], yn);
        dot = fma(X[(size_t)i * d + k], Y[(size_t)j * d + k], dot);
      }
      const double v = (-2.0 * dot + xn) + yn; /* d = -2 x y^T; d.colwise() += xn; d.rowwise() += yn */
      out[(size_t)i * ny + j] = fmax(v, 0.0);  /* cwiseMax(0) */
    }
  }
  return 0;
}

int go_dense_sinkhorn(const double* C, int r, int c, const double* mu, const double* nu,
                      double lambda, int max_iter, double tol, double* v, double* w,
                      double* cost, double* kl, int* iters, int* conv, double* err) {
  int rc = validate_distribution(mu, r);
  if (!rc) rc = validate_distribution(nu, c);
  if (rc) return rc;
  for (int64_t q = 0; q < (int64_t)r * c; ++q)
    REQUIRE(isfinite(C[q]), E_INVALID_ARGUMENT, "cost matrix has non-finite entries");
  REQUIRE(lambda > 0.0, E_INVALID_ARGUMENT, "lambda must be positive");
  REQUIRE(tol > 0.0 && max_iter >= 1, E_INVALID_ARGUMENT, "bad Sinkhorn parameters");
  double* K = (double*)malloc((size_t)r * c * sizeof(double));
  double* phi = (double*)malloc((size_t)r * sizeof(double));
  for (int64_t q = 0; q < (int64_t)r * c; ++q) K[q] = exp(-C[q] / lambda); /* transport.cpp:282 */
  for (int i = 0; i < r && !rc; ++i) {
    double mx = 0.0;
    for (int j = 0; j < c; ++j) mx = fmax(mx, K[(size_t)i * c + j]);
    if (!(mx > 0.0)) rc = fail(E_NUMERICAL_UNDERFLOW, "kernel row underflowed to zero; increase lambda");
  }
  for (int j = 0; j < c && !rc; ++j) {
    double mx = 0.0;
    for (int i = 0; i < r; ++i) mx = fmax(mx, K[(size_t)i * c + j]);
    if (!(mx > 0.0)) rc = fail(E_NUMERICAL_UNDERFLOW, "kernel column underflowed to zero; increase lambda");
  }
  if (rc) {
    free(K);
    free(phi);
    return rc;
  }
  for (int j = 0; j < c; ++j) w[j] = 1.0;
  for (int i = 0; i < r; ++i) v[i] = 0.0;
  *conv = 0;
  *iters = 0;
  *err = INFINITY;
  for (int i = 0; i < r; ++i) { /* phi = K w */
    double s = 0.0;
    for (int j = 0; j < c; ++j) s = fma(K[(size_t)i * c + j], w[j], s);
    phi[i] = s;
  }
  for (int it = 1; it <= max_iter; ++it) {
    for (int i = 0; i < r; ++i) v[i] = mu[i] / fmax(phi[i], K_FLOOR);
    for (int j = 0; j < c; ++j) {
      double s = 0.0;
      for (int i = 0; i < r; ++i) s = fma(K[(size_t)i * c + j], v[i], s);
      w[j] = nu[j] / fmax(s, K_FLOOR);
    }
    double e = 0.0;
    for (int i = 0; i < r; ++i) {
      double s = 0.0;
      for (int j = 0; j < c; ++j) s = fma(K[(size_t)i * c + j], w[j], s);
      phi[i] = s;
      e = e + fabs(v[i] * s - mu[i]);
    }
    *err = e;
    *iters = it;
    if (e <= tol) {
      *conv = 1;
      break;
    }
  }
  double cs = 0.0;
  for (int i = 0; i < r; ++i) {
    double t = 0.0;
    for (int j = 0; j < c; ++j) t = fma(K[(size_t)i * c + j] * C[(size_t)i * c + j], w[j], t);
    cs = fma(v[i], t, cs);
  }
  *cost = cs;
  double k1 = 0.0, k2 = 0.0;
  for (int i = 0; i < r; ++i)
    if (mu[i] > 0.0) k1 += mu[i] * log(fmax(v[i], K_FLOOR));
  for (int j = 0; j < c; ++j)
    if (nu[j] > 0.0) k2 += nu[j] * log(fmax(w[j], K_FLOOR));
  *kl = k1 + k2 - 1.0;
  free(K);
  free(phi);
  return 0;
}
