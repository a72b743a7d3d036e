// geosink_b200.hpp -- C++ drop-in for the reference `geosink` hot-path API, header-only, over the
// C ABI in geosink_b200.h (link libgeosink_b200.so). Names, arguments, results and exceptions
// follow /root/reference/proj/include/geosink/{errors,rng,sparse,graph,heat,transport,
// barycenter}.hpp; Eigen types are replaced by std::vector<double> (vertex signals) and
// `RowMajorXd` (n x B row-major block, as the reference's RowMajorXd). Every compute call runs on
// the GPU; there is no CPU path.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <cstdlib>
#include <limits>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "geosink_b200.h"

namespace geosink {

// ---- errors.hpp:10-85 -------------------------------------------------------------------------
enum class errc {
  dimension_mismatch, duplicate_points, negative_weight, non_positive_time, length_mismatch,
  too_large, index_out_of_range, size_mismatch, degenerate_input, invalid_argument,
  kernel_not_positive, disconnected, solve_failure, numerical_underflow, degenerate_plan, io_error,
};

class Error : public std::runtime_error {
 public:
  Error(errc code, const std::string& what_full) : std::runtime_error(what_full), code_(code) {}
  errc code() const noexcept { return code_; }
  bool is_validation() const noexcept {
    switch (code_) {
      case errc::kernel_not_positive: case errc::disconnected: case errc::solve_failure:
      case errc::numerical_underflow: case errc::degenerate_plan: case errc::io_error:
        return false;
      default:
        return true;
    }
  }
  bool is_io() const noexcept { return code_ == errc::io_error; }

 private:
  errc code_;
};

class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
// One engine context per process (device 0 unless GEOSINK_DEVICE is set).
inline gs_ctx* ctx() {
  static std::unique_ptr<gs_ctx, void (*)(gs_ctx*)> c(
      [] {
        gs_ctx* h = nullptr;
        const char* d = std::getenv("GEOSINK_DEVICE");
        if (gs_ctx_create(d ? std::atoi(d) : 0, &h) != GS_OK)
          throw DeviceError("geosink: no usable CUDA device for the B200 engine");
        return h;
      }(),
      gs_ctx_destroy);
  return c.get();
}
inline void check(int rc) {
  if (rc == GS_OK) return;
  const std::string msg = gs_last_error(ctx());
  if (rc >= 1 && rc <= 16) throw Error(static_cast<errc>(rc - 1), msg);
  throw DeviceError(msg);
}
[[noreturn]] inline void fail(errc c, const char* name, const std::string& what) {
  throw Error(c, std::string(name) + ": " + what);
}
}  // namespace detail

// ---- rng.hpp:13-68 ----------------------------------------------------------------------------
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : seed_(seed), h_(gs_rng_create(seed), gs_rng_destroy) {}
  Rng fork(std::uint64_t stream) const { return Rng(seed_mix(seed_, stream)); }
  std::uint64_t bits() { return gs_rng_bits(h_.get()); }
  double uniform() { return gs_rng_uniform(h_.get()); }
  double uniform(double lo, double hi) { return gs_rng_uniform_range(h_.get(), lo, hi); }
  double normal() { return gs_rng_normal(h_.get()); }
  std::uint64_t below(std::uint64_t n) { return gs_rng_below(h_.get(), n); }
  static std::uint64_t seed_mix(std::uint64_t a, std::uint64_t b) { return gs_rng_seed_mix(a, b); }

 private:
  std::uint64_t seed_;
  std::shared_ptr<gs_rng> h_;
};

// ---- sparse.hpp:23-61 -------------------------------------------------------------------------
struct RowMajorXd {  // n x B, row-major (sparse.hpp:14)
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<double> data_;
  RowMajorXd() = default;
  RowMajorXd(std::size_t r, std::size_t c) : rows_(r), cols_(c), data_(r * c, 0.0) {}
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  const double* data() const { return data_.data(); }
  double& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
  double operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
  std::vector<double> col(std::size_t j) const {
    std::vector<double> v(rows_);
    for (std::size_t i = 0; i < rows_; ++i) v[i] = (*this)(i, j);
    return v;
  }
  void set_col(std::size_t j, const std::vector<double>& v) {
    for (std::size_t i = 0; i < rows_; ++i) (*this)(i, j) = v[i];
  }
};

namespace detail {
inline std::vector<double> to_columns(const RowMajorXd& x) {  // B contiguous n-vectors
  std::vector<double> out(x.rows() * x.cols());
  for (std::size_t j = 0; j < x.cols(); ++j)
    for (std::size_t i = 0; i < x.rows(); ++i) out[j * x.rows() + i] = x(i, j);
  return out;
}
inline void from_columns(const std::vector<double>& c, RowMajorXd& y) {
  for (std::size_t j = 0; j < y.cols(); ++j)
    for (std::size_t i = 0; i < y.rows(); ++i) y(i, j) = c[j * y.rows() + i];
}
}  // namespace detail

struct Triplet {
  int row;
  int col;
  double value;
};

class SparseSymMatrix {
 public:
  SparseSymMatrix() = default;
  static SparseSymMatrix from_triplets(int n, const std::vector<Triplet>& entries) {
    std::vector<int> r(entries.size()), c(entries.size());
    std::vector<double> v(entries.size());
    for (std::size_t e = 0; e < entries.size(); ++e) {
      r[e] = entries[e].row;
      c[e] = entries[e].col;
      v[e] = entries[e].value;
    }
    gs_graph* g = nullptr;
    detail::check(gs_graph_from_triplets(detail::ctx(), n, (int64_t)entries.size(), r.data(), c.data(),
                                         v.data(), GS_MEM_HOST, &g));
    return SparseSymMatrix(g, true);
  }
  int size() const { return h_ ? info().first : 0; }
  std::int64_t stored_entries() const { return h_ ? info().second : 0; }
  const std::vector<int>& row_offsets() const { return host().offs; }
  const std::vector<int>& col_indices() const { return host().cols; }
  const std::vector<double>& values() const { return host().vals; }
  double coeff(int i, int j) const {
    if (i < 0 || i >= size() || j < 0 || j >= size())
      detail::fail(errc::index_out_of_range, "IndexOutOfRange", "coeff index");
    const auto& H = host();
    for (int p = H.offs[i]; p < H.offs[i + 1]; ++p)
      if (H.cols[p] == j) return H.vals[p];
    return 0.0;
  }
  std::vector<double> multiply(const std::vector<double>& x) const {
    if ((int)x.size() != size()) detail::fail(errc::length_mismatch, "LengthMismatch", "matvec size");
    std::vector<double> y(x.size());
    detail::check(gs_graph_multiply(detail::ctx(), h_.get(), x.data(), y.data(), 1, GS_MEM_HOST));
    return y;
  }
  void multiply(const RowMajorXd& x, RowMajorXd& y) const {
    if ((int)x.rows() != size()) detail::fail(errc::length_mismatch, "LengthMismatch", "matmat size");
    const auto cols = detail::to_columns(x);
    std::vector<double> out(cols.size());
    detail::check(gs_graph_multiply(detail::ctx(), h_.get(), cols.data(), out.data(), (int)x.cols(),
                                    GS_MEM_HOST));
    y = RowMajorXd(x.rows(), x.cols());
    detail::from_columns(out, y);
  }
  double gershgorin_bound() const {
    double b = 0.0;
    detail::check(gs_graph_gershgorin(detail::ctx(), h_.get(), &b));
    return b;
  }
  double max_abs() const {
    double m = 0.0;
    for (double v : values()) m = std::max(m, std::abs(v));
    return m;
  }
  gs_graph* handle() const { return h_.get(); }
  explicit SparseSymMatrix(gs_graph* g, bool owned)
      : h_(g, owned ? gs_graph_destroy : [](gs_graph*) {}) {}

 private:
  struct Host {
    std::vector<int> offs, cols;
    std::vector<double> vals;
  };
  std::pair<int, std::int64_t> info() const {
    int n = 0;
    int64_t nnz = 0;
    gs_graph_info(h_.get(), &n, &nnz);
    return {n, nnz};
  }
  const Host& host() const {
    if (!host_) {
      auto h = std::make_shared<Host>();
      const auto [n, nnz] = info();
      h->offs.resize(n + 1);
      h->cols.resize(nnz);
      h->vals.resize(nnz);
      detail::check(gs_graph_download(detail::ctx(), h_.get(), h->offs.data(), h->cols.data(),
                                      h->vals.data(), GS_MEM_HOST));
      host_ = h;
    }
    return *host_;
  }
  std::shared_ptr<gs_graph> h_;
  mutable std::shared_ptr<Host> host_;
};

// ---- graph.hpp:10-42 --------------------------------------------------------------------------
enum class LaplacianKind { combinatorial, normalized };

struct GraphLaplacian {
  SparseSymMatrix matrix;
  LaplacianKind kind = LaplacianKind::combinatorial;
  double lambda_max_bound = 0.0;
  int size() const { return matrix.size(); }
};

struct PointCloud {  // pointcloud.hpp:11-25 (row-major n x d)
  std::vector<double> points;
  int n = 0, d = 0;
};

inline SparseSymMatrix knn_alpha_decay_graph(const PointCloud& cloud, int k, double alpha) {
  gs_graph* g = nullptr;
  detail::check(gs_knn_graph(detail::ctx(), cloud.points.data(), cloud.n, cloud.d, k,
                             GS_KERNEL_ALPHA_DECAY, alpha, GS_MEM_HOST, &g, nullptr));
  return SparseSymMatrix(g, true);
}

inline GraphLaplacian laplacian(const SparseSymMatrix& A, LaplacianKind kind) {
  gs_graph* L = nullptr;
  double lam = 0.0;
  detail::check(gs_laplacian(detail::ctx(), A.handle(), static_cast<int>(kind), &L, &lam, nullptr));
  return GraphLaplacian{SparseSymMatrix(L, true), kind, lam};
}

inline double estimate_lambda_max(const SparseSymMatrix& L) {
  double lam = 0.0;
  detail::check(gs_lambda_max(detail::ctx(), L.handle(), &lam, nullptr));
  return lam;
}

// ---- heat.hpp:12-54 ---------------------------------------------------------------------------
inline std::vector<double> heat_chebyshev_coefficients(double t, int degree) {
  if (degree < 1) detail::fail(errc::invalid_argument, "InvalidArgument", "Chebyshev degree must be >= 1");
  std::vector<double> b(degree + 1);
  detail::check(gs_heat_coefficients(detail::ctx(), t, degree, b.data()));
  return b;
}

class HeatFilter {
 public:
  HeatFilter(const GraphLaplacian& lap, double t, int degree) {
    gs_filter* f = nullptr;
    detail::check(gs_filter_create(detail::ctx(), lap.matrix.handle(), static_cast<int>(lap.kind),
                                   lap.lambda_max_bound, t, degree, &f));
    h_ = std::shared_ptr<gs_filter>(f, gs_filter_destroy);
    int n = 0, dg = 0, kd = 0;
    gs_filter_info(f, &n, &t_, &t_eff_, &scale_, &dg, &kd);
    n_ = n;
    degree_ = dg;
    kind_ = static_cast<LaplacianKind>(kd);
    coeff_.resize(dg + 1);
    gs_filter_coefficients(f, coeff_.data());
  }
  std::vector<double> apply(const std::vector<double>& f) const {
    if ((int)f.size() != n_) detail::fail(errc::length_mismatch, "LengthMismatch", "signal length");
    std::vector<double> y(f.size());
    detail::check(gs_filter_apply(detail::ctx(), h_.get(), f.data(), y.data(), 1, GS_MEM_HOST));
    return y;
  }
  void apply(const RowMajorXd& signals, RowMajorXd& out) const {
    if ((int)signals.rows() != n_) detail::fail(errc::length_mismatch, "LengthMismatch", "signal length");
    const auto cols = detail::to_columns(signals);
    std::vector<double> y(cols.size());
    detail::check(gs_filter_apply(detail::ctx(), h_.get(), cols.data(), y.data(), (int)signals.cols(),
                                  GS_MEM_HOST));
    out = RowMajorXd(signals.rows(), signals.cols());
    detail::from_columns(y, out);
  }
  int size() const { return n_; }
  double time() const { return t_; }
  double effective_time() const { return t_eff_; }
  double scale() const { return scale_; }
  int degree() const { return degree_; }
  const std::vector<double>& coefficients() const { return coeff_; }
  SparseSymMatrix scaled_laplacian() const {
    return SparseSymMatrix(const_cast<gs_graph*>(gs_filter_scaled(h_.get())), false);
  }
  LaplacianKind kind() const { return kind_; }
  gs_filter* handle() const { return h_.get(); }

 private:
  std::shared_ptr<gs_filter> h_;
  int n_ = 0, degree_ = 0;
  double t_ = 0, t_eff_ = 0, scale_ = 1;
  LaplacianKind kind_ = LaplacianKind::combinatorial;
  std::vector<double> coeff_;
};

// ---- heat.hpp:60-84: EulerHeat (implicit Euler: direct below n = 4000 in the automatic mode, the
// reference's lockstep conjugate gradient above) ------------------------------------------------
class EulerHeat {
 public:
  enum class Solver { automatic, direct, lockstep_cg };
  EulerHeat(const GraphLaplacian& lap, double t, int steps, Solver solver = Solver::automatic)
      : n_(lap.size()), steps_(steps), t_(t) {
    gs_euler* e = nullptr;
    const int code = solver == Solver::direct ? GS_EULER_DIRECT
                     : solver == Solver::lockstep_cg ? GS_EULER_LOCKSTEP_CG : GS_EULER_AUTOMATIC;
    detail::check(gs_euler_create_ex(detail::ctx(), lap.matrix.handle(), t, steps, code, &e));
    h_ = std::shared_ptr<gs_euler>(e, gs_euler_destroy);
  }
  std::vector<double> apply(const std::vector<double>& f) const {
    if ((int)f.size() != n_) detail::fail(errc::length_mismatch, "LengthMismatch", "signal length");
    std::vector<double> y(f.size());
    detail::check(gs_euler_apply(detail::ctx(), h_.get(), f.data(), y.data(), 1, GS_MEM_HOST, nullptr));
    return y;
  }
  void apply(const RowMajorXd& signals, RowMajorXd& out) const {
    if ((int)signals.rows() != n_) detail::fail(errc::length_mismatch, "LengthMismatch", "signal length");
    const auto cols = detail::to_columns(signals);
    std::vector<double> y(cols.size());
    detail::check(gs_euler_apply(detail::ctx(), h_.get(), cols.data(), y.data(), (int)signals.cols(),
                                 GS_MEM_HOST, nullptr));
    out = RowMajorXd(signals.rows(), signals.cols());
    detail::from_columns(y, out);
  }
  int size() const { return n_; }
  int steps() const { return steps_; }
  double time() const { return t_; }
  gs_euler* handle() const { return h_.get(); }

 private:
  int n_ = 0, steps_ = 1;
  double t_ = 0.0;
  std::shared_ptr<gs_euler> h_;
};

inline std::vector<double> apply_euler(const GraphLaplacian& lap, double t, int steps, const std::vector<double>& f) {
  return EulerHeat(lap, t, steps).apply(f);
}

// ---- transport.hpp:14-69 ----------------------------------------------------------------------
struct Distribution {
  std::vector<double> weights;
  Distribution() = default;
  explicit Distribution(std::vector<double> w) : weights(std::move(w)) { validate(); }
  static Distribution uniform(int n) {
    if (n < 1) detail::fail(errc::invalid_argument, "InvalidArgument", "empty support");
    return Distribution(std::vector<double>(n, 1.0 / n));
  }
  static Distribution indicator(int n, const std::vector<int>& vertices) {
    if (vertices.empty()) detail::fail(errc::invalid_argument, "InvalidArgument", "empty indicator set");
    std::vector<double> w(n, 0.0);
    for (int v : vertices) {
      if (v < 0 || v >= n) detail::fail(errc::index_out_of_range, "IndexOutOfRange", "indicator vertex out of range");
      w[v] += 1.0;
    }
    const double s = std::accumulate(w.begin(), w.end(), 0.0);
    for (double& x : w) x /= s;
    return Distribution(std::move(w));
  }
  static Distribution from_weights(std::vector<double> w) {
    if (w.empty()) detail::fail(errc::invalid_argument, "InvalidArgument", "empty weight vector");
    for (double x : w)
      if (!(x >= 0.0)) detail::fail(errc::invalid_argument, "InvalidArgument", "weights must be non-negative");
    const double total = std::accumulate(w.begin(), w.end(), 0.0);
    if (!(total > 0.0 && std::isfinite(total)))
      detail::fail(errc::invalid_argument, "InvalidArgument", "weights must have positive mass");
    for (double& x : w) x /= total;
    const double s2 = std::accumulate(w.begin(), w.end(), 0.0);
    for (double& x : w) x /= s2;
    return Distribution(std::move(w));
  }
  std::size_t size() const { return weights.size(); }
  void validate() const {
    if (weights.empty()) detail::fail(errc::length_mismatch, "LengthMismatch", "empty distribution");
    double s = 0.0;
    for (double x : weights) {
      if (!std::isfinite(x)) detail::fail(errc::invalid_argument, "InvalidArgument", "non-finite weights");
      if (x < 0.0) detail::fail(errc::invalid_argument, "InvalidArgument", "negative weights");
      s += x;
    }
    if (!(std::abs(s - 1.0) <= 1e-12)) detail::fail(errc::invalid_argument, "InvalidArgument", "distribution must sum to 1");
  }
};

struct SinkhornParams {
  int max_iter = 500;
  double tol = 1e-6;
};

struct TransportResult {
  std::vector<double> v, w;
  double cost = 0.0;
  double kl = 0.0;
  double lambda = 0.0;
  int iterations = 0;
  bool converged = false;
  double marginal_error = std::numeric_limits<double>::infinity();
  double kl_form_cost() const { return std::sqrt(lambda * std::max(0.0, 1.0 + kl)); }
  double normalized_cost() const { return 2.0 * kl_form_cost(); }
  double dual_cost() const { return lambda * (1.0 + kl); }
};

namespace detail {
inline std::vector<TransportResult> sinkhorn(const HeatFilter& f, const std::vector<Distribution>& mus,
                                             const std::vector<Distribution>& nus,
                                             const std::vector<double>& a, const SinkhornParams& p,
                                             int flags) {
  if (mus.size() != nus.size()) fail(errc::size_mismatch, "SizeMismatch", "pair lists differ in length");
  const int n = f.size(), P = static_cast<int>(mus.size());
  if (P == 0) return {};
  std::vector<double> M(size_t(P) * n), N(size_t(P) * n), v(M.size()), w(M.size());
  for (int q = 0; q < P; ++q) {
    if ((int)mus[q].size() != n || (int)nus[q].size() != n)
      fail(errc::length_mismatch, "LengthMismatch", "distributions must live on the filter's graph");
    std::copy(mus[q].weights.begin(), mus[q].weights.end(), M.begin() + size_t(q) * n);
    std::copy(nus[q].weights.begin(), nus[q].weights.end(), N.begin() + size_t(q) * n);
  }
  if ((int)a.size() != n) fail(errc::length_mismatch, "LengthMismatch", "vertex weights must live on the filter's graph");
  std::vector<double> cost(P), kl(P), err(P);
  std::vector<int> it(P), conv(P);
  check(gs_sinkhorn(ctx(), f.handle(), a.data(), M.data(), N.data(), P, p.max_iter, p.tol, flags,
                    GS_MEM_HOST, v.data(), w.data(), cost.data(), kl.data(), it.data(), conv.data(),
                    err.data(), nullptr, nullptr));
  std::vector<TransportResult> out(P);
  for (int q = 0; q < P; ++q) {
    out[q].v.assign(v.begin() + size_t(q) * n, v.begin() + size_t(q + 1) * n);
    out[q].w.assign(w.begin() + size_t(q) * n, w.begin() + size_t(q + 1) * n);
    out[q].cost = cost[q];
    out[q].kl = kl[q];
    out[q].lambda = 4.0 * f.time();
    out[q].iterations = it[q];
    out[q].converged = conv[q] != 0;
    out[q].marginal_error = err[q];
  }
  return out;
}
}  // namespace detail

inline TransportResult geodesic_sinkhorn(const HeatFilter& filter, const Distribution& mu,
                                         const Distribution& nu, const std::vector<double>& a,
                                         const SinkhornParams& params = {}) {
  return detail::sinkhorn(filter, {mu}, {nu}, a, params, GS_FLAG_SINGLE)[0];
}

inline std::vector<TransportResult> geodesic_sinkhorn_batch(const HeatFilter& filter,
                                                            const std::vector<Distribution>& mus,
                                                            const std::vector<Distribution>& nus,
                                                            const std::vector<double>& a,
                                                            const SinkhornParams& params = {}) {
  return detail::sinkhorn(filter, mus, nus, a, params, 0);
}

// transport.cpp:257-269: Sinkhorn over EulerHeat (the competitor of the Chebyshev filter)
inline std::vector<TransportResult> euler_sinkhorn_batch(const EulerHeat& euler, const std::vector<Distribution>& mus,
                                                         const std::vector<Distribution>& nus,
                                                         const std::vector<double>& a,
                                                         const SinkhornParams& params = {}, int flags = 0) {
  if (mus.size() != nus.size()) detail::fail(errc::size_mismatch, "SizeMismatch", "pair lists differ in length");
  const int n = euler.size(), P = static_cast<int>(mus.size());
  if (P == 0) return {};
  std::vector<double> M(size_t(P) * n), N(M.size()), v(M.size()), w(M.size());
  for (int q = 0; q < P; ++q) {
    if ((int)mus[q].size() != n || (int)nus[q].size() != n)
      detail::fail(errc::length_mismatch, "LengthMismatch", "distributions must live on the filter's graph");
    std::copy(mus[q].weights.begin(), mus[q].weights.end(), M.begin() + size_t(q) * n);
    std::copy(nus[q].weights.begin(), nus[q].weights.end(), N.begin() + size_t(q) * n);
  }
  std::vector<double> cost(P), kl(P), err(P);
  std::vector<int> it(P), conv(P);
  detail::check(gs_euler_sinkhorn(detail::ctx(), euler.handle(), a.data(), M.data(), N.data(), P, params.max_iter,
                                  params.tol, flags, GS_MEM_HOST, v.data(), w.data(), cost.data(), kl.data(),
                                  it.data(), conv.data(), err.data(), nullptr, nullptr));
  std::vector<TransportResult> out(P);
  for (int q = 0; q < P; ++q) {
    out[q].v.assign(v.begin() + size_t(q) * n, v.begin() + size_t(q + 1) * n);
    out[q].w.assign(w.begin() + size_t(q) * n, w.begin() + size_t(q + 1) * n);
    out[q].cost = cost[q];
    out[q].kl = kl[q];
    out[q].lambda = 4.0 * euler.time();
    out[q].iterations = it[q];
    out[q].converged = conv[q] != 0;
    out[q].marginal_error = err[q];
  }
  return out;
}

inline TransportResult euler_sinkhorn(const EulerHeat& euler, const Distribution& mu, const Distribution& nu,
                                      const std::vector<double>& a, const SinkhornParams& params = {}) {
  return euler_sinkhorn_batch(euler, {mu}, {nu}, a, params, GS_FLAG_SINGLE)[0];
}

// transport.cpp:271-311: dense entropic Sinkhorn (the kNN benchmark's baseline); cost is r x c
// row-major (RowMajorXd with n = r rows, B = c columns)
inline TransportResult dense_sinkhorn(const RowMajorXd& cost, const Distribution& mu, const Distribution& nu,
                                      double lambda, const SinkhornParams& params = {}) {
  TransportResult res;
  res.v.resize(cost.rows());
  res.w.resize(cost.cols());
  res.lambda = lambda;
  if (mu.size() != (std::size_t)cost.rows() || nu.size() != (std::size_t)cost.cols()) {
    mu.validate();
    nu.validate();
    detail::fail(errc::length_mismatch, "LengthMismatch", "cost matrix shape does not match the marginals");
  }
  int it = 0, conv = 0;
  detail::check(gs_dense_sinkhorn(detail::ctx(), cost.data(), (int)cost.rows(), (int)cost.cols(),
                                  mu.weights.data(), nu.weights.data(), lambda, params.max_iter, params.tol,
                                  GS_MEM_HOST, res.v.data(), res.w.data(), &res.cost, &res.kl, &it, &conv,
                                  &res.marginal_error));
  res.iterations = it;
  res.converged = conv != 0;
  return res;
}

// transport.cpp:326-376: McCann interpolation at time s by sampling the plan (source rows by
// their mass, then a target within the row); sums are sequential in index order
inline PointCloud mccann_interpolate(const PointCloud& source, const PointCloud& target,
                                     const std::function<std::vector<double>(int)>& plan_row_fn, double s,
                                     int num_samples, std::uint64_t rng_seed) {
  auto check_cloud = [](const PointCloud& c) {
    if (c.n < 1 || c.d < 1) detail::fail(errc::dimension_mismatch, "DimensionMismatch", "point cloud must be non-empty");
    for (double x : c.points)
      if (!std::isfinite(x)) detail::fail(errc::dimension_mismatch, "DimensionMismatch", "point cloud has non-finite entries");
  };
  check_cloud(source);
  check_cloud(target);
  if (source.d != target.d) detail::fail(errc::size_mismatch, "SizeMismatch", "source and target dimensions differ");
  if (!(s >= 0.0 && s <= 1.0)) detail::fail(errc::invalid_argument, "InvalidArgument", "interpolation time must be in [0, 1]");
  if (num_samples < 1) detail::fail(errc::invalid_argument, "InvalidArgument", "need at least one sample");
  const int ms = source.n, mt = target.n;
  std::vector<double> cum(ms);
  double acc = 0.0;
  for (int i = 0; i < ms; ++i) {
    const std::vector<double> row = plan_row_fn(i);
    if ((int)row.size() != mt) detail::fail(errc::length_mismatch, "LengthMismatch", "plan row has wrong length");
    double m = 0.0;
    for (double x : row) m += std::max(x, 0.0);
    acc += m;
    cum[i] = acc;
  }
  const double total = acc;
  if (!(total >= 1.0 - 1e-6))
    detail::fail(errc::degenerate_plan, "DegeneratePlan", "plan mass below 1; transport result unusable for interpolation");
  Rng rng(rng_seed);
  std::vector<int> counts(ms, 0);
  for (int q = 0; q < num_samples; ++q) {
    const double u = rng.uniform() * total;
    const int i = (int)(std::lower_bound(cum.begin(), cum.end(), u) - cum.begin());
    ++counts[std::min(i, ms - 1)];
  }
  PointCloud out;
  out.n = num_samples;
  out.d = source.d;
  out.points.resize((size_t)num_samples * source.d);
  int written = 0;
  std::vector<double> rc(mt);
  for (int i = 0; i < ms; ++i) {
    if (counts[i] == 0) continue;
    const std::vector<double> row = plan_row_fn(i);
    double a2 = 0.0;
    for (int j = 0; j < mt; ++j) rc[j] = (a2 += std::max(row[j], 0.0));
    if (!(a2 > 0.0)) detail::fail(errc::degenerate_plan, "DegeneratePlan", "sampled an empty plan row");
    for (int q = 0; q < counts[i]; ++q) {
      const double u = rng.uniform() * a2;
      const int j = std::min((int)(std::lower_bound(rc.begin(), rc.end(), u) - rc.begin()), mt - 1);
      for (int k = 0; k < source.d; ++k)
        out.points[(size_t)written * source.d + k] =
            (1.0 - s) * source.points[(size_t)i * source.d + k] + s * target.points[(size_t)j * target.d + k];
      ++written;
    }
  }
  return out;
}

// ---- next: plan rows, graph file IO ---------------------------------------------
// transport.cpp:314-324
inline std::vector<double> plan_row(const TransportResult& result, const HeatFilter& filter,
                                    const std::vector<double>& a, int i) {
  const int n = filter.size();
  if ((int)result.v.size() != n || (int)result.w.size() != n)
    detail::fail(errc::length_mismatch, "LengthMismatch", "result does not match the filter's graph");
  std::vector<double> row(n);
  detail::check(gs_plan_rows(detail::ctx(), filter.handle(), a.data(), result.v.data(),
                             result.w.data(), &i, 1, GS_MEM_HOST, row.data()));
  return row;
}

// sparse.cpp:137-174
inline void save_graph(const SparseSymMatrix& m, const std::string& path) {
  if (gs_graph_save(detail::ctx(), m.handle(), path.c_str()) != 0)
    detail::fail(errc::io_error, "IoError", "cannot write '" + path + "'");
}
inline SparseSymMatrix load_graph(const std::string& path) {
  gs_graph* g = nullptr;
  const int rc = gs_graph_load(detail::ctx(), path.c_str(), &g);
  if (rc == 16) detail::fail(errc::io_error, "IoError", "cannot read graph file '" + path + "'");
  detail::check(rc);
  return SparseSymMatrix(g, true);
}

// ---- barycenter.hpp:11-42 ---------------------------------------------------------------------
struct DistributionFamily {
  std::vector<Distribution> members;
  std::vector<double> alphas;  // empty means uniform
  std::string label;
  std::vector<double> resolved_alphas() const {
    if (alphas.empty()) return std::vector<double>(members.size(), 1.0 / members.size());
    return alphas;
  }
  void validate(int n) const {
    if (members.empty()) detail::fail(errc::invalid_argument, "InvalidArgument", "family must be non-empty");
    for (const auto& m : members) {
      m.validate();
      if ((int)m.size() != n) detail::fail(errc::length_mismatch, "LengthMismatch", "family members must share the graph");
    }
    const auto al = resolved_alphas();
    if (al.size() != members.size()) detail::fail(errc::length_mismatch, "LengthMismatch", "one alpha per member required");
    double s = 0.0;
    for (double x : al) {
      if (!(x >= 0.0)) detail::fail(errc::invalid_argument, "InvalidArgument", "alphas must be non-negative");
      s += x;
    }
    if (!(std::abs(s - 1.0) <= 1e-9)) detail::fail(errc::invalid_argument, "InvalidArgument", "alphas must sum to 1");
  }
};

struct BarycenterResult {
  Distribution barycenter;
  std::vector<std::pair<std::vector<double>, std::vector<double>>> scalings;
  int iterations = 0;
  bool converged = false;
  double marginal_error = std::numeric_limits<double>::infinity();
};

inline BarycenterResult sinkhorn_barycenter(const HeatFilter& filter, const DistributionFamily& family,
                                            const std::vector<double>& a,
                                            const SinkhornParams& params = {}) {
  const int n = filter.size();
  family.validate(n);
  if ((int)a.size() != n) detail::fail(errc::length_mismatch, "LengthMismatch", "vertex weights must live on the filter's graph");
  const int m = static_cast<int>(family.members.size());
  std::vector<double> M(size_t(m) * n), V(M.size()), W(M.size()), bary(n);
  for (int c = 0; c < m; ++c)
    std::copy(family.members[c].weights.begin(), family.members[c].weights.end(), M.begin() + size_t(c) * n);
  const auto al = family.resolved_alphas();
  int it = 0, conv = 0;
  double err = 0.0;
  detail::check(gs_barycenter(detail::ctx(), filter.handle(), a.data(), M.data(), m, al.data(),
                              params.max_iter, params.tol, GS_MEM_HOST, nullptr, bary.data(), V.data(),
                              W.data(), &it, &conv, &err));
  BarycenterResult res;
  res.barycenter.weights = std::move(bary);
  for (int c = 0; c < m; ++c)
    res.scalings.emplace_back(std::vector<double>(V.begin() + size_t(c) * n, V.begin() + size_t(c + 1) * n),
                              std::vector<double>(W.begin() + size_t(c) * n, W.begin() + size_t(c + 1) * n));
  res.iterations = it;
  res.converged = conv != 0;
  res.marginal_error = err;
  return res;
}

inline double barycentric_distance(const HeatFilter& filter, const DistributionFamily& family_t,
                                   const DistributionFamily& family_c, const std::vector<double>& a,
                                   const SinkhornParams& params = {}) {
  const auto bt = sinkhorn_barycenter(filter, family_t, a, params);
  const auto bc = sinkhorn_barycenter(filter, family_c, a, params);
  return geodesic_sinkhorn(filter, bt.barycenter, bc.barycenter, a, params).cost;
}

// ---- row partitions (multi-GPU row-partitioned applies) ---------------------
// One rank's contiguous nnz-balanced rows of a filter. Local vectors are indexed like vertices()
// (original vertex ids). `comm` carries the caller's collectives (allreduce + alltoallv on the
// given stream); it may be null only for a single part.
class RowPartition {
 public:
  RowPartition(const HeatFilter& filter, int nparts, int part) : filter_(&filter) {
    gs_part* p = nullptr;
    detail::check(gs_part_create(detail::ctx(), filter.handle(), nparts, part, &p));
    h_ = std::shared_ptr<gs_part>(p, gs_part_destroy);
    int rb = 0, re = 0;
    detail::check(gs_part_info(p, &rb, &re, &n_halo_, nullptr, nullptr));
    vertices_.resize(re - rb);
    detail::check(gs_part_vertices(detail::ctx(), p, vertices_.data(), GS_MEM_HOST));
  }
  int size() const { return static_cast<int>(vertices_.size()); }
  int halo_rows() const { return n_halo_; }
  const std::vector<int>& vertices() const { return vertices_; }
  // heat.cpp:98-114 on the local rows
  std::vector<double> apply(const std::vector<double>& f_local, const gs_comm* comm = nullptr) const {
    if ((int)f_local.size() != size()) detail::fail(errc::length_mismatch, "LengthMismatch", "signal length");
    std::vector<double> y(f_local.size());
    detail::check(gs_part_filter_apply(detail::ctx(), h_.get(), comm, f_local.data(), y.data(), 1, 0, GS_MEM_HOST));
    return y;
  }
  // geodesic_sinkhorn_batch (transport.cpp:249-255) on the local rows: v, w local; scalars global
  std::vector<TransportResult> sinkhorn(const std::vector<std::vector<double>>& mus_local,
                                        const std::vector<std::vector<double>>& nus_local,
                                        const std::vector<double>& a_local, const SinkhornParams& params = {},
                                        const gs_comm* comm = nullptr, int flags = 0) const {
    if (mus_local.size() != nus_local.size())
      detail::fail(errc::size_mismatch, "SizeMismatch", "pair lists differ in length");
    const int n = size(), P = static_cast<int>(mus_local.size());
    if (P == 0) return {};
    std::vector<double> M(size_t(P) * n), N(M.size()), v(M.size()), w(M.size());
    for (int q = 0; q < P; ++q) {
      if ((int)mus_local[q].size() != n || (int)nus_local[q].size() != n)
        detail::fail(errc::length_mismatch, "LengthMismatch", "distributions must live on the partition");
      std::copy(mus_local[q].begin(), mus_local[q].end(), M.begin() + size_t(q) * n);
      std::copy(nus_local[q].begin(), nus_local[q].end(), N.begin() + size_t(q) * n);
    }
    if ((int)a_local.size() != n)
      detail::fail(errc::length_mismatch, "LengthMismatch", "vertex weights must live on the partition");
    std::vector<double> cost(P), kl(P), err(P);
    std::vector<int> it(P), conv(P);
    detail::check(gs_part_sinkhorn(detail::ctx(), h_.get(), comm, a_local.data(), M.data(), N.data(), P,
                                   params.max_iter, params.tol, flags, GS_MEM_HOST, v.data(), w.data(),
                                   cost.data(), kl.data(), it.data(), conv.data(), err.data(), nullptr,
                                   nullptr));
    std::vector<TransportResult> out(P);
    for (int q = 0; q < P; ++q) {
      out[q].v.assign(v.begin() + size_t(q) * n, v.begin() + size_t(q + 1) * n);
      out[q].w.assign(w.begin() + size_t(q) * n, w.begin() + size_t(q + 1) * n);
      out[q].cost = cost[q];
      out[q].kl = kl[q];
      out[q].lambda = 4.0 * filter_->time();
      out[q].iterations = it[q];
      out[q].converged = conv[q] != 0;
      out[q].marginal_error = err[q];
    }
    return out;
  }
  gs_part* handle() const { return h_.get(); }

 private:
  const HeatFilter* filter_;
  std::shared_ptr<gs_part> h_;
  int n_halo_ = 0;
  std::vector<int> vertices_;
};

}  // namespace geosink
