// C++ drop-in API (include/geosink/geosink_b200.hpp) against restated reference tests
// (proj/tests/test_heat.cpp, test_graph.cpp, test_transport.cpp, test_barycenter.cpp). Built and
// run by tests/test_gpu_cpp.py on a GPU box; exit status = number of failed checks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <set>

#include "geosink/geosink_b200.hpp"

using namespace geosink;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    ++g_checks;                                                              \
    if (!(cond)) {                                                           \
      ++g_fail;                                                              \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_CODE(expr, c)                                           \
  do {                                                                       \
    ++g_checks;                                                              \
    bool ok = false;                                                         \
    try {                                                                    \
      expr;                                                                  \
    } catch (const Error& e) {                                               \
      ok = e.code() == (c);                                                  \
    }                                                                        \
    if (!ok) {                                                               \
      ++g_fail;                                                              \
      std::fprintf(stderr, "FAIL %s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #c); \
    }                                                                        \
  } while (0)

// test_util.hpp:20-57 restated
static SparseSymMatrix random_connected_graph(int n, std::uint64_t seed) {
  Rng rng(seed);
  std::set<std::pair<int, int>> edges;
  std::vector<Triplet> trips;
  for (int i = 0; i < n; ++i) {
    const int j = (i + 1) % n;
    edges.emplace(std::min(i, j), std::max(i, j));
    trips.push_back({std::min(i, j), std::max(i, j), rng.uniform(0.3, 1.0)});
  }
  for (int c = 0; c < n; ++c) {
    const int i = (int)rng.below(n), j = (int)rng.below(n);
    const double w = rng.uniform(0.2, 0.8);
    if (i == j || !edges.emplace(std::min(i, j), std::max(i, j)).second) continue;
    trips.push_back({std::min(i, j), std::max(i, j), w});
  }
  return SparseSymMatrix::from_triplets(n, trips);
}
static std::vector<double> random_signal(int n, Rng& rng) {
  std::vector<double> f(n);
  for (auto& x : f) x = rng.normal();
  return f;
}
static Distribution random_distribution(int n, Rng& rng) {
  std::vector<double> w(n);
  for (auto& x : w) x = rng.uniform() + 1e-3;
  return Distribution::from_weights(std::move(w));
}
static double maxabs_diff(const std::vector<double>& a, const std::vector<double>& b) {
  double m = 0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
  return m;
}

int main() {
  // heat: Bessel closed form (test_heat.cpp:87-100) with std::cyl_bessel_i as in the reference
  for (double t : {0.5, 1.0, 5.0, 20.0}) {
    const int degree = 4 * (int)std::ceil(t) + 30;
    const auto b = heat_chebyshev_coefficients(t, degree);
    const double s = std::exp(-t);
    CHECK(std::abs(b[0] - 2.0 * s * std::cyl_bessel_i(0.0, t)) <= 1e-12 * (1 + std::abs(b[0])));
    double sign = -1.0;
    for (int k = 1; k <= std::min(degree, 40); ++k) {
      const double ex = 2.0 * sign * s * std::cyl_bessel_i((double)k, t);
      CHECK(std::abs(b[k] - ex) <= 1e-11 * (1 + std::abs(ex)));
      sign = -sign;
    }
  }
  // two-vertex closed form (test_heat.cpp:135-150)
  {
    const auto lap = laplacian(SparseSymMatrix::from_triplets(2, {{0, 1, 1.0}}), LaplacianKind::combinatorial);
    CHECK(lap.lambda_max_bound >= 2.0 && lap.lambda_max_bound <= 2.02 + 1e-12);
    const HeatFilter f(lap, 1.0, 10);
    const auto out = f.apply({1.0, 0.0});
    CHECK(std::abs(out[0] - 0.5676676416) <= 1e-6 && std::abs(out[1] - 0.4323323584) <= 1e-6);
    const double p = 0.5 * (1 + std::exp(-2.0)), q = 0.5 * (1 - std::exp(-2.0));
    CHECK(maxabs_diff(out, {p, q}) <= 1e-9);
  }
  // batched == per-signal (test_heat.cpp:167-179)
  {
    const auto lap = laplacian(random_connected_graph(40, 9), LaplacianKind::normalized);
    const HeatFilter f(lap, 1.2, 25);
    Rng rng(10);
    RowMajorXd batch(40, 7), out;
    for (int c = 0; c < 7; ++c) batch.set_col(c, random_signal(40, rng));
    f.apply(batch, out);
    for (int c = 0; c < 7; ++c) CHECK(maxabs_diff(out.col(c), f.apply(batch.col(c))) <= 1e-12);
  }
  // constants are fixed points, mass conserved (test_heat.cpp:181-198)
  {
    const auto lap = laplacian(random_connected_graph(35, 5), LaplacianKind::combinatorial);
    const HeatFilter f(lap, 0.8, 30);
    CHECK(maxabs_diff(f.apply(std::vector<double>(35, 1.0)), std::vector<double>(35, 1.0)) <= 1e-9);
  }
  // validation (test_heat.cpp:288-298)
  {
    const auto lap = laplacian(SparseSymMatrix::from_triplets(2, {{0, 1, 1.0}}), LaplacianKind::combinatorial);
    CHECK_THROWS_CODE(HeatFilter(lap, 0.0, 10), errc::non_positive_time);
    CHECK_THROWS_CODE(HeatFilter(lap, 1.0, 0), errc::invalid_argument);
    const HeatFilter f(lap, 1.0, 5);
    CHECK_THROWS_CODE(f.apply(std::vector<double>(3, 0.0)), errc::length_mismatch);
  }
  // graph (test_graph.cpp:41-117)
  {
    PointCloud pc{{0.0, 1.0, 2.0}, 3, 1};
    const auto A = knn_alpha_decay_graph(pc, 1, 2.0);
    CHECK(std::abs(A.coeff(0, 1) - std::exp(-1.0)) <= 1e-12 && A.coeff(0, 2) == 0.0);
    PointCloud tie{{0, 0, 1, 0, 0, 1, -1, 0, 0, -1}, 5, 2};
    const auto T = knn_alpha_decay_graph(tie, 2, 2.0);
    CHECK(T.coeff(2, 3) > 0.0 && T.coeff(3, 4) == 0.0 && T.coeff(1, 4) > 0.0);
    PointCloud dup{{1.0, 1.0}, 2, 1};
    CHECK_THROWS_CODE(knn_alpha_decay_graph(dup, 1, 40.0), errc::duplicate_points);
    const auto L3 = laplacian(SparseSymMatrix::from_triplets(3, {{0, 1, 2.0}}), LaplacianKind::normalized);
    CHECK(L3.matrix.coeff(2, 2) == 1.0 && L3.matrix.coeff(2, 0) == 0.0);
    CHECK_THROWS_CODE(laplacian(SparseSymMatrix::from_triplets(2, {{0, 1, -0.5}}), LaplacianKind::combinatorial),
                      errc::negative_weight);
    CHECK(estimate_lambda_max(SparseSymMatrix::from_triplets(4, {})) == 0.0);
  }
  // transport (test_transport.cpp:224-382)
  {
    const auto lap = laplacian(random_connected_graph(40, 2), LaplacianKind::normalized);
    const HeatFilter f(lap, 1.0, 30);
    const auto u = Distribution::uniform(40);
    const auto res = geodesic_sinkhorn(f, u, u, std::vector<double>(40, 1.0 / 40), {500, 1e-10});
    CHECK(res.converged && res.marginal_error <= 1e-10);
  }
  {
    Rng rng(7);
    const auto lap = laplacian(random_connected_graph(35, 10), LaplacianKind::normalized);
    const HeatFilter f(lap, 0.9, 25);
    const std::vector<double> a(35, 1.0 / 35);
    std::vector<Distribution> mus, nus;
    for (int p = 0; p < 4; ++p) {
      mus.push_back(random_distribution(35, rng));
      nus.push_back(random_distribution(35, rng));
    }
    const auto batch = geodesic_sinkhorn_batch(f, mus, nus, a, {400, 1e-8});
    for (int p = 0; p < 4; ++p) {
      const auto single = geodesic_sinkhorn(f, mus[p], nus[p], a, {400, 1e-8});
      CHECK(batch[p].converged == single.converged && batch[p].iterations == single.iterations);
      CHECK(std::abs(batch[p].cost - single.cost) <= 1e-12 * (1.0 + std::abs(single.cost)));
    }
  }
  {
    const auto lap = laplacian(SparseSymMatrix::from_triplets(4, {{0, 1, 1.0}, {2, 3, 1.0}}),
                               LaplacianKind::combinatorial);
    const HeatFilter f(lap, 1.0, 20);
    CHECK_THROWS_CODE(geodesic_sinkhorn(f, Distribution::indicator(4, {0}), Distribution::indicator(4, {3}),
                                        std::vector<double>(4, 0.25), {500, 1e-9}),
                      errc::disconnected);
  }
  {
    const auto lap = laplacian(random_connected_graph(40, 40), LaplacianKind::normalized);
    const HeatFilter f(lap, 50.0, 3);
    CHECK_THROWS_CODE(geodesic_sinkhorn(f, Distribution::indicator(40, {7}), Distribution::indicator(40, {20}),
                                        std::vector<double>(40, 1.0 / 40), {100, 1e-9}),
                      errc::kernel_not_positive);
  }
  // barycenter (test_barycenter.cpp:72-107)
  {
    std::vector<Triplet> path = {{0, 1, 1.0}, {1, 2, 1.0}};
    const auto lap = laplacian(SparseSymMatrix::from_triplets(3, path), LaplacianKind::combinatorial);
    const HeatFilter f(lap, 0.3, 30);
    DistributionFamily fam;
    fam.members = {Distribution::indicator(3, {0}), Distribution::indicator(3, {2})};
    const auto res = sinkhorn_barycenter(f, fam, std::vector<double>(3, 1.0 / 3), {500, 1e-9});
    CHECK(res.converged);
    CHECK(res.barycenter.weights[1] > res.barycenter.weights[0] && res.barycenter.weights[1] > res.barycenter.weights[2]);
  }
  {
    std::vector<Triplet> cyc;
    for (int i = 0; i < 8; ++i) cyc.push_back({i, (i + 1) % 8, 1.0});
    const auto lap = laplacian(SparseSymMatrix::from_triplets(8, cyc), LaplacianKind::combinatorial);
    const HeatFilter f(lap, 0.5, 30);
    DistributionFamily fam;
    fam.members = {Distribution::indicator(8, {0}), Distribution::indicator(8, {4})};
    const auto res = sinkhorn_barycenter(f, fam, std::vector<double>(8, 1.0 / 8), {500, 1e-10});
    CHECK(res.converged);
    for (int i = 0; i < 8; ++i)
      CHECK(std::abs(res.barycenter.weights[i] - res.barycenter.weights[(i + 4) % 8]) <= 1e-8);
  }
  {
    Rng rng(13);
    const auto lap = laplacian(random_connected_graph(30, 14), LaplacianKind::normalized);
    const HeatFilter f(lap, 0.7, 30);
    const std::vector<double> a(30, 1.0 / 30);
    DistributionFamily t, c;
    for (int i = 0; i < 2; ++i) {
      t.members.push_back(random_distribution(30, rng));
      c.members.push_back(random_distribution(30, rng));
    }
    const double tc = barycentric_distance(f, t, c, a, {500, 1e-8});
    const double ct = barycentric_distance(f, c, t, a, {500, 1e-8});
    CHECK(std::abs(tc - ct) <= 1e-8 * (1.0 + std::abs(tc)));
  }
  // dense Sinkhorn: zero cost gives the product plan (test_transport.cpp:208-215); shape check
  {
    const Distribution mu(std::vector<double>{0.5, 0.3, 0.2}), nu(std::vector<double>{0.2, 0.2, 0.6});
    const auto res = dense_sinkhorn(RowMajorXd(3, 3), mu, nu, 0.7, {500, 1e-12});
    CHECK(res.converged);
    double err = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) err = std::max(err, std::abs(res.v[i] * res.w[j] - mu.weights[i] * nu.weights[j]));
    CHECK(err <= 1e-10);
    CHECK_THROWS_CODE(dense_sinkhorn(RowMajorXd(3, 2), mu, nu, 0.7), errc::length_mismatch);
  }
  // McCann interpolation endpoints (transport.cpp:326-376): s = 0 returns source points
  {
    PointCloud src{{0.0, 1.0, 2.0, 3.0}, 2, 2}, tgt{{5.0, 6.0, 7.0, 8.0, 9.0, 10.0}, 3, 2};
    const auto out = mccann_interpolate(src, tgt, [](int) { return std::vector<double>(3, 1.0 / 6); }, 0.0, 10, 3);
    bool ok = out.n == 10;
    for (int q = 0; q < out.n; ++q) ok = ok && (out.points[2 * q] == 0.0 || out.points[2 * q] == 2.0);
    CHECK(ok);
    CHECK_THROWS_CODE(mccann_interpolate(src, tgt, [](int) { return std::vector<double>(3, 0.1); }, 0.5, 4, 1),
                      errc::degenerate_plan);
  }
  // plan rows rebuild the marginals (acceptance.cpp:168-197); graph file round trip
  {
    Rng rng(4);
    const auto lap = laplacian(random_connected_graph(50, 3), LaplacianKind::normalized);
    const HeatFilter f(lap, 1.0, 40);
    const std::vector<double> a(50, 1.0 / 50);
    const auto mu = random_distribution(50, rng), nu = random_distribution(50, rng);
    const auto res = geodesic_sinkhorn(f, mu, nu, a, {5000, 1e-6});
    CHECK(res.converged);
    double err = 0.0;
    for (int i = 0; i < 50; ++i) {
      const auto row = plan_row(res, f, a, i);
      double srow = 0.0;
      for (double x : row) srow += x;
      err += std::abs(srow - mu.weights[i]);
    }
    CHECK(err <= 1e-6);
    save_graph(lap.matrix, "/tmp/geosink_dropin_graph.txt");
    const auto back = load_graph("/tmp/geosink_dropin_graph.txt");
    CHECK(back.stored_entries() == lap.matrix.stored_entries() && back.values() == lap.matrix.values());
    CHECK_THROWS_CODE(load_graph("/tmp/does/not/exist.txt"), errc::io_error);
  }
  // a single row partition reproduces the unpartitioned engine bit for bit (vertex order aside)
  {
    Rng rng(6);
    const auto lap = laplacian(random_connected_graph(64, 21), LaplacianKind::combinatorial);
    const HeatFilter f(lap, 0.9, 30);
    const std::vector<double> a(64, 1.0 / 64);
    const auto mu = random_distribution(64, rng), nu = random_distribution(64, rng);
    const auto full = geodesic_sinkhorn_batch(f, {mu}, {nu}, a, {300, 1e-9});
    const RowPartition part(f, 1, 0);
    CHECK(part.size() == 64 && part.halo_rows() == 0);
    std::vector<double> ml(64), nl(64), al(64);
    for (int r = 0; r < 64; ++r) {
      ml[r] = mu.weights[part.vertices()[r]];
      nl[r] = nu.weights[part.vertices()[r]];
      al[r] = a[part.vertices()[r]];
    }
    const auto loc = part.sinkhorn({ml}, {nl}, al, {300, 1e-9});
    bool same = loc[0].iterations == full[0].iterations;
    for (int r = 0; r < 64; ++r)
      same = same && loc[0].v[r] == full[0].v[part.vertices()[r]] && loc[0].w[r] == full[0].w[part.vertices()[r]];
    CHECK(same);
    std::vector<double> x(64);
    for (int r = 0; r < 64; ++r) x[r] = rng.normal();
    const auto yf = f.apply(x);
    std::vector<double> xl(64);
    for (int r = 0; r < 64; ++r) xl[r] = x[part.vertices()[r]];
    const auto yl = part.apply(xl);
    bool same_apply = true;
    for (int r = 0; r < 64; ++r) same_apply = same_apply && yl[r] == yf[part.vertices()[r]];
    CHECK(same_apply);
    CHECK_THROWS_CODE(RowPartition(f, 2, 5), errc::invalid_argument);
  }
  // EulerHeat: many implicit steps approach the heat kernel; validation codes
  {
    const auto lap = laplacian(random_connected_graph(40, 8), LaplacianKind::normalized);
    const HeatFilter f(lap, 1.0, 40);
    std::vector<double> x(40);
    for (int i = 0; i < 40; ++i) x[i] = std::sin(0.3 * i);
    const auto ref = f.apply(x);
    const auto y = apply_euler(lap, 1.0, 200, x);
    double e = 0.0, m = 0.0;
    for (int i = 0; i < 40; ++i) {
      e = std::max(e, std::abs(y[i] - ref[i]));
      m = std::max(m, std::abs(ref[i]));
    }
    CHECK(e <= 5e-3 * m);
    CHECK_THROWS_CODE(EulerHeat(lap, -1.0, 2), errc::non_positive_time);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail;
}
