// gs_rng.cpp -- the reference's seeded RNG (proj/include/geosink/rng.hpp:13-68) as host C ABI:
// mt19937_64 raw stream, 53-bit uniforms, Marsaglia polar normals with one cached spare,
// rejection `below`, splitmix `seed_mix`. Used for seeded inputs (workload generators) and the
// power-iteration start vector (graph.cpp:171-174); bit-identical to rng.hpp (tests pin it).
#include <cmath>
#include <cstdint>
#include <random>

#include "geosink_b200.h"

struct gs_rng {
  std::mt19937_64 gen;
  bool have_spare = false;
  double spare = 0.0;
  explicit gs_rng(uint64_t seed) : gen(seed) {}
  double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double normal() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    double u, v, s;
    do {
      u = 2.0 * uniform() - 1.0;
      v = 2.0 * uniform() - 1.0;
      s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    const double m = std::sqrt(-2.0 * std::log(s) / s);
    spare = v * m;
    have_spare = true;
    return u * m;
  }
  uint64_t below(uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
      x = gen();
    } while (x >= limit);
    return x % n;
  }
};

extern "C" {
gs_rng* gs_rng_create(uint64_t seed) { return new gs_rng(seed); }
void gs_rng_destroy(gs_rng* r) { delete r; }
uint64_t gs_rng_bits(gs_rng* r) { return r->gen(); }
double gs_rng_uniform(gs_rng* r) { return r->uniform(); }
double gs_rng_uniform_range(gs_rng* r, double lo, double hi) { return lo + (hi - lo) * r->uniform(); }
double gs_rng_normal(gs_rng* r) { return r->normal(); }
uint64_t gs_rng_below(gs_rng* r, uint64_t n) { return r->below(n); }
uint64_t gs_rng_seed_mix(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// Repeating draw pattern: out[e] for e in [0, count): kind[e % npat] = 0 -> lo + (hi-lo)*U,
// 1 -> hi * N (+ lo), 2 -> below((uint64)hi) as double.
void gs_rng_fill_pattern(gs_rng* r, double* out, int64_t count, const int* kind, const double* lo,
                         const double* hi, int npat) {
  for (int64_t e = 0; e < count; ++e) {
    const int q = (int)(e % npat);
    switch (kind[q]) {
      case 0: out[e] = lo[q] + (hi[q] - lo[q]) * r->uniform(); break;
      case 1: out[e] = lo[q] == 0.0 ? hi[q] * r->normal() : lo[q] + hi[q] * r->normal(); break;
      default: out[e] = (double)r->below((uint64_t)hi[q]); break;
    }
  }
}
}
