// Test infrastructure: exposes the reference's own header-only RNG
// (/root/reference/proj/include/geosink/rng.hpp, compiled from where it lies) through a C ABI so
// tests can pin oracle/geosink_oracle.c's restatement (go_rng_*) against it bit for bit.
// This is the only part of the reference that compiles here: every other translation unit
// includes Eigen3, which is absent.
#include <cstdint>

#include "geosink/rng.hpp"

extern "C" {
void ref_rng_bits(std::uint64_t seed, std::int64_t count, std::uint64_t* out) {
  geosink::Rng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.bits();
}
void ref_rng_uniform(std::uint64_t seed, std::int64_t count, double* out) {
  geosink::Rng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.uniform();
}
void ref_rng_normal(std::uint64_t seed, std::int64_t count, double* out) {
  geosink::Rng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.normal();
}
void ref_rng_below(std::uint64_t seed, std::uint64_t bound, std::int64_t count, std::uint64_t* out) {
  geosink::Rng r(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = r.below(bound);
}
std::uint64_t ref_rng_seed_mix(std::uint64_t a, std::uint64_t b) { return geosink::Rng::seed_mix(a, b); }
}
