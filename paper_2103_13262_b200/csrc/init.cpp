// init.cpp -- init_state on the host (moe_layer.cpp:28-45, gate.cpp:16-21,
// expert.cpp:13-22, rng.hpp:12-28, rng.cpp:6-11).
//
// The reference draws weights from std::mt19937_64 keyed by splitmix64
// substreams; the B200 layer uses the identical generators so a model
// initialised here is the reference's model (fp64 values, rounded once to the
// layer dtype).  Experts are generated on parallel host threads; each expert
// is its own sequential stream, so the result does not depend on threading.
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "init.h"

namespace fmoe_b200 {

uint64_t stream_seed(uint64_t base, uint64_t stream) {
  uint64_t z = base + 0x9E3779B97F4A7C15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

namespace {
constexpr uint64_t kGateStream = 0x67617465ULL;  // "gate" (gate.cpp:14)

// UniformRng::next (rng.hpp:17-20) as the reference build evaluates it:
// lo + u*(hi-lo) contracted to one fused multiply-add.
inline double next_uniform(std::mt19937_64& g, double lo, double span) {
  const double u = static_cast<double>(g() >> 11) * 0x1.0p-53;
  return std::fma(u, span, lo);
}

void fill(std::mt19937_64& g, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = next_uniform(g, -0.1, 0.2);
}
}  // namespace

void init_gate_host(uint64_t seed, int64_t d_m, int64_t total, double* wg) {
  std::mt19937_64 g(stream_seed(seed, kGateStream));
  fill(g, wg, d_m * total);
}

void init_experts_host(uint64_t seed, int64_t first_global, int64_t count, int64_t d_m, int64_t d_h,
                       double* w1, double* b1, double* w2, double* b2) {
  auto one = [&](int64_t s) {
    std::mt19937_64 g(stream_seed(seed, static_cast<uint64_t>(first_global + s)));
    fill(g, w1 + s * d_m * d_h, d_m * d_h);
    fill(g, b1 + s * d_h, d_h);
    fill(g, w2 + s * d_h * d_m, d_h * d_m);
    fill(g, b2 + s * d_m, d_m);
  };
  const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
  const int64_t nthreads = std::min<int64_t>(hw, count);
  if (nthreads <= 1) {
    for (int64_t s = 0; s < count; ++s) one(s);
    return;
  }
  std::vector<std::thread> pool;
  for (int64_t t = 0; t < nthreads; ++t)
    pool.emplace_back([&, t] {
      for (int64_t s = t; s < count; s += nthreads) one(s);
    });
  for (auto& th : pool) th.join();
}

}  // namespace fmoe_b200
