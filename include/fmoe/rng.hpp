// fmoe/rng.hpp -- the reference's seeded generators (reference:
// proj/include/fmoe/rng.hpp, proj/src/rng.cpp:6-11): mt19937_64 streams keyed by
// stream_seed(base, id), uniform doubles lo + u*(hi - lo) with u the top 53
// bits.  The reference build contracts that expression into one fma; it is
// written as std::fma here so the bits do not depend on compiler flags.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

#include "fmoe/matrix.hpp"

namespace fmoe {

std::uint64_t stream_seed(std::uint64_t base_seed, std::uint64_t stream_id);

class UniformRng {
 public:
  explicit UniformRng(std::uint64_t seed) : gen_(seed) {}

  double next(double lo, double hi) {
    const double u = static_cast<double>(gen_() >> 11) * 0x1.0p-53;
    return std::fma(u, hi - lo, lo);
  }
  void fill(Matrix& m, double lo, double hi) {
    for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = next(lo, hi);
  }

 private:
  std::mt19937_64 gen_;
};

}  // namespace fmoe
