// init.h -- host-side reference-identical weight generation (init.cpp).
#pragma once
#include <cstdint>

namespace fmoe_b200 {
uint64_t stream_seed(uint64_t base, uint64_t stream);
void init_gate_host(uint64_t seed, int64_t d_m, int64_t total, double* wg);
void init_experts_host(uint64_t seed, int64_t first_global, int64_t count, int64_t d_m, int64_t d_h,
                       double* w1, double* b1, double* w2, double* b2);
}  // namespace fmoe_b200
