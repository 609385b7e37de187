// Drives the reference API (fmoe/moe_layer.hpp) through libfmoe_dropin.so and
// dumps every result into argv[1] as f64 sections (count, values): forward with a cache, backward,
// backward with an edited copy of the cache, then three train_steps and the
// parameters they leave.  tests/test_dropin.py runs it on the device-resident
// route (default) and on the operator composition (FMOE_DROPIN_PATH=ops) and
// compares the dumps.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fmoe/moe_layer.hpp"
#include "fmoe/rng.hpp"

using namespace fmoe;

// one section: element count (as a double), then the values
static void dump(std::FILE* f, const Matrix& m) {
  const double n = (double)m.size();
  std::fwrite(&n, sizeof(double), 1, f);
  std::fwrite(m.data(), sizeof(double), m.size(), f);
}

// FAST_ROUTE_ROUND_BF16=1: inputs and weight matrices rounded to bf16 values
// (round to nearest even through fp32), biases to fp32 -- the values the bf16
// layer stores -- so both runs of the reduced-precision comparison start from
// the same numbers (the oracle is fed the rounded values)
static double round_bf16(double v) {
  float f = (float)v;
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
  std::memcpy(&f, &u, 4);
  return f;
}
static void round_matrix(Matrix& m, bool to_bf16) {
  for (std::size_t i = 0; i < m.size(); ++i) m.data()[i] = to_bf16 ? round_bf16(m.data()[i]) : (double)(float)m.data()[i];
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::size_t n = argc > 2 ? std::atoi(argv[2]) : 512, d = argc > 3 ? std::atoi(argv[3]) : 128,
                    h = argc > 4 ? std::atoi(argv[4]) : 256, e = argc > 5 ? std::atoi(argv[5]) : 8, k = 2;
  MoEConfig cfg{n, d, h, k, e, 1, 7};
  MoELayerState st = init_state(cfg);
  Matrix x(n, d), dy(n, d), tgt(n, d);
  UniformRng(stream_seed(7, 102)).fill(x, -1.0, 1.0);
  UniformRng(stream_seed(7, 103)).fill(dy, -1.0, 1.0);
  UniformRng(stream_seed(7, 104)).fill(tgt, -1.0, 1.0);
  if (const char* r = std::getenv("FAST_ROUTE_ROUND_BF16"); r && *r == '1') {
    for (Matrix* m : {&x, &dy, &tgt, &st.gate.w_g}) round_matrix(*m, true);
    for (auto& p : st.experts) {
      round_matrix(p.w1, true);
      round_matrix(p.w2, true);
      round_matrix(p.b1, false);
      round_matrix(p.b2, false);
    }
  }
  std::FILE* f = std::fopen(argv[1], "wb");
  MoEForwardCache cache;
  const Matrix y = forward(x, st, nullptr, &cache);
  dump(f, y);
  dump(f, cache.gate_out.scores);
  dump(f, cache.gate_out.topk_scores);
  dump(f, cache.expert_outputs);
  for (const auto& c : cache.expert_caches) {
    dump(f, c.input);
    dump(f, c.preact);
    dump(f, c.hidden);
  }
  auto [dx, g] = backward(dy, cache, st);
  dump(f, dx);
  dump(f, g.d_wg);
  for (const auto& eg : g.experts) {
    dump(f, eg.d_w1);
    dump(f, eg.d_b1);
    dump(f, eg.d_w2);
    dump(f, eg.d_b2);
  }
  // an edited copy of the cache must be honoured (the device route falls back)
  MoEForwardCache edited = cache;
  edited.expert_outputs(0, 0) += 0.5;
  auto [dx2, g2] = backward(dy, edited, st);
  dump(f, dx2);
  dump(f, g2.d_wg);
  for (int s = 0; s < 3; ++s) {
    Matrix loss(1, 1);
    loss(0, 0) = train_step(x, tgt, st, 0.05);
    dump(f, loss);
  }
  dump(f, st.gate.w_g);
  for (const auto& p : st.experts) {
    dump(f, p.w1);
    dump(f, p.b1);
    dump(f, p.w2);
    dump(f, p.b2);
  }
  // forward after training, from the updated (device-resident) parameters
  dump(f, forward(x, st));
  std::fclose(f);
  std::printf("ok\n");
  return 0;
}
