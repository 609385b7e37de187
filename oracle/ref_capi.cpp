// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A flat C entry-point layer over the UNMODIFIED reference implementation
// (/root/reference/proj/src/*.cpp), compiled side by side with the namespace
// renamed (-Dfmoe=fmoe_ref, see oracle/Makefile) into oracle/_ref/libfmoe_ref.so.
// It lets the Python tests and bench.py (--impl reference, cpu_baseline) drive
// the reference's own public API -- gate_forward, build_plan, scatter,
// gather_combine, expert_forward/backward, init_state, forward/backward and the
// expert-parallel collectives over its InProcWorld -- with plain buffers.
//
// Status codes mirror the B200 C-ABI (include/fmoe_b200.h): 0 ok, 1 ShapeError,
// 2 ProtocolError, 3 TransportError, 5 anything else.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "fmoe/checkpoint.hpp"
#include "fmoe/collectives.hpp"
#include "fmoe/dispatch.hpp"
#include "fmoe/errors.hpp"
#include "fmoe/expert.hpp"
#include "fmoe/gate.hpp"
#include "fmoe/matrix.hpp"
#include "fmoe/moe_layer.hpp"
#include "fmoe/rng.hpp"
#include "fmoe/transport.hpp"

using namespace fmoe_ref;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 2;
  } catch (const TransportError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

Matrix to_matrix(const double* p, int64_t r, int64_t c) {
  Matrix m(static_cast<std::size_t>(r), static_cast<std::size_t>(c));
  if (r * c > 0) std::memcpy(m.data(), p, sizeof(double) * static_cast<std::size_t>(r * c));
  return m;
}
IndexMatrix to_index(const int64_t* p, int64_t r, int64_t c) {
  IndexMatrix m(static_cast<std::size_t>(r), static_cast<std::size_t>(c));
  if (r * c > 0) std::memcpy(m.data(), p, sizeof(int64_t) * static_cast<std::size_t>(r * c));
  return m;
}
void out_matrix(const Matrix& m, double* p) {
  if (p && m.size()) std::memcpy(p, m.data(), sizeof(double) * m.size());
}
void out_vec(const std::vector<int64_t>& v, int64_t* p) {
  if (p && !v.empty()) std::memcpy(p, v.data(), sizeof(int64_t) * v.size());
}

DispatchPlan plan_from(const int64_t* idx, int64_t n, int64_t k, int64_t e) {
  return build_plan(to_index(idx, n, k), static_cast<std::size_t>(e));
}

ExpertParams expert_from(const double* w1, const double* b1, const double* w2, const double* b2,
                         int64_t d, int64_t h) {
  return ExpertParams{to_matrix(w1, d, h), to_matrix(b1, 1, h), to_matrix(w2, h, d),
                      to_matrix(b2, 1, d), ParamTag::NoSync};
}

MoELayerState state_from(int64_t n, int64_t d, int64_t h, int64_t e_local, int64_t k,
                         int64_t world, int rank, const double* wg, const double* w1,
                         const double* b1, const double* w2, const double* b2) {
  MoEConfig cfg;
  cfg.n_b = static_cast<std::size_t>(n);
  cfg.d_m = static_cast<std::size_t>(d);
  cfg.d_h = static_cast<std::size_t>(h);
  cfg.k = static_cast<std::size_t>(k);
  cfg.n_e_local = static_cast<std::size_t>(e_local);
  cfg.world_size = static_cast<std::size_t>(world);
  MoELayerState st;
  st.config = cfg;
  st.topology = {static_cast<int>(world), 1};
  st.rank = rank;
  st.gate = GateParams{to_matrix(wg, d, e_local * world), ParamTag::World};
  for (int64_t s = 0; s < e_local; ++s) {
    const int64_t g = rank * e_local + s;
    st.experts.push_back(expert_from(w1 + g * d * h, b1 + g * h, w2 + g * h * d, b2 + g * d, d, h));
  }
  return st;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_stream_seed(uint64_t base, uint64_t id) { return stream_seed(base, id); }

void ref_uniform_fill(uint64_t seed, double* out, int64_t n, double lo, double hi) {
  UniformRng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.next(lo, hi);
}

// init_state(config, rank) for a single worker holding all `e` experts.
int ref_init_state(uint64_t seed, int64_t d, int64_t h, int64_t e, int64_t k, double* wg,
                   double* w1, double* b1, double* w2, double* b2) {
  return guarded([&] {
    MoEConfig cfg;
    cfg.n_b = 1;
    cfg.d_m = static_cast<std::size_t>(d);
    cfg.d_h = static_cast<std::size_t>(h);
    cfg.k = static_cast<std::size_t>(k);
    cfg.n_e_local = static_cast<std::size_t>(e);
    cfg.world_size = 1;
    cfg.seed = seed;
    const MoELayerState st = init_state(cfg, 0);
    out_matrix(st.gate.w_g, wg);
    for (int64_t g = 0; g < e; ++g) {
      out_matrix(st.experts[g].w1, w1 + g * d * h);
      out_matrix(st.experts[g].b1, b1 + g * h);
      out_matrix(st.experts[g].w2, w2 + g * h * d);
      out_matrix(st.experts[g].b2, b2 + g * d);
    }
  });
}

int ref_matmul(const double* a, const double* b, double* out, int64_t m, int64_t p, int64_t n) {
  return guarded([&] { out_matrix(matmul(to_matrix(a, m, p), to_matrix(b, p, n)), out); });
}

int ref_softmax_rows(const double* a, double* out, int64_t r, int64_t c) {
  return guarded([&] { out_matrix(softmax_rows(to_matrix(a, r, c)), out); });
}

int ref_topk_rows(const double* a, int64_t r, int64_t c, int64_t k, int64_t* idx, double* vals) {
  return guarded([&] {
    const TopK t = topk_rows(to_matrix(a, r, c), static_cast<std::size_t>(k));
    std::memcpy(idx, t.indices.data(), sizeof(int64_t) * t.indices.size());
    out_matrix(t.values, vals);
  });
}

int ref_gate_forward(const double* x, const double* wg, int64_t n, int64_t d, int64_t e,
                     int64_t k, double* scores, int64_t* idx, double* vals) {
  return guarded([&] {
    const GateOutput o = gate_forward(to_matrix(x, n, d), GateParams{to_matrix(wg, d, e)},
                                      static_cast<std::size_t>(k));
    out_matrix(o.scores, scores);
    std::memcpy(idx, o.topk_indices.data(), sizeof(int64_t) * o.topk_indices.size());
    out_matrix(o.topk_scores, vals);
  });
}

int ref_gate_backward(const double* x, const double* wg, const double* scores,
                      const int64_t* idx, const double* vals, const double* d_topk, int64_t n,
                      int64_t d, int64_t e, int64_t k, double* d_wg, double* d_x) {
  return guarded([&] {
    GateOutput o;
    o.scores = to_matrix(scores, n, e);
    o.topk_indices = to_index(idx, n, k);
    o.topk_scores = to_matrix(vals, n, k);
    const GateGrads g = gate_backward(to_matrix(x, n, d), GateParams{to_matrix(wg, d, e)}, o,
                                      to_matrix(d_topk, n, k));
    out_matrix(g.d_wg, d_wg);
    out_matrix(g.d_x, d_x);
  });
}

int ref_build_plan(const int64_t* idx, int64_t n, int64_t k, int64_t e, int64_t* counts,
                   int64_t* offsets, int64_t* src_row, int64_t* slot, int64_t* inverse_pos) {
  return guarded([&] {
    const DispatchPlan p = plan_from(idx, n, k, e);
    out_vec(p.counts, counts);
    out_vec(p.offsets, offsets);
    out_vec(p.expanded_src_row, src_row);
    out_vec(p.expanded_slot, slot);
    if (p.inverse_pos.size())
      std::memcpy(inverse_pos, p.inverse_pos.data(), sizeof(int64_t) * p.inverse_pos.size());
  });
}

int ref_scatter(const double* x, const int64_t* idx, int64_t n, int64_t k, int64_t e, int64_t d,
                double* xs) {
  return guarded([&] { out_matrix(scatter(to_matrix(x, n, d), plan_from(idx, n, k, e)), xs); });
}

int ref_gather_combine(const double* ys, const int64_t* idx, const double* w, int64_t n,
                       int64_t k, int64_t e, int64_t d, double* y) {
  return guarded([&] {
    out_matrix(gather_combine(to_matrix(ys, n * k, d), plan_from(idx, n, k, e), to_matrix(w, n, k)), y);
  });
}

int ref_scatter_backward(const double* d_xs, const int64_t* idx, int64_t n, int64_t k, int64_t e,
                         int64_t d, double* dx) {
  return guarded([&] {
    out_matrix(scatter_backward(to_matrix(d_xs, n * k, d), plan_from(idx, n, k, e)), dx);
  });
}

int ref_gather_combine_backward(const double* dy, const double* ys, const int64_t* idx,
                                const double* w, int64_t n, int64_t k, int64_t e, int64_t d,
                                double* d_ys, double* d_w) {
  return guarded([&] {
    const GatherCombineGrads g = gather_combine_backward(
        to_matrix(dy, n, d), to_matrix(ys, n * k, d), plan_from(idx, n, k, e), to_matrix(w, n, k));
    out_matrix(g.d_ys, d_ys);
    out_matrix(g.d_topk_scores, d_w);
  });
}

// multi_expert_forward + multi_expert_backward over `e` experts with the given
// per-expert row counts (blocks contiguous in xs).  d_ys may be NULL.
int ref_multi_expert(const double* xs, const int64_t* counts, int64_t e, int64_t d, int64_t h,
                     const double* w1, const double* b1, const double* w2, const double* b2,
                     const double* d_ys, double* ys, double* d_xs, double* dw1, double* db1,
                     double* dw2, double* db2) {
  return guarded([&] {
    int64_t rows = 0;
    for (int64_t g = 0; g < e; ++g) rows += counts[g];
    std::vector<ExpertParams> ex;
    for (int64_t g = 0; g < e; ++g)
      ex.push_back(expert_from(w1 + g * d * h, b1 + g * h, w2 + g * h * d, b2 + g * d, d, h));
    const std::vector<int64_t> cnt(counts, counts + e);
    MultiExpertResult r = multi_expert_forward(to_matrix(xs, rows, d), cnt, ex);
    out_matrix(r.ys, ys);
    if (d_ys) {
      const MultiExpertGrads g = multi_expert_backward(to_matrix(d_ys, rows, d), r.caches, ex);
      out_matrix(g.d_xs, d_xs);
      for (int64_t i = 0; i < e; ++i) {
        out_matrix(g.experts[i].d_w1, dw1 + i * d * h);
        out_matrix(g.experts[i].d_b1, db1 + i * h);
        out_matrix(g.experts[i].d_w2, dw2 + i * h * d);
        out_matrix(g.experts[i].d_b2, db2 + i * d);
      }
    }
  });
}

// Single-worker MoE layer forward(+backward when dy != NULL) through the
// reference's own forward()/backward() (moe_layer.cpp:67-142).
int ref_moe_forward_backward(const double* x, const double* dy, int64_t n, int64_t d, int64_t h,
                             int64_t e, int64_t k, const double* wg, const double* w1,
                             const double* b1, const double* w2, const double* b2, double* y,
                             int64_t* idx_out, double* dx, double* dwg, double* dw1, double* db1,
                             double* dw2, double* db2) {
  return guarded([&] {
    const MoELayerState st = state_from(n, d, h, e, k, 1, 0, wg, w1, b1, w2, b2);
    MoEForwardCache cache;
    const Matrix xm = to_matrix(x, n, d);
    out_matrix(forward(xm, st, nullptr, &cache), y);
    if (idx_out)
      std::memcpy(idx_out, cache.gate_out.topk_indices.data(),
                  sizeof(int64_t) * cache.gate_out.topk_indices.size());
    if (dy) {
      auto [d_x, grads] = backward(to_matrix(dy, n, d), cache, st, nullptr);
      out_matrix(d_x, dx);
      out_matrix(grads.d_wg, dwg);
      for (int64_t g = 0; g < e; ++g) {
        out_matrix(grads.experts[g].d_w1, dw1 + g * d * h);
        out_matrix(grads.experts[g].d_b1, db1 + g * h);
        out_matrix(grads.experts[g].d_w2, dw2 + g * h * d);
        out_matrix(grads.experts[g].d_b2, db2 + g * d);
      }
    }
  });
}

// naive_forward (moe_layer.cpp:47-65): Alg. 1 per-sample loop.
int ref_naive_forward(const double* x, int64_t n, int64_t d, int64_t h, int64_t e, int64_t k,
                      const double* wg, const double* w1, const double* b1, const double* w2,
                      const double* b2, double* y) {
  return guarded([&] {
    const MoELayerState st = state_from(n, d, h, e, k, 1, 0, wg, w1, b1, w2, b2);
    out_matrix(naive_forward(to_matrix(x, n, d), st), y);
  });
}

// Expert-parallel forward+backward over an InProcWorld of `world` ranks (one
// thread per rank, the reference's run_world_inproc pattern).  Rank r owns
// rows [r*n, (r+1)*n) of x/dy and experts [r*e_local, (r+1)*e_local).
// Outputs are rank-major concatenations; send/recv count matrices
// [world][world*e_local] are returned for the exchange-plan parity checks.
int ref_moe_distributed(const double* x, const double* dy, int64_t world, int64_t n, int64_t d,
                        int64_t h, int64_t e_local, int64_t k, const double* wg, const double* w1,
                        const double* b1, const double* w2, const double* b2, double* y,
                        double* dx, double* dwg, double* dw1, double* db1, double* dw2,
                        double* db2, int64_t* send_counts, int64_t* recv_counts) {
  return guarded([&] {
    InProcWorld w(static_cast<int>(world));
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(world));
    std::vector<std::thread> threads;
    const int64_t et = e_local * world;
    for (int64_t r = 0; r < world; ++r) {
      threads.emplace_back([&, r] {
        try {
          auto t = w.transport(static_cast<int>(r));
          const MoELayerState st =
              state_from(n, d, h, e_local, k, world, static_cast<int>(r), wg, w1, b1, w2, b2);
          MoEForwardCache cache;
          out_matrix(forward(to_matrix(x + r * n * d, n, d), st, t.get(), &cache), y + r * n * d);
          if (send_counts) out_vec(cache.exchange->send_counts, send_counts + r * et);
          if (recv_counts) out_vec(cache.exchange->recv_counts, recv_counts + r * et);
          if (dy) {
            auto [d_x, grads] = backward(to_matrix(dy + r * n * d, n, d), cache, st, t.get());
            out_matrix(d_x, dx + r * n * d);
            out_matrix(grads.d_wg, dwg + r * d * et);
            for (int64_t s = 0; s < e_local; ++s) {
              const int64_t g = r * e_local + s;
              out_matrix(grads.experts[s].d_w1, dw1 + g * d * h);
              out_matrix(grads.experts[s].d_b1, db1 + g * h);
              out_matrix(grads.experts[s].d_w2, dw2 + g * h * d);
              out_matrix(grads.experts[s].d_b2, db2 + g * d);
            }
          }
        } catch (...) {
          errs[static_cast<std::size_t>(r)] = std::current_exception();
        }
      });
    }
    for (auto& th : threads) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

// train_step trajectories (moe_layer.cpp:144-205): `steps` SGD steps of the
// reference's init_state(seed) layer on rank slices of x/target ([world*n, d]),
// world ranks over its InProcWorld (world 1: no transport).  losses[steps] from
// rank 0; final gate (rank 0) and every expert in global order.
int ref_train_steps(int64_t world, int64_t n, int64_t d, int64_t h, int64_t e_local, int64_t k, uint64_t seed,
                    int64_t steps, double lr, const double* x, const double* target, double* losses, double* wg,
                    double* w1, double* b1, double* w2, double* b2) {
  return guarded([&] {
    MoEConfig cfg;
    cfg.n_b = static_cast<std::size_t>(n);
    cfg.d_m = static_cast<std::size_t>(d);
    cfg.d_h = static_cast<std::size_t>(h);
    cfg.k = static_cast<std::size_t>(k);
    cfg.n_e_local = static_cast<std::size_t>(e_local);
    cfg.world_size = static_cast<std::size_t>(world);
    cfg.seed = seed;
    auto run = [&](int r, Transport* t) {
      MoELayerState st = init_state(cfg, r);
      const Matrix xr = to_matrix(x + r * n * d, n, d), tr = to_matrix(target + r * n * d, n, d);
      for (int64_t s = 0; s < steps; ++s) {
        const double l = train_step(xr, tr, st, lr, t);
        if (r == 0) losses[s] = l;
      }
      if (r == 0) out_matrix(st.gate.w_g, wg);
      for (int64_t sl = 0; sl < e_local; ++sl) {
        const int64_t g = r * e_local + sl;
        out_matrix(st.experts[sl].w1, w1 + g * d * h);
        out_matrix(st.experts[sl].b1, b1 + g * h);
        out_matrix(st.experts[sl].w2, w2 + g * h * d);
        out_matrix(st.experts[sl].b2, b2 + g * d);
      }
    };
    if (world == 1) {
      run(0, nullptr);
      return;
    }
    InProcWorld w(static_cast<int>(world));
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(world));
    std::vector<std::thread> threads;
    for (int64_t r = 0; r < world; ++r)
      threads.emplace_back([&, r] {
        try {
          auto t = w.transport(static_cast<int>(r));
          run(static_cast<int>(r), t.get());
        } catch (...) {
          errs[static_cast<std::size_t>(r)] = std::current_exception();
        }
      });
    for (auto& th : threads) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

// CPU-baseline handle: the reference's own init_state + forward/backward at a
// given configuration, inputs from the bench generators (x stream 102, dy
// stream 103; fmoe_bench.cpp:128-134,226-227).  Threads: FMOE_THREADS.
struct RefBench {
  MoELayerState st;
  Matrix x, dy;
};

void* ref_bench_create(uint64_t seed, int64_t n, int64_t d, int64_t h, int64_t e, int64_t k) {
  try {
    MoEConfig cfg;
    cfg.n_b = static_cast<std::size_t>(n);
    cfg.d_m = static_cast<std::size_t>(d);
    cfg.d_h = static_cast<std::size_t>(h);
    cfg.k = static_cast<std::size_t>(k);
    cfg.n_e_local = static_cast<std::size_t>(e);
    cfg.world_size = 1;
    cfg.seed = seed;
    auto* b = new RefBench;
    b->st = init_state(cfg, 0);
    b->x = Matrix(static_cast<std::size_t>(n), static_cast<std::size_t>(d));
    b->dy = Matrix(static_cast<std::size_t>(n), static_cast<std::size_t>(d));
    UniformRng(stream_seed(seed, 102)).fill(b->x, -1.0, 1.0);
    UniformRng(stream_seed(seed, 103)).fill(b->dy, -1.0, 1.0);
    return b;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return nullptr;
  }
}

int ref_bench_step(void* handle) {
  return guarded([&] {
    auto* b = static_cast<RefBench*>(handle);
    MoEForwardCache cache;
    const Matrix y = forward(b->x, b->st, nullptr, &cache);
    auto res = backward(b->dy, cache, b->st, nullptr);
    (void)y;
    (void)res;
  });
}

void ref_bench_destroy(void* handle) { delete static_cast<RefBench*>(handle); }

// make_toy_task (moe_layer.cpp): inputs / targets [n_b * world, d_m].
int ref_toy_task(int64_t n, int64_t d, int64_t h, int64_t k, int64_t el, int64_t world, uint64_t seed, double* x,
                 double* t) {
  return guarded([&] {
    MoEConfig cfg;
    cfg.n_b = static_cast<std::size_t>(n);
    cfg.d_m = static_cast<std::size_t>(d);
    cfg.d_h = static_cast<std::size_t>(h);
    cfg.k = static_cast<std::size_t>(k);
    cfg.n_e_local = static_cast<std::size_t>(el);
    cfg.world_size = static_cast<std::size_t>(world);
    cfg.seed = seed;
    const ToyTask task = make_toy_task(cfg);
    out_matrix(task.inputs, x);
    out_matrix(task.targets, t);
  });
}

// save_checkpoint (checkpoint.cpp:63-92) of the given weights: wg [d, e],
// w1 [e, d, h], b1 [e, h], w2 [e, h, d], b2 [e, d]; meta = n_b, k,
// n_e_local, world_size, seed.
int ref_save_checkpoint(const char* path, int64_t d, int64_t h, int64_t e, const int64_t* meta,
                        const double* wg, const double* w1, const double* b1, const double* w2,
                        const double* b2) {
  return guarded([&] {
    MoEConfig cfg;
    cfg.n_b = static_cast<std::size_t>(meta[0]);
    cfg.d_m = static_cast<std::size_t>(d);
    cfg.d_h = static_cast<std::size_t>(h);
    cfg.k = static_cast<std::size_t>(meta[1]);
    cfg.n_e_local = static_cast<std::size_t>(meta[2]);
    cfg.world_size = static_cast<std::size_t>(meta[3]);
    cfg.seed = static_cast<uint64_t>(meta[4]);
    std::vector<ExpertParams> ex;
    for (int64_t g = 0; g < e; ++g)
      ex.push_back(ExpertParams{to_matrix(w1 + g * d * h, d, h), to_matrix(b1 + g * h, 1, h),
                                to_matrix(w2 + g * h * d, h, d), to_matrix(b2 + g * d, 1, d), ParamTag::NoSync});
    save_checkpoint(path, cfg, GateParams{to_matrix(wg, d, e), ParamTag::World}, ex);
  });
}

// load_checkpoint (checkpoint.cpp:94-122): header (n_b, d_m, d_h, k,
// n_e_local, world_size, seed) and the weights (shapes as above).
int ref_load_checkpoint(const char* path, int64_t* header, double* wg, double* w1, double* b1, double* w2,
                        double* b2) {
  return guarded([&] {
    const Checkpoint c = load_checkpoint(path);
    const MoEConfig& k = c.config;
    const int64_t hv[7] = {(int64_t)k.n_b, (int64_t)k.d_m, (int64_t)k.d_h, (int64_t)k.k,
                           (int64_t)k.n_e_local, (int64_t)k.world_size, (int64_t)k.seed};
    std::memcpy(header, hv, sizeof(hv));
    if (!wg) return;
    const std::size_t d = k.d_m, h = k.d_h;
    out_matrix(c.gate.w_g, wg);
    for (std::size_t g = 0; g < c.experts.size(); ++g) {
      out_matrix(c.experts[g].w1, w1 + g * d * h);
      out_matrix(c.experts[g].b1, b1 + g * h);
      out_matrix(c.experts[g].w2, w2 + g * h * d);
      out_matrix(c.experts[g].b2, b2 + g * d);
    }
  });
}

// Injected-routing CPU baseline: the reference's dispatch +
// expert pool with a given IndexMatrix and scores instead of its gate --
// build_plan -> scatter -> multi_expert_forward -> gather_combine, then
// gather_combine_backward -> multi_expert_backward -> scatter_backward
// (dispatch.cpp:10-126, expert.cpp:85-125).
struct RefRoutedBench {
  MoELayerState st;
  Matrix x, dy, scores;
  IndexMatrix idx;
};

void* ref_bench_routed_create(uint64_t seed, int64_t n, int64_t d, int64_t h, int64_t e, int64_t k,
                              const int64_t* idx, const double* scores) {
  try {
    MoEConfig cfg;
    cfg.n_b = static_cast<std::size_t>(n);
    cfg.d_m = static_cast<std::size_t>(d);
    cfg.d_h = static_cast<std::size_t>(h);
    cfg.k = static_cast<std::size_t>(k);
    cfg.n_e_local = static_cast<std::size_t>(e);
    cfg.world_size = 1;
    cfg.seed = seed;
    auto* b = new RefRoutedBench;
    b->st = init_state(cfg, 0);
    b->x = Matrix(static_cast<std::size_t>(n), static_cast<std::size_t>(d));
    b->dy = Matrix(static_cast<std::size_t>(n), static_cast<std::size_t>(d));
    UniformRng(stream_seed(seed, 102)).fill(b->x, -1.0, 1.0);
    UniformRng(stream_seed(seed, 103)).fill(b->dy, -1.0, 1.0);
    b->idx = IndexMatrix(static_cast<std::size_t>(n), static_cast<std::size_t>(k));
    b->scores = Matrix(static_cast<std::size_t>(n), static_cast<std::size_t>(k));
    for (int64_t i = 0; i < n * k; ++i) {
      b->idx.data()[i] = idx[i];
      b->scores.data()[i] = scores[i];
    }
    return b;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return nullptr;
  }
}

int ref_bench_routed_step(void* handle) {
  return guarded([&] {
    auto* b = static_cast<RefRoutedBench*>(handle);
    const DispatchPlan plan = build_plan(b->idx, b->st.experts.size());
    const Matrix xs = scatter(b->x, plan);
    MultiExpertResult fwd = multi_expert_forward(xs, plan.counts, b->st.experts);
    const Matrix y = gather_combine(fwd.ys, plan, b->scores);
    GatherCombineGrads g = gather_combine_backward(b->dy, fwd.ys, plan, b->scores);
    MultiExpertGrads eg = multi_expert_backward(g.d_ys, fwd.caches, b->st.experts);
    const Matrix dx = scatter_backward(eg.d_xs, plan);
    (void)y;
    (void)dx;
  });
}

void ref_bench_routed_destroy(void* handle) { delete static_cast<RefRoutedBench*>(handle); }

// exchange_counts over an InProcWorld: local_counts [world][E_total] in,
// recv_counts [world][world*e_local] out (collectives.cpp:69-109).
int ref_exchange_counts(const int64_t* local_counts, int64_t world, int64_t total,
                        int64_t* recv_counts) {
  return guarded([&] {
    InProcWorld w(static_cast<int>(world));
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(world));
    std::vector<std::thread> threads;
    for (int64_t r = 0; r < world; ++r)
      threads.emplace_back([&, r] {
        try {
          auto t = w.transport(static_cast<int>(r));
          const ExchangePlan p = exchange_counts(
              std::span<const int64_t>(local_counts + r * total, static_cast<std::size_t>(total)), *t);
          out_vec(p.recv_counts, recv_counts + r * total);
        } catch (...) {
          errs[static_cast<std::size_t>(r)] = std::current_exception();
        }
      });
    for (auto& th : threads) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

}  // extern "C"
