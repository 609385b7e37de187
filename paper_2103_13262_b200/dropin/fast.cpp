// fast.cpp -- the device-resident route of the drop-in's MoE layer
// (reference API: proj/include/fmoe/moe_layer.hpp:57-70, moe_layer.cpp:67-205).
//
// forward / backward / train_step of a single-worker state run as ONE device
// layer (fmoe_layer_*, FMOE_F64 by default) instead of composing the
// operators with a host round trip each:
//   * the parameters stay on the GPU and are re-sent only when a parameter
//     Matrix changed (content identity, fmoe/matrix.hpp);
//   * every result -- y, the forward cache (scores, top-k scores, expert
//     inputs / pre-activations / hidden / outputs), d_x, the gradients, the
//     parameters after train_step -- is a device-backed Matrix whose values
//     reach the host only if the caller reads them;
//   * backward reuses the activations the layer still holds when it is handed
//     the cache of the layer's latest forward, unedited (CacheToken);
//     anything else takes the operator composition (layer.cpp).
// FMOE_F64 runs the same kernels in the same accumulation order as the
// composition, so the numbers are bit-identical to it and to the reference.
// FMOE_DROPIN_DTYPE=f32 (bf16x6 tensor-core products) or bf16 (bf16 storage,
// fp32 accumulation) runs the layer in that precision instead -- within
// SURVEY 8(c)'s fp32 / bf16 tolerances, not bit-identical; in bf16 the cache's
// preact holds relu(preact) (the bf16 fc1 epilogue applies the relu).
// FMOE_DROPIN_PATH=ops disables this route.
#include <cstdlib>
#include <cstring>
#include <optional>
#include <string>

#include "dropin.hpp"
#include "fmoe/errors.hpp"
#include "fmoe/moe_layer.hpp"

namespace fmoe::dropin {

namespace {

bool fast_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FMOE_DROPIN_PATH");
    return !(e && std::string(e) == "ops");
  }();
  return on;
}

fmoe_dtype fast_dtype() {
  static const fmoe_dtype t = [] {
    const char* e = std::getenv("FMOE_DROPIN_DTYPE");
    const std::string v = e ? e : "";
    if (v.empty() || v == "f64") return FMOE_F64;
    if (v == "f32") return FMOE_F32;
    if (v == "bf16") return FMOE_BF16;
    throw ShapeError("FMOE_DROPIN_DTYPE must be f64, f32 or bf16");
  }();
  return t;
}

std::size_t esize(fmoe_dtype t) { return t == FMOE_F64 ? 8 : t == FMOE_F32 ? 4 : 2; }
fmoe_dtype score_t(fmoe_dtype t) { return t == FMOE_F64 ? FMOE_F64 : FMOE_F32; }
fmoe_dtype bias_t(fmoe_dtype t) { return t == FMOE_BF16 ? FMOE_F32 : t; }

struct FastLayer {
  fmoe_layer* layer = nullptr;
  fmoe_layer_config cfg{};
  std::vector<std::uint64_t> wkey;  // content identity of the parameters on the device
  std::uint64_t seq = 0;            // forwards run (cache tokens)
  FastLayer() = default;
  FastLayer(const FastLayer&) = delete;
  ~FastLayer() {
    if (layer) fmoe_layer_destroy(layer);
  }
};

// What a fast forward left in its cache: which forward of which layer, the
// device values it handed out and copies of the host fields, so backward can
// tell that the layer still holds this forward's activations and that the
// cache was not edited.  Keeps the device input alive (the layer's backward
// reads x for the gate gradient).
struct CacheToken {
  const FastLayer* owner = nullptr;
  std::uint64_t seq = 0;
  std::shared_ptr<detail::DeviceStore> x_layer;  // x in the layer dtype (non-f64 layers)
  std::vector<const detail::DeviceStore*> stores;
  IndexMatrix topk;
  std::vector<std::int64_t> counts, offsets, src, slot;
  IndexMatrix inverse_pos;
};

FastLayer& fast_layer(const MoEConfig& c, std::size_t n_b) {
  local();  // the thread's device context first: destroyed after the layer
  thread_local FastLayer fl;
  const fmoe_dtype t = fast_dtype();
  const bool same = fl.layer && (std::size_t)fl.cfg.n_b == n_b && (std::size_t)fl.cfg.d_m == c.d_m &&
                    (std::size_t)fl.cfg.d_h == c.d_h && (std::size_t)fl.cfg.k == c.k &&
                    (std::size_t)fl.cfg.n_e_local == c.n_e_local && fl.cfg.seed == c.seed && fl.cfg.dtype == t;
  if (!same) {
    if (fl.layer) fmoe_layer_destroy(fl.layer);
    fl.layer = nullptr;
    fl.wkey.clear();
    fl.cfg = fmoe_layer_config{(int64_t)n_b, (int64_t)c.d_m, (int64_t)c.d_h, (int64_t)c.k, (int64_t)c.n_e_local,
                               1, 0, c.seed, t};
    check(fmoe_layer_create(local().ctx, &fl.cfg, &fl.layer));
    if (t != FMOE_BF16) check(fmoe_layer_keep_preact(fl.layer, 1));
  }
  return fl;
}

std::vector<std::uint64_t> param_key(const MoELayerState& st) {
  std::vector<std::uint64_t> k;
  k.reserve(3 + 12 * st.experts.size());
  auto add = [&](const Matrix& m) {
    k.push_back(m.content_id());
    k.push_back(m.content_version());
    k.push_back(reinterpret_cast<std::uintptr_t>(m.device_store().get()));
  };
  add(st.gate.w_g);
  for (const auto& e : st.experts)
    for (const Matrix* m : {&e.w1, &e.b1, &e.w2, &e.b2}) add(*m);
  return k;
}

// m (f64, host or device) -> n elements of dtype t at dst, on the device.
void put(const Matrix& m, void* dst, fmoe_dtype t, const Device& d) {
  const std::size_t n = m.size();
  if (!n) return;
  if (t == FMOE_F64) {
    if (const auto& st = m.device_store())
      cuda(cudaMemcpyAsync(dst, st->f64(m.device_offset()), n * 8, cudaMemcpyDeviceToDevice, d.stream), "D2D");
    else
      cuda(cudaMemcpyAsync(dst, m.data(), n * 8, cudaMemcpyHostToDevice, d.stream), "H2D");
    return;
  }
  Buf src = upload(m, d.stream);  // f64 view or upload
  check(fmoe_cast(d.ctx, FMOE_F64, src.get(), t, dst, (int64_t)n));
  check(fmoe_ctx_check(d.ctx));  // `src` may be a temporary upload
}

// The state's parameters onto the layer, when they changed since the last call.
void sync_params(FastLayer& fl, const MoELayerState& st) {
  std::vector<std::uint64_t> key = param_key(st);
  if (key == fl.wkey) return;
  auto& d = local();
  const fmoe_dtype t = fl.cfg.dtype;
  const std::size_t dm = st.config.d_m, dh = st.config.d_h, E = st.experts.size();
  if (st.gate.w_g.rows() != dm || st.gate.w_g.cols() != st.config.total_experts())
    throw ShapeError("forward: gate weights shape mismatch");
  void* wg = nullptr;
  fmoe_expert_params p{};
  check(fmoe_layer_params(fl.layer, &wg, &p));
  put(st.gate.w_g, wg, t, d);
  const std::size_t es = esize(t), bs = esize(bias_t(t));
  for (std::size_t e = 0; e < E; ++e) {
    const ExpertParams& x = st.experts[e];
    if (x.w1.rows() != dm || x.w1.cols() != dh || x.b1.size() != dh || x.w2.rows() != dh || x.w2.cols() != dm ||
        x.b2.size() != dm)
      throw ShapeError("expert_forward: parameter shapes do not match the config");
    put(x.w1, static_cast<char*>(const_cast<void*>(p.w1)) + e * dm * dh * es, t, d);
    put(x.b1, static_cast<char*>(const_cast<void*>(p.b1)) + e * dh * bs, bias_t(t), d);
    put(x.w2, static_cast<char*>(const_cast<void*>(p.w2)) + e * dh * dm * es, t, d);
    put(x.b2, static_cast<char*>(const_cast<void*>(p.b2)) + e * dm * bs, bias_t(t), d);
  }
  if (t == FMOE_BF16) check(fmoe_layer_sync_masters(fl.layer));
  check(fmoe_ctx_check(d.ctx));
  fl.wkey = std::move(key);
}

// n elements of dtype t at src -> a new f64 device store.
std::shared_ptr<detail::DeviceStore> to_f64(const void* src, fmoe_dtype t, std::size_t n, const Device& d) {
  auto st = device_store(n * 8, d);
  if (n) {
    if (t == FMOE_F64)
      cuda(cudaMemcpyAsync(st->ptr, src, n * 8, cudaMemcpyDeviceToDevice, d.stream), "D2D");
    else
      check(fmoe_cast(d.ctx, t, src, FMOE_F64, st->ptr, (int64_t)n));
  }
  return st;
}

// Rows of the layer's (possibly 128/256-aligned) expert blocks -> the
// reference's compact layout (expert e at the exclusive prefix of counts),
// as f64.  `off_a` / `off_c`: aligned / compact block starts.
std::shared_ptr<detail::DeviceStore> compact_rows(const void* src, fmoe_dtype t, std::size_t cols,
                                                  const std::vector<std::int64_t>& counts,
                                                  const std::vector<std::int64_t>& off_a,
                                                  const std::vector<std::int64_t>& off_c, std::size_t rows,
                                                  const Device& d) {
  auto st = device_store(rows * cols * 8, d);
  const std::size_t es = esize(t);
  for (std::size_t e = 0; e < counts.size(); ++e) {
    const std::size_t n = (std::size_t)counts[e] * cols;
    if (!n) continue;
    const char* s = static_cast<const char*>(src) + (std::size_t)off_a[e] * cols * es;
    double* o = st->f64((std::size_t)off_c[e] * cols);
    if (t == FMOE_F64)
      cuda(cudaMemcpyAsync(o, s, n * 8, cudaMemcpyDeviceToDevice, d.stream), "D2D");
    else
      check(fmoe_cast(d.ctx, t, s, FMOE_F64, o, (int64_t)n));
  }
  return st;
}

std::vector<std::int64_t> dl_i32(const int32_t* p, std::size_t n, const Device& d) {
  std::vector<std::int32_t> h(n);
  if (n) cuda(cudaMemcpyAsync(h.data(), p, n * 4, cudaMemcpyDeviceToHost, d.stream), "D2H");
  check(fmoe_ctx_check(d.ctx));
  return std::vector<std::int64_t>(h.begin(), h.end());
}

bool applicable(const MoELayerState& st, std::size_t n_b) {
  const MoEConfig& c = st.config;
  return fast_enabled() && n_b > 0 && c.world_size == 1 && st.experts.size() == c.total_experts() &&
         (fast_dtype() == FMOE_F64 || (c.d_m % 64 == 0 && c.d_h % 64 == 0 && c.total_experts() % 8 == 0 &&
                                       (fast_dtype() != FMOE_BF16 || c.k <= 8)));
}

}  // namespace

std::optional<Matrix> fast_forward(const Matrix& x, const MoELayerState& state, MoEForwardCache* cache) {
  if (!applicable(state, x.rows())) return std::nullopt;
  const MoEConfig& c = state.config;
  FastLayer& fl = fast_layer(c, x.rows());
  auto& d = local();
  sync_params(fl, state);
  const fmoe_dtype t = fl.cfg.dtype;
  const std::size_t n = x.rows(), dm = c.d_m, dh = c.d_h, k = c.k, E = c.total_experts(), nk = n * k;
  // x on the device as f64 (the cache's input) and in the layer dtype (the
  // layer keeps reading it until its backward)
  std::shared_ptr<detail::DeviceStore> x64;
  if (const auto& st = x.device_store(); st && x.device_offset() == 0 && st->bytes == n * dm * 8) {
    x64 = std::const_pointer_cast<detail::DeviceStore>(st);
  } else {
    x64 = device_store(n * dm * 8, d);
    if (const auto& s2 = x.device_store())
      cuda(cudaMemcpyAsync(x64->ptr, s2->f64(x.device_offset()), n * dm * 8, cudaMemcpyDeviceToDevice, d.stream),
           "D2D");
    else
      cuda(cudaMemcpyAsync(x64->ptr, x.data(), n * dm * 8, cudaMemcpyHostToDevice, d.stream), "H2D");
  }
  std::shared_ptr<detail::DeviceStore> xl;
  const void* x_layer = x64->ptr;
  if (t != FMOE_F64) {
    xl = device_store(n * dm * esize(t), d);
    check(fmoe_cast(d.ctx, FMOE_F64, x64->ptr, t, xl->ptr, (int64_t)(n * dm)));
    x_layer = xl->ptr;
  }
  Buf y_l(n * dm * esize(t), d.stream);
  check(fmoe_layer_fwd(fl.layer, x_layer, y_l.get()));
  ++fl.seq;
  Matrix y = device_matrix(n, dm, to_f64(y_l.get(), t, n * dm, d));
  if (cache) {
    const int32_t* idx = nullptr;
    const void *vals = nullptr, *scores = nullptr;
    fmoe_plan plan{};
    check(fmoe_layer_routing(fl.layer, &idx, &vals, &scores, &plan));
    const void *xs = nullptr, *hid = nullptr, *pre = nullptr, *ys = nullptr;
    check(fmoe_layer_activations(fl.layer, &xs, &hid, &pre, &ys));
    auto tok = std::make_shared<CacheToken>();
    tok->owner = &fl;
    tok->seq = fl.seq;
    tok->x_layer = xl;
    cache->input = device_matrix(n, dm, x64);
    cache->gate_out.scores = device_matrix(n, E, to_f64(scores, score_t(t), n * E, d));
    cache->gate_out.topk_scores = device_matrix(n, k, to_f64(vals, score_t(t), nk, d));
    const std::vector<std::int64_t> topk = dl_i32(idx, nk, d);
    cache->gate_out.topk_indices = IndexMatrix(n, k);
    std::memcpy(cache->gate_out.topk_indices.data(), topk.data(), nk * 8);
    // the plan in the reference's compact layout (dispatch.cpp:10-47)
    DispatchPlan& P = cache->plan;
    P.num_experts = E;
    P.k = k;
    P.n_b = n;
    P.counts = dl_i32(plan.counts, E, d);
    const std::vector<std::int64_t> off_a = dl_i32(plan.offsets, E, d);
    P.offsets.assign(E, 0);
    for (std::size_t e = 1; e < E; ++e) P.offsets[e] = P.offsets[e - 1] + P.counts[e - 1];
    const std::vector<std::int64_t> src_a = dl_i32(plan.src_row, (std::size_t)plan.capacity, d);
    const std::vector<std::int64_t> slot_a = dl_i32(plan.slot, (std::size_t)plan.capacity, d);
    const std::vector<std::int64_t> inv_a = dl_i32(plan.inverse_pos, nk, d);
    P.expanded_src_row.assign(nk, 0);
    P.expanded_slot.assign(nk, 0);
    for (std::size_t e = 0; e < E; ++e)
      for (std::int64_t r = 0; r < P.counts[e]; ++r) {
        P.expanded_src_row[(std::size_t)(P.offsets[e] + r)] = src_a[(std::size_t)(off_a[e] + r)];
        P.expanded_slot[(std::size_t)(P.offsets[e] + r)] = slot_a[(std::size_t)(off_a[e] + r)];
      }
    P.inverse_pos = IndexMatrix(n, k);
    for (std::size_t f = 0; f < nk; ++f) {
      const std::size_t e = (std::size_t)topk[f];
      P.inverse_pos.data()[f] = inv_a[f] - off_a[e] + P.offsets[e];
    }
    cache->exchange.reset();
    cache->local_block_counts = P.counts;
    // expert-side activations, compact, f64
    auto ys_c = compact_rows(ys, t, dm, P.counts, off_a, P.offsets, nk, d);
    auto xs_c = compact_rows(xs, t, dm, P.counts, off_a, P.offsets, nk, d);
    auto hid_c = compact_rows(hid, t, dh, P.counts, off_a, P.offsets, nk, d);
    auto pre_c = pre ? compact_rows(pre, t, dh, P.counts, off_a, P.offsets, nk, d) : hid_c;
    cache->expert_outputs = device_matrix(nk, dm, ys_c);
    cache->expert_caches.assign(E, ForwardCache{});
    for (std::size_t e = 0; e < E; ++e) {
      const std::size_t r0 = (std::size_t)P.offsets[e], rows = (std::size_t)P.counts[e];
      cache->expert_caches[e] = ForwardCache{device_matrix(rows, dm, xs_c, r0 * dm),
                                             device_matrix(rows, dh, pre_c, r0 * dh),
                                             device_matrix(rows, dh, hid_c, r0 * dh)};
    }
    tok->stores = {x64.get(), cache->gate_out.scores.device_store().get(),
                   cache->gate_out.topk_scores.device_store().get(), ys_c.get(), xs_c.get(), hid_c.get(),
                   pre_c.get()};
    tok->topk = cache->gate_out.topk_indices;
    tok->counts = P.counts;
    tok->offsets = P.offsets;
    tok->src = P.expanded_src_row;
    tok->slot = P.expanded_slot;
    tok->inverse_pos = P.inverse_pos;
    cache->device_token = tok;
  }
  check(fmoe_ctx_check(d.ctx));
  return y;
}

std::optional<std::pair<Matrix, MoEGrads>> fast_backward(const Matrix& d_y, const MoEForwardCache& cache,
                                                         const MoELayerState& state) {
  auto tok = std::static_pointer_cast<const CacheToken>(cache.device_token);
  if (!tok || cache.exchange.has_value() || !applicable(state, cache.input.rows())) return std::nullopt;
  const MoEConfig& c = state.config;
  FastLayer& fl = fast_layer(c, cache.input.rows());
  if (tok->owner != &fl || tok->seq != fl.seq) return std::nullopt;  // the layer moved on
  // the cache must be the one the forward produced, unedited
  const std::size_t E = c.total_experts();
  if (cache.expert_caches.size() != E) return std::nullopt;
  auto st_of = [](const Matrix& m) { return m.device_store().get(); };
  if (st_of(cache.input) != tok->stores[0] || st_of(cache.gate_out.scores) != tok->stores[1] ||
      st_of(cache.gate_out.topk_scores) != tok->stores[2] || st_of(cache.expert_outputs) != tok->stores[3])
    return std::nullopt;
  for (const ForwardCache& fc : cache.expert_caches)
    if (st_of(fc.input) != tok->stores[4] || st_of(fc.hidden) != tok->stores[5] || st_of(fc.preact) != tok->stores[6])
      return std::nullopt;
  const DispatchPlan& P = cache.plan;
  if (!(cache.gate_out.topk_indices == tok->topk) || P.counts != tok->counts || P.offsets != tok->offsets ||
      P.expanded_src_row != tok->src || P.expanded_slot != tok->slot || !(P.inverse_pos == tok->inverse_pos))
    return std::nullopt;
  const std::size_t n = cache.input.rows(), dm = c.d_m, dh = c.d_h;
  if (d_y.rows() != n || d_y.cols() != dm) return std::nullopt;  // the composition reports the mismatch
  auto& d = local();
  sync_params(fl, state);  // backward uses the state's parameters as they are now
  const fmoe_dtype t = fl.cfg.dtype;
  Buf dy64 = upload(d_y, d.stream);
  const void* dy_l = dy64.get();
  Buf dyc;
  if (t != FMOE_F64) {
    dyc = Buf(n * dm * esize(t), d.stream);
    check(fmoe_cast(d.ctx, FMOE_F64, dy64.get(), t, dyc.get(), (int64_t)(n * dm)));
    dy_l = dyc.get();
  }
  Buf dx_l(n * dm * esize(t), d.stream);
  check(fmoe_layer_bwd(fl.layer, dy_l, dx_l.get()));
  Matrix d_x = device_matrix(n, dm, to_f64(dx_l.get(), t, n * dm, d));
  void* dwg = nullptr;
  fmoe_expert_grads g{};
  check(fmoe_layer_grads(fl.layer, &dwg, &g));
  const fmoe_dtype gt = t == FMOE_F64 ? FMOE_F64 : FMOE_F32;
  MoEGrads grads;
  grads.d_wg = device_matrix(dm, E, to_f64(dwg, score_t(t), dm * E, d));
  auto w1 = to_f64(g.d_w1, gt, E * dm * dh, d), b1 = to_f64(g.d_b1, gt, E * dh, d);
  auto w2 = to_f64(g.d_w2, gt, E * dh * dm, d), b2 = to_f64(g.d_b2, gt, E * dm, d);
  grads.experts.resize(E);
  for (std::size_t e = 0; e < E; ++e)
    grads.experts[e] = ExpertGrads{device_matrix(dm, dh, w1, e * dm * dh), device_matrix(1, dh, b1, e * dh),
                                   device_matrix(dh, dm, w2, e * dh * dm), device_matrix(1, dm, b2, e * dm)};
  check(fmoe_ctx_check(d.ctx));
  return std::make_pair(std::move(d_x), std::move(grads));
}

std::optional<double> fast_train_step(const Matrix& x, const Matrix& target, MoELayerState& state, double lr) {
  if (!applicable(state, x.rows())) return std::nullopt;
  const MoEConfig& c = state.config;
  if (x.cols() != c.d_m) throw ShapeError("forward: input cols != d_m");
  if (!target.same_shape(x)) throw ShapeError("train_step: target shape != output shape");
  FastLayer& fl = fast_layer(c, x.rows());
  auto& d = local();
  sync_params(fl, state);
  const fmoe_dtype t = fl.cfg.dtype;
  const std::size_t n = x.rows(), dm = c.d_m, dh = c.d_h, E = c.total_experts();
  auto in = [&](const Matrix& m, Buf& keep64, Buf& keep) -> const void* {
    keep64 = upload(m, d.stream);
    if (t == FMOE_F64) return keep64.get();
    keep = Buf(n * dm * esize(t), d.stream);
    check(fmoe_cast(d.ctx, FMOE_F64, keep64.get(), t, keep.get(), (int64_t)(n * dm)));
    return keep.get();
  };
  Buf x64, xl, t64, tl;
  const void* xp = in(x, x64, xl);
  const void* tp = in(target, t64, tl);
  double loss = 0.0;
  check(fmoe_layer_train_step(fl.layer, xp, tp, lr, &loss));  // forward, MSE, backward, SGD (moe_layer.cpp:144-205)
  ++fl.seq;
  // the state takes the updated parameters: device snapshots, read back only on host access
  void* wg = nullptr;
  fmoe_expert_params p{};
  check(fmoe_layer_params(fl.layer, &wg, &p));
  state.gate.w_g = device_matrix(dm, E, to_f64(wg, t, dm * E, d));
  auto w1 = to_f64(p.w1, t, E * dm * dh, d), b1 = to_f64(p.b1, bias_t(t), E * dh, d);
  auto w2 = to_f64(p.w2, t, E * dh * dm, d), b2 = to_f64(p.b2, bias_t(t), E * dm, d);
  for (std::size_t e = 0; e < E; ++e) {
    ExpertParams& ep = state.experts[e];
    ep.w1 = device_matrix(dm, dh, w1, e * dm * dh);
    ep.b1 = device_matrix(1, dh, b1, e * dh);
    ep.w2 = device_matrix(dh, dm, w2, e * dh * dm);
    ep.b2 = device_matrix(1, dm, b2, e * dm);
  }
  check(fmoe_ctx_check(d.ctx));
  fl.wkey = param_key(state);  // already on the layer (bf16: its fp32 masters stay authoritative)
  return loss;
}

}  // namespace fmoe::dropin
