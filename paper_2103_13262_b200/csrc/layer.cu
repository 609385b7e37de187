// layer.cu -- the MoE layer (moe_layer.cpp:67-142) orchestrated on one
// stream: gate -> plan -> scatter -> experts -> gather_combine, and the
// backward pass in the reference's order.  All buffers are allocated once at
// creation (sized for n_b tokens, worst-case padded expert blocks), so a
// forward+backward step performs no allocation and no host synchronisation
// on a single GPU.
//
// FMOE_BF16 (product path), per step:
//   fwd: gate GEMM+softmax+top-k (tcgen05) | plan x3 | scatter | fc1 (tcgen05,
//        bias+relu) | fc2 (tcgen05, bias) | gather_combine
//   bwd: gather_combine_bwd + gate Jacobian | dgrad fc2 (relu mask, d_b1
//        partials) | dgrad fc1 | gate dx | scatter_backward  [d_x final] |
//        wgrad fc2 | db2 | wgrad fc1 | db1 | gate dWg (split-K) + reduce
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "init.h"
#include "layer.cuh"
#include "ops.cuh"

namespace fmoe_b200 {

namespace {
__global__ void count_out_of_range(const int32_t* __restrict__ idx, int64_t n, int32_t E, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && (unsigned)__ldg(idx + i) >= (unsigned)E) atomicAdd(bad, 1);
}

template <typename T>
T* dalloc(std::vector<void*>& owned, int64_t n) {
  void* p = nullptr;
  const size_t bytes = std::max<int64_t>(n, 1) * sizeof(T);
  CK(cudaMalloc(&p, bytes));
  owned.push_back(p);
  return reinterpret_cast<T*>(p);
}
void* dalloc_bytes(std::vector<void*>& owned, int64_t bytes) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<int64_t>(bytes, 256)));
  owned.push_back(p);
  return p;
}
}  // namespace

Layer::Layer(Ctx* c, const fmoe_layer_config& cf) : ctx(c), cfg(cf) {
  if (cfg.n_b < 0 || cfg.d_m < 1 || cfg.d_h < 1 || cfg.n_e_local < 1 || cfg.world_size < 1)
    shape_error("MoEConfig: all dimensions must be at least 1");
  E = cfg.n_e_local * cfg.world_size;
  if (cfg.k < 1 || cfg.k > E) shape_error("MoEConfig: k must lie in [1, total experts]");
  if (cfg.rank < 0 || cfg.rank >= cfg.world_size) shape_error("init_state: rank out of range");
  t = cfg.dtype;
  const bool bf = t == FMOE_BF16;
  if (bf) {
    if (cfg.d_m % 64 || cfg.d_h % 64)
      shape_error("bf16 layer needs d_m and d_h to be multiples of 64");
    if (E % 8) shape_error("bf16 layer needs a total expert count that is a multiple of 8");
    if (cfg.k > 8) shape_error("bf16 layer supports k <= 8");
  }
  es = dtype_size(t);
  ss = score_size(t);
  gs = bf ? 4 : es;  // gradient element size
  const int64_t n = cfg.n_b, d = cfg.d_m, h = cfg.d_h, k = cfg.k, el = cfg.n_e_local;
  // parameters
  wg = dalloc_bytes(owned, d * E * es);
  w1 = dalloc_bytes(owned, el * d * h * es);
  w2 = dalloc_bytes(owned, el * h * d * es);
  b1 = dalloc_bytes(owned, el * h * (bf ? 4 : es));
  b2 = dalloc_bytes(owned, el * d * (bf ? 4 : es));
  // gradients
  dwg = dalloc_bytes(owned, d * E * ss);
  dw1 = dalloc_bytes(owned, el * d * h * gs);
  dw2 = dalloc_bytes(owned, el * h * d * gs);
  db1 = dalloc_bytes(owned, el * h * gs);
  db2 = dalloc_bytes(owned, el * d * gs);
  // routing
  scores = dalloc_bytes(owned, n * E * ss);
  vals = dalloc_bytes(owned, n * k * ss);
  idx = dalloc<int32_t>(owned, n * k);
  plan.n_b = n;
  plan.k = k;
  plan.n_experts = E;
  const bool ep_mode = cfg.world_size > 1;  // EP: plan/xs/ys are the send layout
  // bf16 expert blocks: 256-row aligned (CTA-pair GEMM tiles) when experts
  // average >= 1024 rows, else 128 (single-CTA tiles waste less padding)
  // FMOE_F32 runs its expert GEMMs on the tensor cores (bf16x3, f32x.cu) over
  // the same aligned blocks; FMOE_F32_SIMT=1 keeps the reference layout and
  // the SIMT fp32 kernels
  const bool f32tc = t == FMOE_F32 && !ep_mode && f32_tc_enabled() && d % 64 == 0 && h % 64 == 0 && E % 8 == 0;
  plan.align = ((bf || f32tc) && !ep_mode) ? expert_block_align(n * k, E) : 1;
  plan.capacity = plan_capacity(n, k, E, plan.align);
  plan.counts = dalloc<int32_t>(owned, E);
  plan.offsets = dalloc<int32_t>(owned, E + 1);
  plan.src_row = dalloc<int32_t>(owned, plan.capacity);
  plan.slot = dalloc<int32_t>(owned, plan.capacity);
  plan.inverse_pos = dalloc<int32_t>(owned, n * k);
  plan.tile_expert = dalloc<int32_t>(owned, plan.capacity / 128 + 1);
  plan.n_tiles = dalloc<int32_t>(owned, 1);
  plan.scratch = dalloc_bytes(owned, plan_scratch_bytes(n, k, E));
  const int64_t cap = plan.capacity;
  // activations (forward cache)
  xs = dalloc_bytes(owned, cap * d * es);
  if (!ep_mode) hidden = dalloc_bytes(owned, cap * h * es);
  ys = dalloc_bytes(owned, cap * d * es);
  if (!bf || E > 256) logits = dalloc_bytes(owned, n * E * ss);
  // backward scratch
  d_ys = dalloc_bytes(owned, cap * d * es);
  if (!ep_mode) d_pre = dalloc_bytes(owned, cap * h * es);
  d_xs = dalloc_bytes(owned, cap * d * es);
  d_w = dalloc_bytes(owned, n * k * ss);
  dz = dalloc_bytes(owned, n * E * ss);
  dz_bf16 = dalloc<__nv_bfloat16>(owned, n * E);
  gdx = dalloc_bytes(owned, n * d * es);
  const int64_t S = gate_dwg_splits(n);
  part = dalloc<float>(owned, S * d * E + S + 64);
  if (!ep_mode) tpart = dalloc<float>(owned, experts_bwd_part_floats(plan, d, h));
  if (!ep_mode && bf) relu_bits = dalloc<uint32_t>(owned, cap * (h / 32));
  if (f32tc) f32_planes = dalloc<__nv_bfloat16>(owned, f32_planes_elems(n, d, h, E, el, cap));
  gather_xs = bf && !ep_mode && n > 0 && gather_enabled();
  if (cfg.world_size > 1) ep_alloc();
}

// The expanded input rows as a buffer (the operator-level cache view,
// fmoe_layer_activations): a gathering layer scatters them only when asked.
void Layer::ensure_xs() {
  if (xs_fresh || !fwd_done || cfg.world_size > 1) return;
  scatter(ctx, t, x_saved, cfg.d_m, plan, xs);
  xs_fresh = true;
}

Layer::~Layer() {
  ep_free(ep);
  for (auto* evs : {hio.x_done, hio.dy_done, hio.y_ready, hio.dx_ready, hio.compute_done, hio.out_done})
    for (int s = 0; s < 2; ++s)
      if (evs[s]) cudaEventDestroy(evs[s]);
  for (void* p : owned) cudaFree(p);
  if (h_stage) cudaFreeHost(h_stage);
}

void Layer::set_keep_preact(bool keep) {
  if (!keep) {
    preact_kept = false;
    return;
  }
  if (t == FMOE_BF16) shape_error("keep_preact: the bf16 layer applies relu in the fc1 epilogue");
  if (cfg.world_size > 1) shape_error("keep_preact: single-worker layers only");
  if (!preact) preact = dalloc_bytes(owned, plan.capacity * cfg.d_h * es);
  preact_kept = true;
}

F32Planes Layer::planes_view() const {
  if (!f32_planes) return F32Planes{};
  return f32_planes_at(f32_planes, cfg.n_b, cfg.d_m, cfg.d_h, E, cfg.n_e_local, plan.capacity);
}

fmoe_expert_params Layer::params() const { return fmoe_expert_params{w1, b1, w2, b2}; }
fmoe_expert_grads Layer::grads() const { return fmoe_expert_grads{dw1, db1, dw2, db2}; }

// init_state (moe_layer.cpp:28-45): reference generators, rounded once.
void Layer::init_weights() {
  const int64_t d = cfg.d_m, h = cfg.d_h, el = cfg.n_e_local;
  std::vector<double> g(d * E), a1(el * d * h), c1(el * h), a2(el * h * d), c2(el * d);
  init_gate_host(cfg.seed, d, E, g.data());
  init_experts_host(cfg.seed, cfg.rank * el, el, d, h, a1.data(), c1.data(), a2.data(), c2.data());
  auto upload = [&](const std::vector<double>& src, void* dst, fmoe_dtype as) {
    if (as == FMOE_F64) {
      CK(cudaMemcpy(dst, src.data(), src.size() * 8, cudaMemcpyHostToDevice));
    } else if (as == FMOE_F32) {
      std::vector<float> f(src.begin(), src.end());
      CK(cudaMemcpy(dst, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
    } else {
      std::vector<__nv_bfloat16> b(src.size());
      for (size_t i = 0; i < src.size(); ++i) b[i] = __float2bfloat16_rn((float)src[i]);
      CK(cudaMemcpy(dst, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
    }
  };
  const fmoe_dtype bias_t = t == FMOE_BF16 ? FMOE_F32 : t;
  upload(g, wg, t);
  upload(a1, w1, t);
  upload(c1, b1, bias_t);
  upload(a2, w2, t);
  upload(c2, b2, bias_t);
  masters_fresh = false;  // bf16 training re-widens its fp32 masters
}

void Layer::forward(const void* x, void* y) {
  const int64_t n = cfg.n_b, d = cfg.d_m, k = cfg.k;
  // moe_layer.cpp:70-75: validate the transport before any work is issued
  if (cfg.world_size > 1) ep_check();
  x_saved = x;
  fwd_done = false;
  routed = false;
  prof_slot = ctx_take_slot(ctx);
  ctx_mark(ctx, MARK_FWD_BEGIN);
  if (f32_planes)  // FMOE_F32 on the tensor cores: logits as a bf16x6 product (f32x.cu)
    gate_fwd_f32tc(ctx, (const float*)x, (const float*)wg, n, d, E, k, (float*)scores, idx, (float*)vals,
                   (float*)logits, planes_view());
  else
    gate_fwd(ctx, t, x, wg, n, d, E, k, scores, idx, vals, logits);  // gate.cpp:23-35
  ctx_mark(ctx, MARK_GATE);
  dispatch_and_experts(x, y);
}

// Injected routing (the reference feeds a sampled
// IndexMatrix straight into build_plan, dispatch.hpp:28): the gate is skipped,
// topk_idx [n_b, k] int32 / topk_scores [n_b, k] (score dtype) drive the same
// plan -> scatter -> experts -> gather_combine; backward then yields d_x from
// scatter_backward alone and d(topk_scores) (routing_grad), no gate gradients.
void Layer::forward_routed(const void* x, const int32_t* topk_idx, const void* topk_scores, void* y) {
  const int64_t n = cfg.n_b, k = cfg.k;
  if (cfg.world_size > 1) ep_check();
  x_saved = x;
  fwd_done = false;
  routed = true;
  // build_plan validates before any work (dispatch.cpp:21-23): injected
  // indices are checked here, synchronously, so a bad IndexMatrix throws
  // ShapeError from this call and no kernel ever sees it
  if (n * k > 0) {
    CK(cudaMemsetAsync(ctx->d_error, 0, sizeof(int), ctx->stream));
    count_out_of_range<<<(unsigned)ceil_div(n * k, 256), 256, 0, ctx->stream>>>(topk_idx, n * k, (int32_t)E,
                                                                                ctx->d_error);
    CK_LAUNCH(ctx);
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, ctx->d_error, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (bad) shape_error("build_plan: expert index out of range (" + std::to_string(bad) + " entries)");
  }
  prof_slot = ctx_take_slot(ctx);
  ctx_mark(ctx, MARK_FWD_BEGIN);
  CK(cudaMemcpyAsync(idx, topk_idx, (size_t)n * k * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(vals, topk_scores, (size_t)n * k * ss, cudaMemcpyDeviceToDevice, ctx->stream));
  ctx_mark(ctx, MARK_GATE);
  dispatch_and_experts(x, y);
}

void Layer::dispatch_and_experts(const void* x, void* y) {
  const int64_t d = cfg.d_m, h = cfg.d_h;
  if (cfg.world_size > 1) {
    ep_forward(x, y);
    fwd_done = true;
    return;
  }
  plan_build(ctx, idx, plan);                                     // dispatch.cpp:10-47
  ctx_mark(ctx, MARK_PLAN);
  // dispatch.cpp:49-59: a scatter pass, or (bf16, one GPU) folded into fc1's
  // A-load as a TMA gather of x's rows -- no xs write / re-read
  const RowGather gth{x, cfg.n_b, plan.src_row};
  if (!gather_xs) scatter(ctx, t, x, d, plan, xs);
  xs_fresh = !gather_xs;
  ctx_mark(ctx, MARK_SCATTER);
  const F32Planes pv = planes_view();
  experts_fwd(ctx, t, plan, d, h, params(), xs, hidden, ys, relu_bits, preact_kept ? preact : nullptr, nullptr,
              nullptr, f32_planes ? &pv : nullptr, gather_xs ? &gth : nullptr);  // expert.cpp:85-102
  gather_combine(ctx, t, ys, d, plan, vals, y);                   // dispatch.cpp:61-78
  ctx_mark(ctx, MARK_GATHER);
  fwd_done = true;
}

void Layer::backward(const void* dy, void* dx, cudaEvent_t dx_ready) {
  if (!fwd_done) protocol_error("backward: no forward cache");
  const int64_t n = cfg.n_b, d = cfg.d_m, h = cfg.d_h, k = cfg.k;
  ctx->prof_slot = prof_slot;  // the forward's profiling slot
  if (cfg.world_size > 1) {
    ep_backward(dy, dx);
    if (dx_ready) CK(cudaEventRecord(dx_ready, ctx->stream));
    ctx->prof_slot = -1;
    return;
  }
  const bool bf = t == FMOE_BF16, gate = bf && !routed;
  ctx_mark(ctx, MARK_BWD_BEGIN);
  // dispatch.cpp:97-126 (+ gate.cpp:44-59 fused on the bf16 path)
  gather_combine_bwd(ctx, t, dy, ys, d, plan, vals, d_ys, d_w, gate ? scores : nullptr, gate ? idx : nullptr,
                     gate ? dz_bf16 : nullptr);
  ctx_mark(ctx, MARK_GCB);
  if (routed) {  // injected routing: no gate (see forward_routed), zero gate gradient
    CK(cudaMemsetAsync(dwg, 0, (size_t)d * E * ss, ctx->stream));
    const int ph = bf ? EXPERTS_BWD_DGRAD : EXPERTS_BWD_ALL;
    const F32Planes pv = planes_view();
    experts_bwd(ctx, t, plan, d, h, params(), xs, hidden, d_ys, d_xs, grads(), d_pre, tpart, relu_bits,
                nullptr, ph, nullptr, nullptr, f32_planes ? &pv : nullptr);
    scatter_bwd(ctx, t, d_xs, d, plan, dx, nullptr);
    ctx_mark(ctx, MARK_GATE_DX);
    if (dx_ready) CK(cudaEventRecord(dx_ready, ctx->stream));
    if (bf) {
      const RowGather gth{x_saved, cfg.n_b, plan.src_row};
      experts_bwd(ctx, t, plan, d, h, params(), xs, hidden, d_ys, d_xs, grads(), d_pre, tpart, relu_bits,
                  nullptr, EXPERTS_BWD_WGRAD, nullptr, nullptr, nullptr, gather_xs ? &gth : nullptr);
    }
  } else if (bf) {
    // Data gradients first (expert.cpp:47-48,55), then the gate d_x on the
    // tensor cores (gate.cpp:63, TMA-store epilogue) and scatter_backward
    // adding it in the reference order (dispatch.cpp:80-95, moe_layer.cpp:140):
    // d_x is final here and can leave the GPU while the weight gradients
    // (expert.cpp:42-45,50-53; gate.cpp:62) are still being computed.
    experts_bwd(ctx, t, plan, d, h, params(), xs, hidden, d_ys, d_xs, grads(), d_pre, tpart, relu_bits,
                nullptr, EXPERTS_BWD_DGRAD);
    gate_dx_bf16(ctx, dz_bf16, wg, n, d, E, nullptr, nullptr, 0, gdx);
    scatter_bwd(ctx, t, d_xs, d, plan, dx, gdx);
    ctx_mark(ctx, MARK_GATE_DX);
    if (dx_ready) CK(cudaEventRecord(dx_ready, ctx->stream));
    const RowGather gth{x_saved, cfg.n_b, plan.src_row};
    experts_bwd(ctx, t, plan, d, h, params(), xs, hidden, d_ys, d_xs, grads(), d_pre, tpart, relu_bits,
                nullptr, EXPERTS_BWD_WGRAD, nullptr, nullptr, nullptr, gather_xs ? &gth : nullptr);
    gate_dwg_bf16(ctx, x_saved, dz_bf16, n, d, E, part, (float*)dwg);  // gate.cpp:62
    ctx_mark(ctx, MARK_GATE_DWG);
  } else {
    const F32Planes pv = planes_view();
    experts_bwd(ctx, t, plan, d, h, params(), xs, hidden, d_ys, d_xs, grads(), d_pre, tpart, relu_bits, nullptr,
                EXPERTS_BWD_ALL, nullptr, nullptr, f32_planes ? &pv : nullptr);  // expert.cpp:104-125
    if (f32_planes) {  // gate.cpp:44-63: Jacobian on SIMT fp32, d_wg / d_x as bf16x6 products
      gate_dlogits(ctx, t, scores, idx, d_w, n, E, k, dz);
      gate_bwd_f32tc(ctx, (const float*)dz, n, d, E, part, (float*)dwg, (float*)gdx, planes_view());
    } else {
      gate_bwd(ctx, t, x_saved, wg, scores, idx, d_w, n, d, E, k, dwg, gdx, dz, nullptr, nullptr);
    }
    ctx_mark(ctx, MARK_GATE_DWG);
    scatter_bwd(ctx, t, d_xs, d, plan, dx, gdx);  // dispatch.cpp:80-95, moe_layer.cpp:140
    ctx_mark(ctx, MARK_GATE_DX);
    if (dx_ready) CK(cudaEventRecord(dx_ready, ctx->stream));
  }
  ctx->prof_slot = -1;
}

// Forward+backward on host buffers.  The PCIe copies run on the context's two
// copy streams and overlap the kernels: inside a step d_y uploads while the
// forward runs, y downloads during the backward and d_x (final before the
// weight gradients, see backward) while they run; across steps (the async
// form) the next step's uploads overlap this step's kernels and this step's
// downloads the next step's kernels, through two device buffer sets.  Set s
// is reused by step t+2 only after step t's kernels (inputs) and downloads
// (outputs) are done -- event-ordered, no host synchronisation.
void Layer::host_io_setup() {
  const size_t bytes = (size_t)(cfg.n_b * cfg.d_m) * es;
  if (!io) {
    io = dalloc_bytes(owned, 8 * std::max<size_t>(bytes, 16));
    for (auto* evs : {hio.x_done, hio.dy_done, hio.y_ready, hio.dx_ready, hio.compute_done, hio.out_done})
      for (int s = 0; s < 2; ++s) CK(cudaEventCreateWithFlags(&evs[s], cudaEventDisableTiming));
  }
  if (!ctx->copy_in) {
    CK(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
    for (auto& e : ctx->ev_io) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
}

void Layer::step_host_submit(const void* x_host, const void* dy_host, void* y_host, void* dx_host) {
  host_io_setup();
  const size_t bytes = (size_t)(cfg.n_b * cfg.d_m) * es;
  const int s = (int)(hio.seq & 1);
  const bool reuse = hio.seq >= 2;  // set s was used by step seq-2
  uint8_t* b = reinterpret_cast<uint8_t*>(io) + (size_t)s * 4 * bytes;
  void *x = b, *y = b + bytes, *gy = b + 2 * bytes, *gx = b + 3 * bytes;
  const bool bwd = dy_host != nullptr;
  // uploads: after step seq-2's kernels released this set's inputs
  if (reuse) CK(cudaStreamWaitEvent(ctx->copy_in, hio.compute_done[s], 0));
  if (bytes) CK(cudaMemcpyAsync(x, x_host, bytes, cudaMemcpyHostToDevice, ctx->copy_in));
  CK(cudaEventRecord(hio.x_done[s], ctx->copy_in));
  if (bwd) {
    if (bytes) CK(cudaMemcpyAsync(gy, dy_host, bytes, cudaMemcpyHostToDevice, ctx->copy_in));
    CK(cudaEventRecord(hio.dy_done[s], ctx->copy_in));
  }
  // kernels: after the inputs landed and step seq-2's downloads left this set
  CK(cudaStreamWaitEvent(ctx->stream, hio.x_done[s], 0));
  if (reuse) CK(cudaStreamWaitEvent(ctx->stream, hio.out_done[s], 0));
  forward(x, y);
  CK(cudaEventRecord(hio.y_ready[s], ctx->stream));
  CK(cudaStreamWaitEvent(ctx->copy_out, hio.y_ready[s], 0));
  if (y_host && bytes) CK(cudaMemcpyAsync(y_host, y, bytes, cudaMemcpyDeviceToHost, ctx->copy_out));
  if (bwd) {
    CK(cudaStreamWaitEvent(ctx->stream, hio.dy_done[s], 0));
    backward(gy, gx, hio.dx_ready[s]);
    if (dx_host) {
      CK(cudaStreamWaitEvent(ctx->copy_out, hio.dx_ready[s], 0));
      if (bytes) CK(cudaMemcpyAsync(dx_host, gx, bytes, cudaMemcpyDeviceToHost, ctx->copy_out));
    }
  }
  CK(cudaEventRecord(hio.compute_done[s], ctx->stream));
  CK(cudaEventRecord(hio.out_done[s], ctx->copy_out));
  ++hio.seq;
}

void Layer::step_host_wait() {
  if (hio.seq == 0) return;
  const int s = (int)((hio.seq - 1) & 1);  // the last step: its streams are ordered after the earlier ones
  CK(cudaEventSynchronize(hio.out_done[s]));
  CK(cudaEventSynchronize(hio.compute_done[s]));
}

void Layer::step_host(const void* x_host, const void* dy_host, void* y_host, void* dx_host) {
  step_host_submit(x_host, dy_host, y_host, dx_host);
  step_host_wait();
}

}  // namespace fmoe_b200
