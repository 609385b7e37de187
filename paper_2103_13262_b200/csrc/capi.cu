#include <vector>
// capi.cu -- the extern "C" boundary (include/fmoe_b200.h): context, operator
// entry points and status/error mapping.  Internal exceptions never cross it.
#include <cstring>
#include <string>

#include "ops.cuh"

namespace fmoe_b200 {
thread_local std::string g_last_error;

int guard_status(const std::exception& e) {
  g_last_error = e.what();
  if (auto* f = dynamic_cast<const Error*>(&e)) return f->code;
  return FMOE_ERR_CUDA;
}

void* ctx_workspace(Ctx* ctx, size_t bytes);
}  // namespace fmoe_b200

using namespace fmoe_b200;

#define FMOE_GUARD(...)                               \
  try {                                               \
    __VA_ARGS__;                                      \
    return FMOE_OK;                                   \
  } catch (const std::exception& e) {                 \
    return guard_status(e);                           \
  } catch (...) {                                     \
    g_last_error = "unknown error";                   \
    return FMOE_ERR_CUDA;                             \
  }

namespace {
void need(const void* p, const char* what) {
  if (!p) shape_error(std::string(what) + " is null");
}
Ctx* C(fmoe_ctx* c) {
  if (!c) shape_error("null context");
  return reinterpret_cast<Ctx*>(c);
}
void check_plan(const fmoe_plan* p) {
  if (!p) shape_error("null plan");
  need(p->counts, "plan.counts");
  need(p->offsets, "plan.offsets");
  need(p->inverse_pos, "plan.inverse_pos");
}

}  // namespace

namespace fmoe_b200 {
void* ctx_workspace(Ctx* ctx, size_t bytes) {
  if (bytes < 256) bytes = 256;
  if (ctx->ws_size < bytes) {
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->ws) CK(cudaFree(ctx->ws));
    ctx->ws = nullptr;
    CK(cudaMalloc(&ctx->ws, bytes));
    ctx->ws_size = bytes;
  }
  return ctx->ws;
}
}  // namespace fmoe_b200

extern "C" {

const char* fmoe_last_error(void) { return g_last_error.c_str(); }
const char* fmoe_version(void) { return "fmoe_b200 0.1 (sm_100a)"; }

int fmoe_ctx_create(int device, void* stream, fmoe_ctx** out) {
  FMOE_GUARD({
    need(out, "out");
    CK(cudaSetDevice(device));
    auto* c = new Ctx;
    c->device = device;
    c->stream = reinterpret_cast<cudaStream_t>(stream);
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaMalloc(&c->d_error, sizeof(int)));
    CK(cudaMemset(c->d_error, 0, sizeof(int)));
    *out = reinterpret_cast<fmoe_ctx*>(c);
  })
}

int fmoe_ctx_destroy(fmoe_ctx* ctx) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    cudaFree(c->d_error);
    if (c->d_probe) cudaFree(c->d_probe);
    if (c->ws) cudaFree(c->ws);
    if (c->pws) cudaFree(c->pws);
    if (c->copy_in) cudaStreamDestroy(c->copy_in);
    if (c->copy_out) cudaStreamDestroy(c->copy_out);
    for (auto e : c->ev_io)
      if (e) cudaEventDestroy(e);
    delete c;
  })
}

int fmoe_ctx_set_stream(fmoe_ctx* ctx, void* stream) {
  FMOE_GUARD(C(ctx)->stream = reinterpret_cast<cudaStream_t>(stream))
}

int64_t fmoe_ctx_launches(const fmoe_ctx* ctx) {
  return ctx ? reinterpret_cast<const Ctx*>(ctx)->launches : 0;
}

int fmoe_ctx_profile(fmoe_ctx* ctx, int n_steps) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    if (c->prof) {
      CK(cudaStreamSynchronize(c->stream));
      for (auto e : c->prof->ev) cudaEventDestroy(e);
      delete c->prof;
      c->prof = nullptr;
    }
    if (n_steps > 0) {
      auto* p = new Prof;
      p->steps = n_steps;
      p->ev.resize((size_t)n_steps * N_MARKS);
      p->prev.assign((size_t)n_steps * N_MARKS, (int8_t)-1);
      p->last.assign((size_t)n_steps, (int8_t)-1);
      for (auto& e : p->ev) CK(cudaEventCreate(&e));
      c->prof = p;
    }
  })
}

int fmoe_ctx_profile_read(fmoe_ctx* ctx, float* stage_ms, int n_stages, int* steps_done) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    Prof* p = c->prof;
    if (!p) shape_error("profiling not armed");
    CK(cudaStreamSynchronize(c->stream));
    for (int i = 0; i < n_stages; ++i) stage_ms[i] = 0.f;
    for (int s = 0; s < p->used; ++s)
      for (int i = 1; i < N_MARKS && i < n_stages; ++i) {
        const int from = p->prev[(size_t)s * N_MARKS + i];
        if (from < 0) continue;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, p->ev[(size_t)s * N_MARKS + from], p->ev[(size_t)s * N_MARKS + i]));
        stage_ms[i] += ms;
      }
    if (steps_done) *steps_done = p->used;
  })
}

int fmoe_ctx_profile_step_ms(fmoe_ctx* ctx, float* step_ms, int n) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    Prof* p = c->prof;
    if (!p) shape_error("profiling not armed");
    CK(cudaStreamSynchronize(c->stream));
    for (int s = 0; s < n; ++s) {
      step_ms[s] = 0.f;
      if (s >= p->used || p->last[s] < 0) continue;
      const size_t b = (size_t)s * N_MARKS;
      // slot s's first mark to the next slot's first mark (the last slot: to its last mark)
      cudaEvent_t to = (s + 1 < p->used && p->last[s + 1] >= 0) ? p->ev[b + N_MARKS + MARK_FWD_BEGIN]
                                                              : p->ev[b + p->last[s]];
      CK(cudaEventElapsedTime(&step_ms[s], p->ev[b + MARK_FWD_BEGIN], to));
    }
  })
}

int fmoe_ctx_clock_probe(fmoe_ctx* ctx, int max_launches) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    CK(cudaStreamSynchronize(c->stream));
    if (c->d_probe) cudaFree(c->d_probe);
    c->d_probe = nullptr;
    c->probe_cap = c->probe_next = 0;
    if (max_launches > 0) {
      CK(cudaMalloc(&c->d_probe, (size_t)max_launches * 4 * 8));
      CK(cudaMemset(c->d_probe, 0, (size_t)max_launches * 4 * 8));
      c->probe_cap = max_launches;
    }
  })
}

int fmoe_ctx_clock_probe_read(fmoe_ctx* ctx, double* sm_mhz, int* launches) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    if (!c->d_probe) shape_error("clock probe not armed");
    CK(cudaStreamSynchronize(c->stream));
    std::vector<unsigned long long> v((size_t)c->probe_next * 4);
    if (!v.empty()) CK(cudaMemcpy(v.data(), c->d_probe, v.size() * 8, cudaMemcpyDeviceToHost));
    double cyc = 0.0, ns = 0.0;
    int n = 0;
    for (int i = 0; i < c->probe_next; ++i) {
      const unsigned long long* q = v.data() + 4 * i;
      if (q[2] <= q[0] || q[3] <= q[1]) continue;
      cyc += (double)(q[2] - q[0]);
      ns += (double)(q[3] - q[1]);
      ++n;
    }
    if (sm_mhz) *sm_mhz = ns > 0 ? cyc / ns * 1e3 : 0.0;
    if (launches) *launches = n;
  })
}

int fmoe_ctx_check(fmoe_ctx* ctx) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    CK(cudaStreamSynchronize(c->stream));
    int flag = 0;
    CK(cudaMemcpy(&flag, c->d_error, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) {
      CK(cudaMemset(c->d_error, 0, sizeof(int)));
      shape_error("build_plan: expert index out of range");
    }
  })
}

int fmoe_gate_fwd(fmoe_ctx* ctx, fmoe_dtype dtype, const void* x, const void* w_g, int64_t n_b,
                  int64_t d_m, int64_t n_experts, int64_t k, void* scores, int32_t* topk_idx,
                  void* topk_scores) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    if (n_b < 0 || d_m < 1 || n_experts < 1) shape_error("gate_forward: bad shape");
    if (k < 1 || k > n_experts) shape_error("gate_forward: k out of range");
    if (n_b == 0) return FMOE_OK;
    need(x, "x"); need(w_g, "w_g"); need(scores, "scores"); need(topk_idx, "topk_idx");
    need(topk_scores, "topk_scores");
    void* ws = nullptr;
    if (dtype != FMOE_BF16 || n_experts > 256)
      ws = ctx_workspace(c, (size_t)(n_b * n_experts) * score_size(dtype));
    gate_fwd(c, dtype, x, w_g, n_b, d_m, n_experts, k, scores, topk_idx, topk_scores, ws);
  })
}

int fmoe_gate_bwd(fmoe_ctx* ctx, fmoe_dtype dtype, const void* x, const void* w_g,
                  const void* scores, const int32_t* topk_idx, const void* d_topk, int64_t n_b,
                  int64_t d_m, int64_t n_experts, int64_t k, void* d_wg, void* d_x) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    if (k < 1 || k > n_experts) shape_error("gate_backward: k out of range");
    need(d_wg, "d_wg");
    const size_t ss = score_size(dtype);
    const int64_t S = gate_dwg_splits(n_b);
    size_t bytes = (size_t)(n_b * n_experts) * ss;                    // dz
    const size_t o_bf = (bytes + 255) / 256 * 256;
    bytes = o_bf + (size_t)(n_b * n_experts) * 2;                     // dz bf16
    const size_t o_part = (bytes + 255) / 256 * 256;
    bytes = o_part + (size_t)(S * d_m * n_experts) * 4 + (S + 1) * 4 + 256;  // partials + offsets
    uint8_t* ws = (uint8_t*)ctx_workspace(c, bytes);
    gate_bwd(c, dtype, x, w_g, scores, topk_idx, d_topk, n_b, d_m, n_experts, k, d_wg, d_x, ws,
             (__nv_bfloat16*)(ws + o_bf), (float*)(ws + o_part));
  })
}

int fmoe_plan_sizes(int64_t n_b, int64_t k, int64_t n_experts, int64_t align, int64_t* capacity,
                    int64_t* scratch_bytes) {
  FMOE_GUARD({
    if (n_b < 0 || k < 1 || n_experts < 1) shape_error("plan: bad sizes");
    if (capacity) *capacity = plan_capacity(n_b, k, n_experts, align);
    if (scratch_bytes) *scratch_bytes = plan_scratch_bytes(n_b, k, n_experts);
  })
}

int fmoe_plan_build(fmoe_ctx* ctx, const int32_t* topk_idx, fmoe_plan* plan, int validate) {
  FMOE_GUARD({
    Ctx* c = C(ctx);
    check_plan(plan);
    if (plan->n_b * plan->k > 0) need(topk_idx, "topk_idx");
    if (plan->capacity < plan_capacity(plan->n_b, plan->k, plan->n_experts, plan->align))
      shape_error("build_plan: capacity too small for this alignment");
    plan_build(c, topk_idx, *plan);
    if (validate) {
      CK(cudaStreamSynchronize(c->stream));
      int flag = 0;
      CK(cudaMemcpy(&flag, c->d_error, sizeof(int), cudaMemcpyDeviceToHost));
      if (flag) {
        CK(cudaMemset(c->d_error, 0, sizeof(int)));
        shape_error("build_plan: expert index out of range [0, " + std::to_string(plan->n_experts) + ")");
      }
    }
  })
}

int fmoe_scatter(fmoe_ctx* ctx, fmoe_dtype dtype, const void* x, int64_t d, const fmoe_plan* plan,
                 void* xs) {
  FMOE_GUARD({
    check_plan(plan);
    scatter(C(ctx), dtype, x, d, *plan, xs);
  })
}

int fmoe_gather_combine(fmoe_ctx* ctx, fmoe_dtype dtype, const void* ys, int64_t d,
                        const fmoe_plan* plan, const void* topk_scores, void* y) {
  FMOE_GUARD({
    check_plan(plan);
    gather_combine(C(ctx), dtype, ys, d, *plan, topk_scores, y);
  })
}

int fmoe_scatter_bwd(fmoe_ctx* ctx, fmoe_dtype dtype, const void* d_xs, int64_t d,
                     const fmoe_plan* plan, void* d_x) {
  FMOE_GUARD({
    check_plan(plan);
    scatter_bwd(C(ctx), dtype, d_xs, d, *plan, d_x);
  })
}

int fmoe_gather_combine_bwd(fmoe_ctx* ctx, fmoe_dtype dtype, const void* d_y, const void* ys,
                            int64_t d, const fmoe_plan* plan, const void* topk_scores, void* d_ys,
                            void* d_topk) {
  FMOE_GUARD({
    check_plan(plan);
    gather_combine_bwd(C(ctx), dtype, d_y, ys, d, *plan, topk_scores, d_ys, d_topk, nullptr, nullptr,
                       nullptr);
  })
}

int fmoe_experts_fwd(fmoe_ctx* ctx, fmoe_dtype dtype, const fmoe_plan* blocks, int64_t d_m,
                     int64_t d_h, fmoe_expert_params params, const void* xs, void* hidden, void* ys) {
  FMOE_GUARD({
    check_plan(blocks);
    experts_fwd(C(ctx), dtype, *blocks, d_m, d_h, params, xs, hidden, ys);
  })
}

int fmoe_experts_bwd(fmoe_ctx* ctx, fmoe_dtype dtype, const fmoe_plan* blocks, int64_t d_m,
                     int64_t d_h, fmoe_expert_params params, const void* xs, const void* hidden,
                     const void* d_ys, void* d_xs, fmoe_expert_grads grads) {
  FMOE_GUARD({
    check_plan(blocks);
    Ctx* c = C(ctx);
    const size_t pre_bytes = ((size_t)(blocks->capacity * d_h) * dtype_size(dtype) + 255) / 256 * 256;
    uint8_t* ws = (uint8_t*)ctx_workspace(
        c, pre_bytes + (size_t)experts_bwd_part_floats(*blocks, d_m, d_h) * 4 + 256);
    experts_bwd(c, dtype, *blocks, d_m, d_h, params, xs, hidden, d_ys, d_xs, grads, ws,
                (float*)(ws + pre_bytes));
  })
}

}  // extern "C"
