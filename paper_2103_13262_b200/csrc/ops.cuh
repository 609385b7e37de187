// ops.cuh -- internal operator entry points shared by the C-ABI and the layer.
#pragma once

#include "common.cuh"
#include "plan.cuh"

namespace fmoe_b200 {

// Device scratch owned by the context (grow-only; the layer preallocates so
// its hot path never reallocates).
void* ctx_workspace(Ctx* ctx, size_t bytes);

void gate_fwd(Ctx* ctx, fmoe_dtype t, const void* x, const void* wg, int64_t n, int64_t d, int64_t e,
              int64_t k, void* scores, int32_t* idx, void* vals, void* logits_ws);
// dz_ws: [n, e] in score type (and a bf16 copy for FMOE_BF16 when dz_bf16 != null);
// part_ws: fp32 split-K partials for the bf16 d_wg.
void gate_bwd(Ctx* ctx, fmoe_dtype t, const void* x, const void* wg, const void* scores,
              const int32_t* idx, const void* d_topk, int64_t n, int64_t d, int64_t e, int64_t k,
              void* d_wg, void* d_x, void* dz_ws, __nv_bfloat16* dz_bf16, float* part_ws);
// d_wg of the bf16 path from a bf16 dz (tensor cores, deterministic split-K).
void gate_dwg_bf16(Ctx* ctx, const void* x, const __nv_bfloat16* dz, int64_t n, int64_t d, int64_t e,
                   float* part_ws, float* d_wg);
int64_t gate_dwg_splits(int64_t n);
// bf16 d_x of the gate (+ scatter_backward when d_xs/inverse_pos are given).
void gate_dx_bf16(Ctx* ctx, const __nv_bfloat16* dz, const void* wg, int64_t n, int64_t d, int64_t e,
                  const __nv_bfloat16* d_xs, const int32_t* inverse_pos, int64_t k, void* d_x);

// relu_bits (optional, bf16): [capacity, h/32] bitmap of hidden > 0 written by
// fc1 and consumed by experts_bwd instead of re-reading `hidden` for the mask.
// Fused global_gather target of a bf16 expert GEMM's output rows (see
// tc::Params::route_out): per (local expert, source rank) chunk of the receive
// layout, the source rank's buffer and the destination row of the chunk.
struct RowRoute {
  void* const* out = nullptr;      // [W] device pointers (peer buffers)
  const int32_t* start = nullptr;  // [el*W] first receive row of chunk (e, s)
  const int32_t* rows = nullptr;   // [el*W]
  const int32_t* dst = nullptr;    // [el*W] first row in source s's send layout
  int world = 1;
};
// Overlapped expert-parallel exchange (ep.cu): the first GEMM of a pass (fc1
// forward, dgrad fc2 backward) waits per tile for its rows' chunks to arrive
// (tc::Params::arrive_*), deals row tiles in `mtile_order` and leaves SMs free
// for the concurrent push kernel (grid_limit).
struct Arrival {
  const uint32_t* flags = nullptr;  // [el*W] chunk flags (local memory, written by the senders)
  uint32_t epoch = 0;
  const int32_t* rt = nullptr;      // [start[C], rows[C]]
  int W = 1, C = 0;
  const int* mtile_order = nullptr;
  int grid_limit = 0;
};
// FMOE_F32 GEMMs on the tensor cores (f32x.cu, "bf16x6"): fp32 operands
// split into three bf16 planes ([p0: n][p1: n][p2: n]).  The layer keeps the
// planes of x, xs, hidden and the weights from the forward for the backward;
// per-operator expert calls pass NULL and split into context scratch.
struct F32Planes {
  __nv_bfloat16 *x = nullptr, *wg = nullptr, *dz = nullptr;
  __nv_bfloat16 *xs = nullptr, *hidden = nullptr, *d_ys = nullptr, *d_pre = nullptr, *w1 = nullptr, *w2 = nullptr;
};
// bf16, one GPU: the expanded input rows xs[r] = x[plan.src_row[r]] read straight
// from x by TMA gather4 in fc1 and in the fc1 weight gradient instead of from a
// scattered copy (tc::Params::gather_rows); `xs` is then not read.
struct RowGather {
  const void* x = nullptr;       // [n_b, d] bf16
  int64_t n_b = 0;
  const int32_t* rows = nullptr;  // plan.src_row: [capacity], -1 = padding
};
void experts_fwd(Ctx* ctx, fmoe_dtype t, const fmoe_plan& b, int64_t d, int64_t h,
                 const fmoe_expert_params& w, const void* xs, void* hidden, void* ys,
                 uint32_t* relu_bits = nullptr, void* preact = nullptr, const RowRoute* ys_route = nullptr,
                 const Arrival* arrive = nullptr, const F32Planes* planes = nullptr,
                 const RowGather* gather = nullptr);
// preact (SIMT dtypes only, optional): also keep x*w1 + b1 before the relu
// (ForwardCache::preact, expert.hpp:31-35).
// d_pre_ws: [capacity, h] dtype scratch; mask (SIMT dtypes only, optional): the
// relu-backward operand, preact (strict > 0, matrix.cpp:147-153), default hidden.
// Row alignment of bf16 expert blocks for `rows` routed rows over `experts`:
// 256 (CTA-pair tiles, cta_group::2) once experts average >= 1024 rows, else
// 128 -- with small experts the 256-row padding would cost more than pairs gain.
#ifndef FMOE_PAIR_MIN_ROWS
#define FMOE_PAIR_MIN_ROWS 1024
#endif
inline int64_t expert_block_align(int64_t rows, int64_t experts) {
  return rows >= FMOE_PAIR_MIN_ROWS * experts ? 256 : 128;
}
// phase (bf16 only): the data-gradient GEMMs (d_pre, d_xs) and the weight
// gradients (d_w2, d_b2, d_w1, d_b1) can be issued separately, so d_x is
// final -- and can leave the GPU -- while the weight gradients still run.
enum { EXPERTS_BWD_ALL = 0, EXPERTS_BWD_DGRAD = 1, EXPERTS_BWD_WGRAD = 2 };
void experts_bwd(Ctx* ctx, fmoe_dtype t, const fmoe_plan& b, int64_t d, int64_t h,
                 const fmoe_expert_params& w, const void* xs, const void* hidden, const void* d_ys,
                 void* d_xs, const fmoe_expert_grads& g, void* d_pre_ws, float* part_ws,
                 const uint32_t* relu_bits = nullptr, const void* mask = nullptr,
                 int phase = EXPERTS_BWD_ALL, const RowRoute* dxs_route = nullptr,
                 const Arrival* arrive = nullptr, const F32Planes* planes = nullptr,
                 const RowGather* gather = nullptr);
// FMOE_TC_GATHER=1 enables the gathered A-loads (off by default: slower, see ops.cu)
bool gather_enabled();
// true when an FMOE_F32 expert call takes the tensor-core route: a 128-row
// aligned plan with its tile table, d_m and d_h multiples of 64, and
// FMOE_F32_SIMT unset (=1 keeps the SIMT fp32 kernels, the reference's order)
bool f32_tc_route(const fmoe_plan& b, int64_t d, int64_t h);
bool f32_tc_enabled();
void split_bf16x3(Ctx* ctx, const float* src, __nv_bfloat16* planes, int64_t n);
// a layer's planes: element count and carving of one allocation
int64_t f32_planes_elems(int64_t n, int64_t d, int64_t h, int64_t e, int64_t el, int64_t cap);
F32Planes f32_planes_at(__nv_bfloat16* base, int64_t n, int64_t d, int64_t h, int64_t e, int64_t el, int64_t cap);
// the layer's gate products on the tensor cores (softmax / top-k / Jacobian on SIMT fp32)
void gate_fwd_f32tc(Ctx* ctx, const float* x, const float* wg, int64_t n, int64_t d, int64_t e, int64_t k,
                    float* scores, int32_t* idx, float* vals, float* logits, const F32Planes& pl);
void gate_bwd_f32tc(Ctx* ctx, const float* dz, int64_t n, int64_t d, int64_t e, float* part_ws, float* d_wg,
                    float* d_x, const F32Planes& pl);
void experts_fwd_f32tc(Ctx* ctx, const fmoe_plan& b, int64_t d, int64_t h, const fmoe_expert_params& w,
                       const void* xs, void* hidden, void* ys, void* preact, const F32Planes* pl);
void experts_bwd_f32tc(Ctx* ctx, const fmoe_plan& b, int64_t d, int64_t h, const fmoe_expert_params& w,
                       const void* xs, const void* hidden, const void* d_ys, void* d_xs, const fmoe_expert_grads& g,
                       void* d_pre, const void* mask, int* group_order, const F32Planes* pl);
void relu_rows_f32(Ctx* ctx, const float* in, float* out, int64_t n);

// allreduce_sum over ctx's transport (ep.cu): in place, ascending-rank order.
void allreduce_sum(Ctx* c, fmoe_dtype dt, void* buf, int64_t n, const int* group, int64_t gs);

// fp32 scratch floats experts_bwd needs for the bf16 bias-gradient partials
int64_t experts_bwd_part_floats(const fmoe_plan& b, int64_t d, int64_t h);

}  // namespace fmoe_b200
