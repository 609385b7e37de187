// f32x.cu -- FMOE_F32 on the tcgen05 tensor cores ("bf16x6", see
// tc_gemm.cuh): multi_expert_forward / multi_expert_backward
// (expert.cpp:24-57, 85-125) and the gate products of the layer
// (gate.cpp:23-35, 44-63) at fp32-class accuracy, for 128-row aligned plans.
//
// Every fp32 GEMM operand is first split into three bf16 planes, a0 = bf16(a),
// a1 = bf16(a - a0), a2 = bf16(a - a0 - a1), stored back to back ([a0: n]
// [a1: n][a2: n]); the grouped GEMM contracts the six plane pairs whose
// weights are >= 2^-16 into one fp32 accumulator and writes fp32 results
// through the EPI_F32X epilogue (bias, relu, strict > 0 mask in the SIMT
// kernel's order) or EPI_F32 (weight gradients, logits, d_x, d_wg partials).
// The split is a pure HBM pass (4 bytes in, 6 bytes out per element); the
// layer keeps the planes of x, xs, hidden and the weights from the forward for
// the backward, so each operand is split once per step.  Bias gradients stay
// the fp32 column sums of d_ys / d_pre over each expert's real rows
// (block_colsum, expert.cpp:43-53); softmax / top-k and the softmax Jacobian
// stay on the SIMT fp32 kernels (gate.cu).
#include <algorithm>
#include <cstdlib>

#include "ops.cuh"
#include "plan.cuh"
#include "tc_gemm.cuh"

namespace fmoe_b200 {

namespace {

constexpr int NP = 3;  // planes per operand

__device__ __forceinline__ void split1(float a, __nv_bfloat16& p0, __nv_bfloat16& p1, __nv_bfloat16& p2) {
  p0 = __float2bfloat16_rn(a);
  const float r1 = a - __bfloat162float(p0);  // exact in fp32
  p1 = __float2bfloat16_rn(r1);
  p2 = __float2bfloat16_rn(r1 - __bfloat162float(p1));  // exact in fp32
}

// 4 elements per thread: one 16-byte load, three 8-byte stores.
__global__ void split_bf16x3_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ planes, int64_t n) {
  const int64_t i4 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  __nv_bfloat16* q0 = planes;
  __nv_bfloat16* q1 = planes + n;
  __nv_bfloat16* q2 = planes + 2 * n;
  if (i4 + 4 <= n && (n & 3) == 0) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(src + i4));
    __align__(8) __nv_bfloat16 a[4], b[4], c[4];
    split1(v.x, a[0], b[0], c[0]);
    split1(v.y, a[1], b[1], c[1]);
    split1(v.z, a[2], b[2], c[2]);
    split1(v.w, a[3], b[3], c[3]);
    *reinterpret_cast<uint2*>(q0 + i4) = *reinterpret_cast<const uint2*>(a);
    *reinterpret_cast<uint2*>(q1 + i4) = *reinterpret_cast<const uint2*>(b);
    *reinterpret_cast<uint2*>(q2 + i4) = *reinterpret_cast<const uint2*>(c);
  } else {
    for (int64_t i = i4; i < n && i < i4 + 4; ++i) split1(src[i], q0[i], q1[i], q2[i]);
  }
}

// Tensor maps over the three planes of a row-major [outer, inner] matrix.
struct Maps {
  CUtensorMap p[NP];
};
Maps maps(const __nv_bfloat16* planes, int64_t inner, int64_t outer, uint32_t box_inner, uint32_t box_outer) {
  Maps m;
  for (int i = 0; i < NP; ++i)
    m.p[i] = tc::make_tmap(planes + (int64_t)i * inner * outer, inner, outer, inner * 2, box_inner, box_outer);
  return m;
}

// One split product: the six bf16 passes of tc_gemm.cuh into one accumulator.
void gemm6(Ctx* ctx, int bn, bool a_mn, bool b_mn, const Maps& a, const Maps& b, tc::Params p, int64_t max_tiles,
           int cg) {
  p.phases = tc::SPLIT_PASSES;
  p.sel_a = tc::SPLIT_SEL_A;
  p.sel_b = tc::SPLIT_SEL_B;
  p.probe = ctx_probe_slot(ctx);
  const tc::SplitMaps sm{a.p[1], a.p[2], b.p[1], b.p[2]};
  tc::launch(ctx, bn, a_mn, b_mn, a.p[0], b.p[0], p, max_tiles, cg, &sm);
}

__nv_bfloat16* planes_ws(Ctx* ctx, int64_t elems) {
  // grow-only; per-operator calls (no layer-owned planes) split into it
  const size_t bytes = (size_t)std::max<int64_t>(elems, 64) * NP * sizeof(__nv_bfloat16);
  if (ctx->pws_size < bytes) {
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->pws) CK(cudaFree(ctx->pws));
    ctx->pws = nullptr;
    CK(cudaMalloc(&ctx->pws, bytes));
    ctx->pws_size = bytes;
  }
  return reinterpret_cast<__nv_bfloat16*>(ctx->pws);
}

}  // namespace

void split_bf16x3(Ctx* ctx, const float* src, __nv_bfloat16* planes, int64_t n) {
  if (n <= 0) return;
  split_bf16x3_kernel<<<(unsigned)ceil_div(ceil_div(n, 4), 256), 256, 0, ctx->stream>>>(src, planes, n);
  CK_LAUNCH(ctx);
}

bool f32_tc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FMOE_F32_SIMT");
    return !(e && std::atoi(e) != 0);
  }();
  return on;
}

bool f32_tc_route(const fmoe_plan& b, int64_t d, int64_t h) {
  return f32_tc_enabled() && b.align % 128 == 0 && b.tile_expert && b.n_tiles && d % 64 == 0 && h % 64 == 0;
}

int64_t f32_planes_elems(int64_t n, int64_t d, int64_t h, int64_t e, int64_t el, int64_t cap) {
  return NP * (n * d + d * e + n * e + 2 * cap * d + 2 * cap * h + 2 * el * d * h);
}

F32Planes f32_planes_at(__nv_bfloat16* base, int64_t n, int64_t d, int64_t h, int64_t e, int64_t el, int64_t cap) {
  F32Planes v{};
  v.x = base;
  v.wg = v.x + NP * n * d;
  v.dz = v.wg + NP * d * e;
  v.xs = v.dz + NP * n * e;
  v.d_ys = v.xs + NP * cap * d;
  v.hidden = v.d_ys + NP * cap * d;
  v.d_pre = v.hidden + NP * cap * h;
  v.w1 = v.d_pre + NP * cap * h;
  v.w2 = v.w1 + NP * el * d * h;
  return v;
}

// ------------------------------------------------------------------ gate
void gate_fwd_f32tc(Ctx* ctx, const float* x, const float* wg, int64_t n, int64_t d, int64_t e, int64_t k,
                    float* scores, int32_t* idx, float* vals, float* logits, const F32Planes& pl) {
  if (k < 1 || k > e) shape_error("gate_forward: k out of range");
  if (n == 0) return;
  split_bf16x3(ctx, x, pl.x, n * d);
  split_bf16x3(ctx, wg, pl.wg, d * e);
  // logits = x Wg (gate.cpp:30): A = x [n, d] K-major, B = Wg [d, E] MN-major
  const Maps a = maps(pl.x, d, n, 64, 128), b = maps(pl.wg, e, d, 64, 64);
  tc::Params p{};
  p.mode = tc::RAGGED_M; p.M = (int)n; p.N = (int)e; p.K = (int)d;
  p.epi = tc::EPI_F32; p.C = logits; p.ldc = e;
  const int bn = e <= 64 ? 64 : e <= 128 ? 128 : 256;
  gemm6(ctx, bn, false, true, a, b, p, ceil_div(n, 128) * ceil_div(e, bn), 1);
  gate_softmax_topk(ctx, FMOE_F32, logits, n, e, k, scores, idx, vals, false);  // gate.cpp:31-33
}

void gate_bwd_f32tc(Ctx* ctx, const float* dz, int64_t n, int64_t d, int64_t e, float* part_ws, float* d_wg,
                    float* d_x, const F32Planes& pl) {
  if (n == 0) {
    if (d * e) CK(cudaMemsetAsync(d_wg, 0, (size_t)(d * e) * 4, ctx->stream));
    return;
  }
  split_bf16x3(ctx, dz, pl.dz, n * e);
  {  // d_wg = x^T dz (gate.cpp:62): split-K partials over token ranges + ordered reduce
    const int64_t S = gate_dwg_splits(n);
    const int64_t per = ceil_div(ceil_div(n, S), 64) * 64;
    const Maps a = maps(pl.x, d, n, 64, 64), b = maps(pl.dz, e, n, 64, 64);  // both MN-major
    tc::Params p{};
    p.mode = tc::RAGGED_K; p.M = (int)d; p.N = (int)e; p.K = (int)n; p.n_groups = (int)S; p.k_split = (int)per;
    p.epi = tc::EPI_F32; p.C = part_ws; p.ldc = e; p.c_group_stride = d * e;
    const int bn = e <= 64 ? 64 : e <= 128 ? 128 : 256;
    gemm6(ctx, bn, true, true, a, b, p, S * ceil_div(d, 128) * ceil_div(e, bn), 1);
    reduce_splits(ctx, part_ws, S, d * e, d_wg);
  }
  if (d_x) {  // d_x = dz Wg^T (gate.cpp:63): A = dz [n, E] K-major; B(k=e, n=c) = Wg[c][e] K-major
    const Maps a = maps(pl.dz, e, n, 64, 128), b = maps(pl.wg, e, d, 64, 256);
    tc::Params p{};
    p.mode = tc::RAGGED_M; p.M = (int)n; p.N = (int)d; p.K = (int)e;
    p.epi = tc::EPI_F32; p.C = d_x; p.ldc = d;
    gemm6(ctx, 256, false, false, a, b, p, ceil_div(n, 128) * ceil_div(d, 256), 1);
  }
}

// --------------------------------------------------------------- experts
void experts_fwd_f32tc(Ctx* ctx, const fmoe_plan& b, int64_t d, int64_t h, const fmoe_expert_params& w,
                       const void* xs, void* hidden, void* ys, void* preact, const F32Planes* pl) {
  const int64_t E = b.n_experts, cap = b.capacity;
  const int cg = b.align % 256 == 0 ? 2 : 1;
  const int64_t max_tiles = cap / (128 * cg);
  // operand planes: the layer's (kept for the backward) or per-call scratch
  F32Planes s{};
  if (pl) {
    s = *pl;
  } else {
    __nv_bfloat16* ws = planes_ws(ctx, cap * d + E * d * h + cap * h + E * h * d);
    s.xs = ws;
    s.w1 = s.xs + NP * cap * d;
    s.hidden = s.w1 + NP * E * d * h;
    s.w2 = s.hidden + NP * cap * h;
  }
  split_bf16x3(ctx, (const float*)xs, s.xs, cap * d);
  split_bf16x3(ctx, (const float*)w.w1, s.w1, E * d * h);
  split_bf16x3(ctx, (const float*)w.w2, s.w2, E * h * d);
  {  // fc1: hidden = relu(xs W1 + b1); A = xs [cap, d] K-major, B = W1 [E*d, h] MN-major
    const Maps a = maps(s.xs, d, cap, 64, 128), bb = maps(s.w1, h, E * d, 64, 64);
    tc::Params p{};
    p.mode = tc::RAGGED_M; p.M = (int)cap; p.N = (int)h; p.K = (int)d;
    p.tile_group = b.tile_expert; p.n_mtiles = b.n_tiles; p.b_group_rows = (int)d;
    p.epi = tc::EPI_F32X; p.C = preact ? preact : hidden; p.ldc = h;
    p.bias = (const float*)w.b1; p.bias_group_stride = h; p.relu = preact ? 0 : 1;
    gemm6(ctx, 256, false, true, a, bb, p, max_tiles * ceil_div(h, 256), cg);
    if (preact) relu_rows_f32(ctx, (const float*)preact, (float*)hidden, cap * h);  // cache.preact kept
    ctx_mark(ctx, MARK_FC1);
  }
  split_bf16x3(ctx, (const float*)hidden, s.hidden, cap * h);
  {  // fc2: ys = hidden W2 + b2; A = hidden [cap, h] K-major, B = W2 [E*h, d] MN-major
    const Maps a = maps(s.hidden, h, cap, 64, 128), bb = maps(s.w2, d, E * h, 64, 64);
    tc::Params p{};
    p.mode = tc::RAGGED_M; p.M = (int)cap; p.N = (int)d; p.K = (int)h;
    p.tile_group = b.tile_expert; p.n_mtiles = b.n_tiles; p.b_group_rows = (int)h;
    p.epi = tc::EPI_F32X; p.C = ys; p.ldc = d;
    p.bias = (const float*)w.b2; p.bias_group_stride = d;
    gemm6(ctx, 256, false, true, a, bb, p, max_tiles * ceil_div(d, 256), cg);
    ctx_mark(ctx, MARK_FC2);
  }
}

void experts_bwd_f32tc(Ctx* ctx, const fmoe_plan& b, int64_t d, int64_t h, const fmoe_expert_params& w,
                       const void* xs, const void* hidden, const void* d_ys, void* d_xs, const fmoe_expert_grads& g,
                       void* d_pre, const void* mask, int* group_order, const F32Planes* pl) {
  const int64_t E = b.n_experts, cap = b.capacity;
  const int cg = b.align % 256 == 0 ? 2 : 1;
  const int64_t max_tiles = cap / (128 * cg);
  F32Planes s{};
  if (pl) {
    s = *pl;
  } else {  // per-call scratch: the forward's planes are not kept
    __nv_bfloat16* ws = planes_ws(ctx, 2 * cap * d + 2 * E * d * h + 2 * cap * h);
    s.xs = ws;
    s.w1 = s.xs + NP * cap * d;
    s.hidden = s.w1 + NP * E * d * h;
    s.w2 = s.hidden + NP * cap * h;
    s.d_ys = s.w2 + NP * E * h * d;
    s.d_pre = s.d_ys + NP * cap * d;
    split_bf16x3(ctx, (const float*)xs, s.xs, cap * d);
    split_bf16x3(ctx, (const float*)w.w1, s.w1, E * d * h);
    split_bf16x3(ctx, (const float*)hidden, s.hidden, cap * h);
    split_bf16x3(ctx, (const float*)w.w2, s.w2, E * h * d);
  }
  split_bf16x3(ctx, (const float*)d_ys, s.d_ys, cap * d);
  {  // dgrad fc2: d_pre = (d_ys W2^T) * (mask > 0); B(k=c, n=j) = W2[e][j][c] -> K-major [E*h, d]
    const Maps a = maps(s.d_ys, d, cap, 64, 128), bb = maps(s.w2, d, E * h, 64, 256 / cg);
    tc::Params p{};
    p.mode = tc::RAGGED_M; p.M = (int)cap; p.N = (int)h; p.K = (int)d;
    p.tile_group = b.tile_expert; p.n_mtiles = b.n_tiles; p.b_group_rows = (int)h;
    p.epi = tc::EPI_F32X; p.C = d_pre; p.ldc = h;
    p.maskf = (const float*)(mask ? mask : hidden); p.ldm = h;
    gemm6(ctx, 256, false, false, a, bb, p, max_tiles * ceil_div(h, 256), cg);
    ctx_mark(ctx, MARK_DGRAD2);
  }
  order_groups_desc(ctx, b.offsets, E, group_order);  // heaviest expert first
  {  // wgrad fc2: d_w2[e] = hidden_e^T d_ys_e (M = h, N = d, K = rows of e)
    const Maps a = maps(s.hidden, h, cap, 64, 64), bb = maps(s.d_ys, d, cap, 64, 64);
    tc::Params p{};
    p.mode = tc::RAGGED_K; p.M = (int)h; p.N = (int)d; p.n_groups = (int)E; p.k_offsets = b.offsets;
    p.group_order = group_order;
    p.epi = tc::EPI_F32; p.C = g.d_w2; p.ldc = d; p.c_group_stride = h * d;
    gemm6(ctx, 256, true, true, a, bb, p, E * ceil_div(h, 128 * cg) * ceil_div(d, 256), cg);
    ctx_mark(ctx, MARK_WGRAD2);
  }
  block_colsum(ctx, FMOE_F32, d_ys, d, b.offsets, b.counts, E, g.d_b2);  // expert.cpp:43-45
  ctx_mark(ctx, MARK_DB2);
  split_bf16x3(ctx, (const float*)d_pre, s.d_pre, cap * h);
  {  // dgrad fc1: d_xs = d_pre W1^T; B(k=j, n=c) = W1[e][c][j] -> K-major [E*d, h]
    const Maps a = maps(s.d_pre, h, cap, 64, 128), bb = maps(s.w1, h, E * d, 64, 256 / cg);
    tc::Params p{};
    p.mode = tc::RAGGED_M; p.M = (int)cap; p.N = (int)d; p.K = (int)h;
    p.tile_group = b.tile_expert; p.n_mtiles = b.n_tiles; p.b_group_rows = (int)d;
    p.epi = tc::EPI_F32X; p.C = d_xs; p.ldc = d;
    gemm6(ctx, 256, false, false, a, bb, p, max_tiles * ceil_div(d, 256), cg);
    ctx_mark(ctx, MARK_DGRAD1);
  }
  {  // wgrad fc1: d_w1[e] = xs_e^T d_pre_e (M = d, N = h)
    const Maps a = maps(s.xs, d, cap, 64, 64), bb = maps(s.d_pre, h, cap, 64, 64);
    tc::Params p{};
    p.mode = tc::RAGGED_K; p.M = (int)d; p.N = (int)h; p.n_groups = (int)E; p.k_offsets = b.offsets;
    p.group_order = group_order;
    p.epi = tc::EPI_F32; p.C = g.d_w1; p.ldc = h; p.c_group_stride = d * h;
    gemm6(ctx, 256, true, true, a, bb, p, E * ceil_div(d, 128 * cg) * ceil_div(h, 256), cg);
    ctx_mark(ctx, MARK_WGRAD1);
  }
  block_colsum(ctx, FMOE_F32, d_pre, h, b.offsets, b.counts, E, g.d_b1);  // expert.cpp:51-53
  ctx_mark(ctx, MARK_DB1);
}

}  // namespace fmoe_b200
