// ops.cu -- gate and expert-pool operators for every dtype.
//
// FMOE_F64 / FMOE_F32 run the SIMT kernels (gemm_simt.cu, gate.cu) in the
// reference's accumulation order.  FMOE_BF16 runs the tcgen05 grouped GEMM
// (tc_gemm.cu): operands are used in their stored layouts through K-major or
// MN-major TMA descriptors, so no transpose is ever materialised.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "gemm_simt.cuh"
#include "ops.cuh"
#include "tc_gemm.cuh"

namespace fmoe_b200 {

void* ctx_workspace(Ctx* ctx, size_t bytes);

namespace {


__global__ void cast_f32_bf16(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __float2bfloat16_rn(in[i]);
}

// relu (matrix.cpp:140-145): x < 0 -> 0, so -0.0 survives.
template <typename T>
__global__ void relu_kernel(const T* __restrict__ in, T* __restrict__ out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const T v = in[i];
    out[i] = v < T(0) ? T(0) : v;
  }
}
template <typename T>
void relu_rows(Ctx* ctx, const T* in, T* out, int64_t n) {
  if (n <= 0) return;
  relu_kernel<T><<<(unsigned)ceil_div(n, 256), 256, 0, ctx->stream>>>(in, out, n);
  CK_LAUNCH(ctx);
}
}  // namespace

void relu_rows_f32(Ctx* ctx, const float* in, float* out, int64_t n) { relu_rows<float>(ctx, in, out, n); }

namespace {

int pick_bn(int64_t n) { return n <= 64 ? 64 : n <= 128 ? 128 : 256; }

void require_bf16_dims(int64_t d, int64_t h) {
  if (d % 64 || h % 64)
    shape_error("bf16 tensor-core path needs d_m and d_h to be multiples of 64 (got " +
                std::to_string(d) + ", " + std::to_string(h) + ")");
}

// CTA-pair (cta_group::2) tiles need expert blocks aligned to 256 rows.
int pair_mode(const fmoe_plan& b) { return b.align % 256 == 0 ? 2 : 1; }

std::vector<int32_t> host_counts(Ctx* ctx, const fmoe_plan& b) {
  std::vector<int32_t> c((size_t)b.n_experts);
  if (!c.empty())
    CK(cudaMemcpyAsync(c.data(), b.counts, c.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return c;
}

}  // namespace

int64_t gate_dwg_splits(int64_t n) {
  // ~2 waves of (d/128 x 1) tiles over 148 SMs; each split a multiple of 64 rows
  return std::max<int64_t>(1, std::min<int64_t>(37, ceil_div(n, 512)));
}

// ---------------------------------------------------------------- gate fwd
void gate_fwd(Ctx* ctx, fmoe_dtype t, const void* x, const void* wg, int64_t n, int64_t d, int64_t e,
              int64_t k, void* scores, int32_t* idx, void* vals, void* logits_ws) {
  if (k < 1 || k > e) shape_error("gate_forward: k out of range");
  if (n == 0) return;
  if (t == FMOE_F64 || t == FMOE_F32) {
    auto run = [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      SimtParams<T> p;
      p.M = n; p.N = e; p.K = d;
      p.A = (const T*)x; p.sa_m = d; p.sa_k = 1;
      p.B = (const T*)wg; p.sb_k = e; p.sb_n = 1;
      p.C = (T*)logits_ws; p.ldc = e;
      simt_gemm<T>(ctx, p, n);
    };
    if (t == FMOE_F64) run((double*)nullptr); else run((float*)nullptr);
    gate_softmax_topk(ctx, t, logits_ws, n, e, k, scores, idx, vals, false);
    return;
  }
  // bf16: x [n, d] K-major; Wg [d, E] used MN-major (B(k=c, n=e) = Wg[c][e]).
  if (d % 64) shape_error("bf16 gate needs d_m multiple of 64");
  if (e % 8) shape_error("bf16 gate needs the expert count to be a multiple of 8");
  const CUtensorMap ta = tc::make_tmap(x, d, n, d * 2, 64, 128);
  const CUtensorMap tb = tc::make_tmap(wg, e, d, e * 2, 64, 64);
  tc::Params p{};
  p.mode = tc::RAGGED_M;
  p.M = (int)n; p.N = (int)e; p.K = (int)d;
  if (e <= 256) {
    p.epi = tc::EPI_GATE;
    p.scores = (float*)scores;
    p.topk_idx = idx;
    p.topk_val = (float*)vals;
    p.topk = k <= 8 ? (int)k : 0;
    p.row_split = 1;  // balanced row ranges per SM (tc_gemm.cuh)
    const int bn = pick_bn(e);
    tc::launch(ctx, bn, false, true, ta, tb, p, ceil_div(n, 128));
    if (k > 8) gate_softmax_topk(ctx, FMOE_F32, nullptr, n, e, k, scores, idx, vals, true);
  } else {
    p.epi = tc::EPI_F32;
    p.C = logits_ws; p.ldc = e;
    tc::launch(ctx, 256, false, true, ta, tb, p, ceil_div(n, 128) * ceil_div(e, 256));
    gate_softmax_topk(ctx, FMOE_F32, logits_ws, n, e, k, scores, idx, vals, false);
  }
}

// ---------------------------------------------------------------- gate bwd
void gate_dwg_bf16(Ctx* ctx, const void* x, const __nv_bfloat16* dz, int64_t n, int64_t d, int64_t e,
                   float* part_ws, float* d_wg) {
  if (n == 0) {  // no tokens: the gate gradient is zero
    if (d * e) CK(cudaMemsetAsync(d_wg, 0, (size_t)(d * e) * 4, ctx->stream));
    return;
  }
  const int64_t S = gate_dwg_splits(n);
  const int64_t per = ceil_div(ceil_div(n, S), 64) * 64;
  const CUtensorMap ta = tc::make_tmap(x, d, n, d * 2, 64, 64);   // x^T: MN-major
  const CUtensorMap tb = tc::make_tmap(dz, e, n, e * 2, 64, 64);  // dz: MN-major
  tc::Params p{};
  p.mode = tc::RAGGED_K;
  p.M = (int)d; p.N = (int)e; p.K = (int)n; p.n_groups = (int)S; p.k_split = (int)per;  // split s: rows [s*per, ...)
  p.epi = tc::EPI_F32; p.C = part_ws; p.ldc = e; p.c_group_stride = d * e;
  const int bn = pick_bn(e);
  tc::launch(ctx, bn, true, true, ta, tb, p, S * ceil_div(d, 128) * ceil_div(e, bn));
  reduce_splits(ctx, part_ws, S, d * e, d_wg);
}

void gate_dx_bf16(Ctx* ctx, const __nv_bfloat16* dz, const void* wg, int64_t n, int64_t d, int64_t e,
                  const __nv_bfloat16* d_xs, const int32_t* inverse_pos, int64_t k, void* d_x) {
  if (n == 0) return;
  const CUtensorMap ta = tc::make_tmap(dz, e, n, e * 2, 64, 128);   // dz [n, E] K-major
  const CUtensorMap tb = tc::make_tmap(wg, e, d, e * 2, 64, 256);   // Wg^T: B(k=e, n=c) = Wg[c][e], K-major
  tc::Params p{};
  p.mode = tc::RAGGED_M;
  p.M = (int)n; p.N = (int)d; p.K = (int)e;
  p.epi = d_xs ? tc::EPI_GATE_DX : tc::EPI_BF16;
  p.C = d_x; p.ldc = d;
  p.gather_src = d_xs; p.inverse_pos = inverse_pos; p.gk = (int)k;
  tc::launch(ctx, 256, false, false, ta, tb, p, ceil_div(n, 128) * ceil_div(d, 256));
}

void gate_bwd(Ctx* ctx, fmoe_dtype t, const void* x, const void* wg, const void* scores,
              const int32_t* idx, const void* d_topk, int64_t n, int64_t d, int64_t e, int64_t k,
              void* d_wg, void* d_x, void* dz_ws, __nv_bfloat16* dz_bf16, float* part_ws) {
  if (n == 0) {
    const size_t bytes = (size_t)(d * e) * score_size(t);
    if (bytes) CK(cudaMemsetAsync(d_wg, 0, bytes, ctx->stream));
    return;
  }
  gate_dlogits(ctx, t, scores, idx, d_topk, n, e, k, dz_ws);
  if (t == FMOE_F64 || t == FMOE_F32) {
    auto run = [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      SimtParams<T> p;  // d_wg = x^T dz, sum over rows ascending (gate.cpp:62)
      p.M = d; p.N = e; p.K = n;
      p.A = (const T*)x; p.sa_m = 1; p.sa_k = d;
      p.B = (const T*)dz_ws; p.sb_k = e; p.sb_n = 1;
      p.C = (T*)d_wg; p.ldc = e;
      simt_gemm<T>(ctx, p, d);
      if (d_x) {  // d_x = dz Wg^T, sum over experts ascending (gate.cpp:63)
        SimtParams<T> q;
        q.M = n; q.N = d; q.K = e;
        q.A = (const T*)dz_ws; q.sa_m = e; q.sa_k = 1;
        q.B = (const T*)wg; q.sb_k = 1; q.sb_n = e;
        q.C = (T*)d_x; q.ldc = d;
        simt_gemm<T>(ctx, q, n);
      }
    };
    if (t == FMOE_F64) run((double*)nullptr); else run((float*)nullptr);
    return;
  }
  cast_f32_bf16<<<(unsigned)ceil_div(n * e, 256), 256, 0, ctx->stream>>>((const float*)dz_ws, dz_bf16, n * e);
  CK_LAUNCH(ctx);
  gate_dwg_bf16(ctx, x, dz_bf16, n, d, e, part_ws, (float*)d_wg);
  if (d_x) gate_dx_bf16(ctx, dz_bf16, wg, n, d, e, nullptr, nullptr, 0, d_x);
}

// ----------------------------------------------------------------- experts
static void set_arrival(tc::Params& p, const Arrival* a) {
  if (!a) return;
  p.arrive_flags = a->flags;
  p.arrive_epoch = a->epoch;
  p.arrive_rt = a->rt;
  p.arrive_W = a->W;
  p.arrive_C = a->C;
  p.mtile_order = a->mtile_order;
  p.grid_limit = a->grid_limit;
}

static void set_route(tc::Params& p, const RowRoute* r) {
  if (!r) return;
  p.route_out = r->out;
  p.route_start = r->start;
  p.route_rows = r->rows;
  p.route_dst = r->dst;
  p.route_world = r->world;
}

// Off by default: measured ~3x slower than scatter + tile loads on the
// tensor-bound fc1 / fc1 weight gradient (32 four-row gathers per 16 KiB stage
// cannot feed the MMA; profiles/r02q_gather_ab.log).  FMOE_TC_GATHER=1 enables.
bool gather_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("FMOE_TC_GATHER");
    return v && std::atoi(v) != 0;
  }();
  return on;
}

void experts_fwd(Ctx* ctx, fmoe_dtype t, const fmoe_plan& b, int64_t d, int64_t h,
                 const fmoe_expert_params& w, const void* xs, void* hidden, void* ys,
                 uint32_t* relu_bits, void* preact, const RowRoute* ys_route, const Arrival* arrive,
                 const F32Planes* planes, const RowGather* gather) {
  const int64_t E = b.n_experts;
  if (E == 0 || b.capacity == 0) return;
  if (t == FMOE_F32 && !ys_route && f32_tc_route(b, d, h)) {  // tensor cores, bf16x3 (f32x.cu)
    experts_fwd_f32tc(ctx, b, d, h, w, xs, hidden, ys, preact, planes);
    return;
  }
  if (t == FMOE_F64 || t == FMOE_F32) {
    if (ys_route) shape_error("experts_fwd: routed outputs are bf16-only");
    const auto cnt = host_counts(ctx, b);
    const int64_t max_m = cnt.empty() ? 0 : *std::max_element(cnt.begin(), cnt.end());
    if (max_m == 0) return;
    auto run = [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      SimtParams<T> p;  // hidden = relu(xs W1 + b1)   (expert.cpp:30-31)
      p.mode = SIMT_RAGGED_M; p.G = E; p.offsets = b.offsets; p.counts = b.counts;
      p.N = h; p.K = d;
      p.A = (const T*)xs; p.sa_m = d; p.sa_k = 1;
      p.B = (const T*)w.w1; p.sb_k = h; p.sb_n = 1; p.b_group_stride = d * h;
      p.C = (T*)(preact ? preact : hidden); p.ldc = h;
      p.bias = (const T*)w.b1; p.bias_group_stride = h; p.relu = preact ? 0 : 1;
      simt_gemm<T>(ctx, p, max_m);
      if (preact) relu_rows<T>(ctx, (const T*)preact, (T*)hidden, b.capacity * h);  // cache.preact kept
      SimtParams<T> q;  // ys = hidden W2 + b2       (expert.cpp:32)
      q.mode = SIMT_RAGGED_M; q.G = E; q.offsets = b.offsets; q.counts = b.counts;
      q.N = d; q.K = h;
      q.A = (const T*)hidden; q.sa_m = h; q.sa_k = 1;
      q.B = (const T*)w.w2; q.sb_k = d; q.sb_n = 1; q.b_group_stride = h * d;
      q.C = (T*)ys; q.ldc = d;
      q.bias = (const T*)w.b2; q.bias_group_stride = d;
      simt_gemm<T>(ctx, q, max_m);
    };
    if (t == FMOE_F64) run((double*)nullptr); else run((float*)nullptr);
    return;
  }
  require_bf16_dims(d, h);
  if (b.align % 128 != 0 || !b.tile_expert) shape_error("bf16 experts need a 128-row aligned plan");
  const int cg = pair_mode(b);  // 256-aligned blocks -> CTA-pair tiles
  const int64_t cap = b.capacity;
  const int64_t max_tiles = cap / (128 * cg);
  {  // fc1: A = xs [cap, d] K-major (or its rows gathered from x); B = W1 [E*d, h] MN-major
    const CUtensorMap ta = gather ? tc::make_tmap(gather->x, d, gather->n_b, d * 2, 64, 1)
                                  : tc::make_tmap(xs, d, cap, d * 2, 64, 128);
    const CUtensorMap tb = tc::make_tmap(w.w1, h, E * d, h * 2, 64, 64);
    tc::Params p{};
    if (gather) {
      p.gather_rows = gather->rows;
      p.gather_oob = (int)gather->n_b;
    }
    p.mode = tc::RAGGED_M; p.M = (int)cap; p.N = (int)h; p.K = (int)d;
    p.tile_group = b.tile_expert; p.n_mtiles = b.n_tiles; p.b_group_rows = (int)d;
    p.epi = tc::EPI_BF16; p.C = hidden; p.ldc = h;
    p.bias = (const float*)w.b1; p.bias_group_stride = h; p.relu = 1;
    p.relu_bits_out = relu_bits;
    set_arrival(p, arrive);  // EP overlap: tiles wait for their rows, arrival order
    p.probe = ctx_probe_slot(ctx);
    tc::launch(ctx, 256, false, true, ta, tb, p, max_tiles * ceil_div(h, 256), cg);
    ctx_mark(ctx, MARK_FC1);
  }
  {  // fc2: A = hidden [cap, h] K-major; B = W2 [E*h, d] MN-major
    const CUtensorMap ta = tc::make_tmap(hidden, h, cap, h * 2, 64, 128);
    const CUtensorMap tb = tc::make_tmap(w.w2, d, E * h, d * 2, 64, 64);
    tc::Params p{};
    p.mode = tc::RAGGED_M; p.M = (int)cap; p.N = (int)d; p.K = (int)h;
    p.tile_group = b.tile_expert; p.n_mtiles = b.n_tiles; p.b_group_rows = (int)h;
    p.epi = tc::EPI_BF16; p.C = ys; p.ldc = d;
    p.bias = (const float*)w.b2; p.bias_group_stride = d; p.relu = 0;
    set_route(p, ys_route);
    p.probe = ctx_probe_slot(ctx);
    tc::launch(ctx, 256, false, true, ta, tb, p, max_tiles * ceil_div(d, 256), cg);
    ctx_mark(ctx, MARK_FC2);
  }
}

void experts_bwd(Ctx* ctx, fmoe_dtype t, const fmoe_plan& b, int64_t d, int64_t h,
                 const fmoe_expert_params& w, const void* xs, const void* hidden, const void* d_ys,
                 void* d_xs, const fmoe_expert_grads& g, void* d_pre, float* part_ws,
                 const uint32_t* relu_bits, const void* mask, int phase, const RowRoute* dxs_route,
                 const Arrival* arrive, const F32Planes* planes, const RowGather* gather) {
  const int64_t E = b.n_experts;
  if (E == 0) return;
  if (t == FMOE_F32 && phase == EXPERTS_BWD_ALL && !dxs_route && part_ws && f32_tc_route(b, d, h)) {
    // tensor cores, bf16x3 (f32x.cu); group order after the bias partials
    int* order = reinterpret_cast<int*>(part_ws + (b.capacity / 128 + 1) * (d + h));
    experts_bwd_f32tc(ctx, b, d, h, w, xs, hidden, d_ys, d_xs, g, d_pre, mask, order, planes);
    return;
  }
  if (t == FMOE_F64 || t == FMOE_F32) {
    if (phase != EXPERTS_BWD_ALL || dxs_route) shape_error("experts_bwd: phased / routed backward is bf16-only");
    const auto cnt = host_counts(ctx, b);
    const int64_t max_m = cnt.empty() ? 0 : *std::max_element(cnt.begin(), cnt.end());
    auto run = [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      {  // d_w2 = hidden^T d_y (expert.cpp:42)
        SimtParams<T> p;
        p.mode = SIMT_RAGGED_K; p.G = E; p.offsets = b.offsets; p.counts = b.counts;
        p.M = h; p.N = d;
        p.A = (const T*)hidden; p.sa_m = 1; p.sa_k = h;
        p.B = (const T*)d_ys; p.sb_k = d; p.sb_n = 1;
        p.C = (T*)g.d_w2; p.ldc = d; p.c_group_stride = h * d;
        simt_gemm<T>(ctx, p, h);
      }
      block_colsum(ctx, t, d_ys, d, b.offsets, b.counts, E, g.d_b2);  // expert.cpp:43-45
      if (max_m > 0) {  // d_pre = relu_backward(d_y W2^T, preact) (expert.cpp:47-48)
        SimtParams<T> p;
        p.mode = SIMT_RAGGED_M; p.G = E; p.offsets = b.offsets; p.counts = b.counts;
        p.N = h; p.K = d;
        p.A = (const T*)d_ys; p.sa_m = d; p.sa_k = 1;
        p.B = (const T*)w.w2; p.sb_k = 1; p.sb_n = d; p.b_group_stride = h * d;
        p.C = (T*)d_pre; p.ldc = h;
        p.mask = (const T*)(mask ? mask : hidden); p.ldm = h;
        simt_gemm<T>(ctx, p, max_m);
      }
      {  // d_w1 = x^T d_pre (expert.cpp:50)
        SimtParams<T> p;
        p.mode = SIMT_RAGGED_K; p.G = E; p.offsets = b.offsets; p.counts = b.counts;
        p.M = d; p.N = h;
        p.A = (const T*)xs; p.sa_m = 1; p.sa_k = d;
        p.B = (const T*)d_pre; p.sb_k = h; p.sb_n = 1;
        p.C = (T*)g.d_w1; p.ldc = h; p.c_group_stride = d * h;
        simt_gemm<T>(ctx, p, d);
      }
      block_colsum(ctx, t, d_pre, h, b.offsets, b.counts, E, g.d_b1);  // expert.cpp:51-53
      if (max_m > 0) {  // d_x = d_pre W1^T (expert.cpp:55)
        SimtParams<T> p;
        p.mode = SIMT_RAGGED_M; p.G = E; p.offsets = b.offsets; p.counts = b.counts;
        p.N = d; p.K = h;
        p.A = (const T*)d_pre; p.sa_m = h; p.sa_k = 1;
        p.B = (const T*)w.w1; p.sb_k = 1; p.sb_n = h; p.b_group_stride = d * h;
        p.C = (T*)d_xs; p.ldc = d;
        simt_gemm<T>(ctx, p, max_m);
      }
    };
    if (t == FMOE_F64) run((double*)nullptr); else run((float*)nullptr);
    return;
  }
  require_bf16_dims(d, h);
  if (b.align % 128 != 0 || !b.tile_expert) shape_error("bf16 experts need a 128-row aligned plan");
  const int cg = pair_mode(b);
  const int64_t cap = b.capacity;
  const int64_t max_tiles = cap / (128 * cg);  // (pair) row tiles
  const bool do_dgrad = phase != EXPERTS_BWD_WGRAD, do_wgrad = phase != EXPERTS_BWD_DGRAD;
  if (do_dgrad) {  // dgrad fc2: d_pre = (d_ys W2^T) * (hidden > 0); B(k=c, n=j) = W2[e][j][c] -> K-major [E*h, d]
    const CUtensorMap ta = tc::make_tmap(d_ys, d, cap, d * 2, 64, 128);
    const CUtensorMap tb = tc::make_tmap(w.w2, d, E * h, d * 2, 64, 256 / cg);
    tc::Params p{};
    p.mode = tc::RAGGED_M; p.M = (int)cap; p.N = (int)h; p.K = (int)d;
    p.tile_group = b.tile_expert; p.n_mtiles = b.n_tiles; p.b_group_rows = (int)h;
    p.epi = tc::EPI_MASK_BF16; p.C = d_pre; p.ldc = h; p.mask = (const __nv_bfloat16*)hidden; p.ldm = h;
    p.colsum_part = part_ws;  // d_b1 = colsum(d_pre) fused into the epilogue (expert.cpp:51-53)
    p.relu_bits = relu_bits;  // 1 bit per activation instead of re-reading hidden
    set_arrival(p, arrive);   // EP overlap: tiles wait for their d_ys rows, arrival order
    p.probe = ctx_probe_slot(ctx);
    tc::launch(ctx, 256, false, false, ta, tb, p, max_tiles * ceil_div(h, 256), cg);
    ctx_mark(ctx, MARK_DGRAD2);
  }
  // weight-gradient tiles heaviest expert first (skewed routing)
  int* group_order = nullptr;
  if (do_wgrad) {
    group_order = reinterpret_cast<int*>(part_ws + (cap / 128 + 1) * (d + h));
    order_groups_desc(ctx, b.offsets, E, group_order);
  }
  if (do_wgrad) {  // wgrad fc2: d_w2[e] = hidden_e^T d_ys_e  (M = h, N = d, K = rows of e)
    const CUtensorMap ta = tc::make_tmap(hidden, h, cap, h * 2, 64, 64);
    const CUtensorMap tb = tc::make_tmap(d_ys, d, cap, d * 2, 64, 64);
    tc::Params p{};
    p.mode = tc::RAGGED_K; p.M = (int)h; p.N = (int)d; p.n_groups = (int)E; p.k_offsets = b.offsets;
    p.group_order = group_order;
    p.epi = tc::EPI_F32; p.C = g.d_w2; p.ldc = d; p.c_group_stride = h * d;
    p.probe = ctx_probe_slot(ctx);
    tc::launch(ctx, 256, true, true, ta, tb, p, E * ceil_div(h, 128 * cg) * ceil_div(d, 256), cg);
    ctx_mark(ctx, MARK_WGRAD2);
  }
  // d_b2 = colsum(d_ys) per expert (expert.cpp:43-45): tile partials + ordered reduce
  const int64_t t128 = cap / 128;  // 128-row tiles (bias partials)
  float* part_b2 = part_ws + t128 * h;
  if (do_wgrad) {
    tile_colsum(ctx, (const __nv_bfloat16*)d_ys, d, b.n_tiles, t128, part_b2);
    // d_b1's partials (dgrad-fc2 epilogue) are complete here too: one reduce launch for both
    reduce_tile_partials(ctx, part_b2, d, b.offsets, E, (float*)g.d_b2, part_ws, h, (float*)g.d_b1);
    ctx_mark(ctx, MARK_DB2);
  }
  if (do_dgrad) {  // dgrad fc1: d_xs = d_pre W1^T; B(k=j, n=c) = W1[e][c][j] -> K-major [E*d, h]
    const CUtensorMap ta = tc::make_tmap(d_pre, h, cap, h * 2, 64, 128);
    const CUtensorMap tb = tc::make_tmap(w.w1, h, E * d, h * 2, 64, 256 / cg);
    tc::Params p{};
    p.mode = tc::RAGGED_M; p.M = (int)cap; p.N = (int)d; p.K = (int)h;
    p.tile_group = b.tile_expert; p.n_mtiles = b.n_tiles; p.b_group_rows = (int)d;
    p.epi = tc::EPI_BF16; p.C = d_xs; p.ldc = d;
    set_route(p, dxs_route);
    p.probe = ctx_probe_slot(ctx);
    tc::launch(ctx, 256, false, false, ta, tb, p, max_tiles * ceil_div(d, 256), cg);
    ctx_mark(ctx, MARK_DGRAD1);
  }
  if (do_wgrad) {  // wgrad fc1: d_w1[e] = xs_e^T d_pre_e  (M = d, N = h; xs rows gathered from x when asked)
    const CUtensorMap ta = gather ? tc::make_tmap(gather->x, d, gather->n_b, d * 2, 64, 1)
                                  : tc::make_tmap(xs, d, cap, d * 2, 64, 64);
    const CUtensorMap tb = tc::make_tmap(d_pre, h, cap, h * 2, 64, 64);
    tc::Params p{};
    if (gather) {
      p.gather_rows = gather->rows;
      p.gather_oob = (int)gather->n_b;
    }
    p.mode = tc::RAGGED_K; p.M = (int)d; p.N = (int)h; p.n_groups = (int)E; p.k_offsets = b.offsets;
    p.group_order = group_order;
    p.epi = tc::EPI_F32; p.C = g.d_w1; p.ldc = h; p.c_group_stride = d * h;
    p.probe = ctx_probe_slot(ctx);
    tc::launch(ctx, 256, true, true, ta, tb, p, E * ceil_div(d, 128 * cg) * ceil_div(h, 256), cg);
    ctx_mark(ctx, MARK_WGRAD1);
  }
  // no MARK_DB1 on this path: d_b1 was reduced with d_b2 above, and a mark
  // right behind MARK_WGRAD1 would only add an event record (~3 us) to the step
}

int64_t experts_bwd_part_floats(const fmoe_plan& b, int64_t d, int64_t h) {
  // bias-gradient tile partials, then the weight-gradient group order (ints)
  return (b.capacity / 128 + 1) * (d + h) + b.n_experts + 64;
}

}  // namespace fmoe_b200
