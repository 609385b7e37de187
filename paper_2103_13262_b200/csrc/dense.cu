// dense.cu -- C-ABI of the dense matrix primitives the gate and the experts are
// built from (matrix.hpp:77-100) and of the expert operators with the full
// ForwardCache (expert.hpp:31-35).  These exist so the C++ drop-in
// (include/fmoe/*.hpp, libfmoe_dropin.so) can expose matmul / softmax_rows /
// topk_rows with the same bits gate_forward produces: they run the very
// kernels the FMOE_F64 / FMOE_F32 gate uses (gemm_simt.cu, gate.cu).
#include <string>
#include <type_traits>

#include "gemm_simt.cuh"
#include "ops.cuh"

namespace fmoe_b200 {
void gate_softmax_topk(Ctx* ctx, fmoe_dtype t, const void* logits, int64_t n, int64_t e, int64_t k,
                       void* scores, int32_t* idx, void* vals, bool scores_ready);
}

using namespace fmoe_b200;

#define FMOE_GUARD(...)               \
  try {                               \
    __VA_ARGS__;                      \
    return FMOE_OK;                   \
  } catch (const std::exception& e) { \
    return guard_status(e);           \
  } catch (...) {                     \
    g_last_error = "unknown error";   \
    return FMOE_ERR_CUDA;             \
  }

namespace {
template <typename S, typename D>
__global__ void cast_kernel(const S* __restrict__ src, D* __restrict__ dst, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (std::is_same<D, __nv_bfloat16>::value && std::is_same<S, double>::value)
      dst[i] = __double2bfloat16(src[i]);  // one rounding
    else if constexpr (std::is_same<D, __nv_bfloat16>::value)
      dst[i] = __float2bfloat16_rn((float)to_f(src[i]));
    else if constexpr (std::is_same<S, __nv_bfloat16>::value)
      dst[i] = (D)__bfloat162float(src[i]);
    else
      dst[i] = (D)src[i];  // f64 -> f32 rounds to nearest even, f32 -> f64 exact
  }
}

Ctx* CD(fmoe_ctx* c) {
  if (!c) shape_error("null context");
  return reinterpret_cast<Ctx*>(c);
}
void simt_only(fmoe_dtype t, const char* who) {
  if (t != FMOE_F64 && t != FMOE_F32) shape_error(std::string(who) + ": dtype must be FMOE_F64 or FMOE_F32");
}
}  // namespace

extern "C" {

int fmoe_matmul(fmoe_ctx* ctx, fmoe_dtype dtype, const void* a, const void* b, int64_t m, int64_t p,
                int64_t n, void* c) {
  FMOE_GUARD({
    Ctx* x = CD(ctx);
    simt_only(dtype, "matmul");
    if (m < 0 || p < 0 || n < 0) shape_error("matmul: negative shape");
    if (m == 0 || n == 0) return FMOE_OK;
    auto run = [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      SimtParams<T> q;  // C = A B, one fma chain per element, k ascending from +0.0
      q.M = m; q.N = n; q.K = p;
      q.A = (const T*)a; q.sa_m = p; q.sa_k = 1;
      q.B = (const T*)b; q.sb_k = n; q.sb_n = 1;
      q.C = (T*)c; q.ldc = n;
      simt_gemm<T>(x, q, m);
    };
    if (dtype == FMOE_F64) run((double*)nullptr); else run((float*)nullptr);
  })
}

int fmoe_softmax_rows(fmoe_ctx* ctx, fmoe_dtype dtype, const void* a, int64_t rows, int64_t cols, void* out) {
  FMOE_GUARD({
    Ctx* x = CD(ctx);
    simt_only(dtype, "softmax_rows");
    if (rows < 0 || cols < 0) shape_error("softmax_rows: negative shape");
    if (rows == 0 || cols == 0) return FMOE_OK;
    gate_softmax_topk(x, dtype, a, rows, cols, 0, out, nullptr, nullptr, false);
  })
}

int fmoe_topk_rows(fmoe_ctx* ctx, fmoe_dtype dtype, const void* a, int64_t rows, int64_t cols, int64_t k,
                   int32_t* idx, void* vals) {
  FMOE_GUARD({
    Ctx* x = CD(ctx);
    simt_only(dtype, "topk_rows");
    if (k < 1 || k > cols)
      shape_error("topk_rows: k out of range [1, " + std::to_string(cols) + "]");
    if (rows == 0) return FMOE_OK;
    gate_softmax_topk(x, dtype, nullptr, rows, cols, k, const_cast<void*>(a), idx, vals, true);
  })
}

int fmoe_experts_fwd_cached(fmoe_ctx* ctx, fmoe_dtype dtype, const fmoe_plan* blocks, int64_t d_m, int64_t d_h,
                            fmoe_expert_params params, const void* xs, void* preact, void* hidden, void* ys) {
  FMOE_GUARD({
    Ctx* x = CD(ctx);
    simt_only(dtype, "experts_fwd_cached");
    if (!blocks || !blocks->counts || !blocks->offsets) shape_error("null block plan");
    if (!preact || !hidden) shape_error("experts_fwd_cached: preact and hidden are required");
    experts_fwd(x, dtype, *blocks, d_m, d_h, params, xs, hidden, ys, nullptr, preact);
  })
}

int fmoe_experts_bwd_cached(fmoe_ctx* ctx, fmoe_dtype dtype, const fmoe_plan* blocks, int64_t d_m, int64_t d_h,
                            fmoe_expert_params params, const void* xs, const void* preact, const void* hidden,
                            const void* d_ys, void* d_xs, fmoe_expert_grads grads) {
  FMOE_GUARD({
    Ctx* x = CD(ctx);
    simt_only(dtype, "experts_bwd_cached");
    if (!blocks || !blocks->counts || !blocks->offsets) shape_error("null block plan");
    if (!preact || !hidden) shape_error("experts_bwd_cached: preact and hidden are required");
    const size_t pre_bytes = ((size_t)(blocks->capacity * d_h) * dtype_size(dtype) + 255) / 256 * 256;
    uint8_t* ws = (uint8_t*)ctx_workspace(x, pre_bytes + 256);
    experts_bwd(x, dtype, *blocks, d_m, d_h, params, xs, hidden, d_ys, d_xs, grads, ws, nullptr, nullptr,
                preact);
  })
}

int fmoe_cast(fmoe_ctx* ctx, fmoe_dtype from, const void* src, fmoe_dtype to, void* dst, int64_t n) {
  FMOE_GUARD({
    Ctx* x = CD(ctx);
    if (n < 0) shape_error("cast: negative size");
    if (n == 0) return FMOE_OK;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), 148 * 16);
    dispatch_dtype(from, [&](auto* ts) {
      using S = std::remove_pointer_t<decltype(ts)>;
      dispatch_dtype(to, [&](auto* td) {
        using D = std::remove_pointer_t<decltype(td)>;
        cast_kernel<S, D><<<grid, 256, 0, x->stream>>>((const S*)src, (D*)dst, n);
      });
    });
    CK_LAUNCH(x);
  })
}

}  // extern "C"
