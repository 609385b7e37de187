// gate.cu -- softmax + top-k selection and the softmax-Jacobian backward of
// the gate (gate.cpp:23-65) for the SIMT dtypes, plus small reductions.
// The bf16 product path fuses softmax/top-k into the tcgen05 gate GEMM's
// epilogue (tc_gemm.cu epi_gate) and the Jacobian into gather_combine_bwd.
#include <type_traits>

#include "common.cuh"
#include "glibc_exp.cuh"
#include "plan.cuh"

namespace fmoe_b200 {
namespace {

// One thread per token row.  softmax_rows (matrix.cpp:155-170): running max,
// exp(l - max) summed sequentially in expert order, then a division;
// topk_rows (matrix.cpp:172-189): k passes, each taking the largest element
// strictly below the previous pick in (value desc, index asc) order -- the
// stable-sort order of the reference without a scratch array.
template <typename A>
__global__ void softmax_topk_kernel(const A* __restrict__ logits, int64_t n, int e, int k,
                                    A* __restrict__ scores, int32_t* __restrict__ idx,
                                    A* __restrict__ vals, bool scores_ready) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  A* s = scores + i * e;
  if (!scores_ready) {
    const A* l = logits + i * e;
    A mx = -INFINITY;
    for (int c = 0; c < e; ++c) mx = l[c] > mx ? l[c] : mx;
    A sum = A(0);
    for (int c = 0; c < e; ++c) {
      // fp64 parity: glibc's exp, bit for bit (glibc_exp.cuh); fp32: CUDA expf
      A v;
      if constexpr (std::is_same<A, double>::value)
        v = glibc_exp(l[c] - mx);
      else
        v = exp(l[c] - mx);
      s[c] = v;
      sum += v;
    }
    for (int c = 0; c < e; ++c) s[c] = s[c] / sum;
  }
  A pv = A(0);
  int pi = -1;
  for (int j = 0; j < k; ++j) {
    int best = -1;
    A bv = A(0);
    for (int c = 0; c < e; ++c) {
      const A v = s[c];
      const bool below = (pi < 0) || (v < pv) || (v == pv && c > pi);
      if (below && (best < 0 || v > bv)) {
        best = c;
        bv = v;
      }
    }
    if (best < 0) {
      // only NaN is left (a NaN logit makes the whole row NaN): the
      // reference's stable sort keeps column order, so take the lowest column
      // not chosen yet -- indices always stay in [0, e)
      for (int c = 0; c < e && best < 0; ++c) {
        bool used = false;
        for (int q = 0; q < j; ++q) used |= idx[i * k + q] == c;
        if (!used) {
          best = c;
          bv = s[c];
        }
      }
    }
    idx[i * k + j] = best;
    vals[i * k + j] = bv;
    pv = bv;
    pi = best;
  }
}

// gate_backward's d_logits (gate.cpp:44-59): ds = scatter of d_topk into the
// selected columns; dot = <ds, s> in the reference build's order (paired
// products unfused, a final odd term fused); dz = s * (ds - dot).
template <typename A>
__global__ void dlogits_kernel(const A* __restrict__ scores, const int32_t* __restrict__ idx,
                               const A* __restrict__ d_topk, int64_t n, int e, int k,
                               A* __restrict__ dz) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const A* s = scores + i * e;
  A* o = dz + i * e;
  for (int c = 0; c < e; ++c) o[c] = A(0);
  for (int j = 0; j < k; ++j) o[idx[i * k + j]] += d_topk[i * k + j];
  A dot = A(0);
  const int paired = e & ~1;
  for (int c = 0; c < paired; ++c) {
    A prod;
    if constexpr (std::is_same<A, double>::value)
      prod = __dmul_rn(o[c], s[c]);
    else
      prod = __fmul_rn(o[c], s[c]);
    dot += prod;
  }
  if (e & 1) dot = fma(o[paired], s[paired], dot);
  for (int c = 0; c < e; ++c) o[c] = s[c] * (o[c] - dot);
}

__global__ void reduce_splits_kernel(const float* __restrict__ part, int64_t n_splits, int64_t n,
                                     float* __restrict__ out) {
  pdl_wait();  // launched right behind the split-K GEMM
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = 0.f;
  for (int64_t s = 0; s < n_splits; ++s) acc += part[s * n + i];
  out[i] = acc;
}

}  // namespace

void gate_softmax_topk(Ctx* ctx, fmoe_dtype t, const void* logits, int64_t n, int64_t e, int64_t k,
                       void* scores, int32_t* idx, void* vals, bool scores_ready) {
  if (n == 0) return;
  const unsigned grid = (unsigned)ceil_div(n, 128);
  if (t == FMOE_F64)
    softmax_topk_kernel<double><<<grid, 128, 0, ctx->stream>>>(
        (const double*)logits, n, (int)e, (int)k, (double*)scores, idx, (double*)vals, scores_ready);
  else
    softmax_topk_kernel<float><<<grid, 128, 0, ctx->stream>>>(
        (const float*)logits, n, (int)e, (int)k, (float*)scores, idx, (float*)vals, scores_ready);
  CK_LAUNCH(ctx);
}

void gate_dlogits(Ctx* ctx, fmoe_dtype t, const void* scores, const int32_t* idx, const void* d_topk,
                  int64_t n, int64_t e, int64_t k, void* dz) {
  if (n == 0) return;
  const unsigned grid = (unsigned)ceil_div(n, 128);
  if (t == FMOE_F64)
    dlogits_kernel<double><<<grid, 128, 0, ctx->stream>>>((const double*)scores, idx, (const double*)d_topk,
                                                         n, (int)e, (int)k, (double*)dz);
  else
    dlogits_kernel<float><<<grid, 128, 0, ctx->stream>>>((const float*)scores, idx, (const float*)d_topk,
                                                        n, (int)e, (int)k, (float*)dz);
  CK_LAUNCH(ctx);
}

void reduce_splits(Ctx* ctx, const float* part, int64_t n_splits, int64_t n, float* out) {
  if (n == 0) return;
  CK(launch_pdl(reduce_splits_kernel, dim3((unsigned)ceil_div(n, 256)), dim3(256), 0, ctx->stream, part, n_splits, n,
                out));
  CK_LAUNCH(ctx);
}

}  // namespace fmoe_b200
