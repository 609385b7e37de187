// gemm_simt.cu -- grouped SIMT GEMM for the FMOE_F64 parity mode and FMOE_F32.
//
// Every output element is one fused multiply-add chain over k in ascending
// order starting from +0.0 -- the accumulation order the reference's matmul
// guarantees (matrix.hpp:77-80, matrix.cpp:56-88) -- so FMOE_F64 results are
// bit-identical to the reference.  Bias is a separate rounded add after the
// full dot product (add_bias_rows, matrix.cpp:128-138), relu keeps -0.0
// (matrix.cpp:140-145) and the relu-backward mask is strict x > 0
// (matrix.cpp:147-153).  Tiles: 64x64 outputs per 256-thread CTA, 4x4 per
// thread, K staged through shared memory in steps of 16.
#include <type_traits>

#include "common.cuh"
#include "gemm_simt.cuh"

namespace fmoe_b200 {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

template <typename T>
__global__ void __launch_bounds__(256) simt_gemm_kernel(SimtParams<T> p) {
  __shared__ T sa[TK][TM + 1];
  __shared__ T sb[TK][TN + 1];
  const int g = blockIdx.z;
  int64_t M = p.M, K = p.K, row0 = 0, kofs = 0;
  const T* B = p.B;
  T* Cp = p.C;
  const T* bias = p.bias;
  if (p.mode == SIMT_RAGGED_M) {
    row0 = p.offsets[g];
    M = p.counts[g];
    B += (int64_t)g * p.b_group_stride;
    if (bias) bias += (int64_t)g * p.bias_group_stride;
  } else if (p.mode == SIMT_RAGGED_K) {
    kofs = p.offsets[g];
    K = p.counts[g];
    Cp += (int64_t)g * p.c_group_stride;
  }
  const int64_t m_base = (int64_t)blockIdx.y * TM;
  const int64_t n_base = (int64_t)blockIdx.x * TN;
  if (m_base >= M) return;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
  for (int64_t k0 = 0; k0 < K; k0 += TK) {
    for (int t = threadIdx.x; t < TK * TM; t += 256) {
      const int kk = t / TM, mm = t % TM;
      const int64_t m = m_base + mm, k = k0 + kk;
      sa[kk][mm] = (m < M && k < K) ? p.A[(row0 + m) * p.sa_m + (kofs + k) * p.sa_k] : T(0);
    }
    for (int t = threadIdx.x; t < TK * TN; t += 256) {
      const int kk = t / TN, nn = t % TN;
      const int64_t n = n_base + nn, k = k0 + kk;
      sb[kk][nn] = (n < p.N && k < K) ? B[(kofs + k) * p.sb_k + n * p.sb_n] : T(0);
    }
    __syncthreads();
    const int kmax = (int)((K - k0) < TK ? (K - k0) : TK);
    for (int kk = 0; kk < kmax; ++kk) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(sa[kk][ty * 4 + a], sb[kk][tx * 4 + b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t m = m_base + ty * 4 + a;
    if (m >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t n = n_base + tx * 4 + b;
      if (n >= p.N) continue;
      T v = acc[a][b];
      if (bias) v = v + bias[n];
      if (p.relu) v = v < T(0) ? T(0) : v;
      if (p.mask) v = p.mask[(row0 + m) * p.ldm + n] > T(0) ? v : T(0);
      Cp[(row0 + m) * p.ldc + n] = v;
    }
  }
}

}  // namespace

template <typename T>
void simt_gemm(Ctx* ctx, const SimtParams<T>& p, int64_t max_m) {
  if (p.N <= 0 || p.G <= 0) return;
  int64_t m_tiles = ceil_div(max_m, TM);
  if (m_tiles < 1) m_tiles = 1;
  dim3 grid((unsigned)ceil_div(p.N, TN), (unsigned)m_tiles, (unsigned)p.G);
  simt_gemm_kernel<T><<<grid, 256, 0, ctx->stream>>>(p);
  CK_LAUNCH(ctx);
}

template void simt_gemm<double>(Ctx*, const SimtParams<double>&, int64_t);
template void simt_gemm<float>(Ctx*, const SimtParams<float>&, int64_t);

}  // namespace fmoe_b200
