// gemm_simt.cuh -- grouped SIMT GEMM (parity / fp32 modes), see gemm_simt.cu.
#pragma once

#include "common.cuh"

namespace fmoe_b200 {

enum SimtMode : int { SIMT_PLAIN = 0, SIMT_RAGGED_M = 1, SIMT_RAGGED_K = 2 };

// C(m, n) = epi( sum_k A(m, k) * B(k, n) ),  A(m,k) = A[m*sa_m + k*sa_k],
// B(k,n) = B[k*sb_k + n*sb_n].
//   RAGGED_M: group g owns rows [offsets[g], offsets[g]+counts[g]) of A and C;
//             B and bias advance by b_group_stride / bias_group_stride.
//   RAGGED_K: group g contracts over rows [offsets[g], +counts[g]) of A and B
//             (weight gradients); C advances by c_group_stride.
template <typename T>
struct SimtParams {
  int mode = SIMT_PLAIN;
  int64_t M = 0, N = 0, K = 0;
  int64_t G = 1;
  const int32_t* offsets = nullptr;
  const int32_t* counts = nullptr;
  const T* A = nullptr;
  int64_t sa_m = 0, sa_k = 0;
  const T* B = nullptr;
  int64_t sb_k = 0, sb_n = 0, b_group_stride = 0;
  T* C = nullptr;
  int64_t ldc = 0, c_group_stride = 0;
  const T* bias = nullptr;
  int64_t bias_group_stride = 0;
  int relu = 0;
  const T* mask = nullptr;  // strict > 0 mask, same row space as C
  int64_t ldm = 0;
};

// max_m: upper bound on rows per group (RAGGED_M) or M (other modes).
template <typename T>
void simt_gemm(Ctx* ctx, const SimtParams<T>& p, int64_t max_m);

}  // namespace fmoe_b200
