// permute.cu -- local_scatter / local_gather (+ weighted combine) and their
// backward passes (dispatch.cpp:49-126), HBM-bound row permutations.
//
// One warp per token row; rows move as 128-bit vectors with several loads in
// flight per lane.  scatter reads each token once and writes its k copies
// (algorithmic bytes s*d*(N + N*k)); gather_combine reads the k expert rows
// and writes the token once.  Accumulation follows the reference's slot
// order (fma chain for the combine, plain adds for scatter_backward) in the
// accumulate type (fp64 for FMOE_F64, fp32 otherwise), so FMOE_F64 results
// are bit-identical to dispatch.cpp.
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "peer.cuh"
#include "plan.cuh"

namespace fmoe_b200 {

namespace {

template <typename T>
using AccOf = typename std::conditional<std::is_same<T, double>::value, double, float>::type;

template <typename T>
struct Vec {
  static constexpr int N = 16 / sizeof(T);
};

template <typename T, typename A>
__device__ __forceinline__ void unpack16(const uint4& u, A (&o)[Vec<T>::N]) {
  const T* p = reinterpret_cast<const T*>(&u);
#pragma unroll
  for (int i = 0; i < Vec<T>::N; ++i) o[i] = (A)to_f(p[i]);
}
template <typename T, typename A>
__device__ __forceinline__ uint4 pack16(const A (&o)[Vec<T>::N]) {
  uint4 u;
  T* p = reinterpret_cast<T*>(&u);
#pragma unroll
  for (int i = 0; i < Vec<T>::N; ++i) {
    if constexpr (std::is_same<T, double>::value)
      p[i] = o[i];
    else
      p[i] = from_f<T>((float)o[i]);
  }
  return u;
}

__device__ __forceinline__ int64_t warp_id_global() {
  return ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
}

// Pad rows of an aligned plan: warp slot `w` -> (expert, r < align); -1 for
// no pad row (including the grid's rounding warps past the last expert).
__device__ __forceinline__ int64_t pad_row(const fmoe_plan& p, int64_t w) {
  if (w >= p.n_experts * p.align) return -1;
  const int e = (int)(w / p.align), r = (int)(w % p.align);
  const int64_t row = (int64_t)p.offsets[e] + p.counts[e] + r;
  return row < p.offsets[e + 1] ? row : -1;
}

// ------------------------------------------------------------------ scatter
// Pure byte copy: element type only sets the row size.  With a route (expert
// parallelism over peer memory) slot (i, j) is written straight into the
// receive buffer of its expert's rank: the local scatter and the global
// scatter (collectives.cpp:146-203) become one pass.
__global__ void scatter_kernel(const uint8_t* __restrict__ x, int64_t row_bytes, fmoe_plan p,
                               uint8_t* __restrict__ xs, ScatterRoute route) {
  pdl_wait();
  const int64_t w = warp_id_global();
  const int lane = threadIdx.x & 31;
  const int k = (int)p.k;
  if (w < p.n_b) {
    const uint8_t* src = x + w * row_bytes;
    auto dest = [&](int j) -> uint8_t* {
      const int64_t pos = __ldg(p.inverse_pos + w * k + j);
      if (!route.idx) return xs + pos * row_bytes;
      const int g = __ldg(route.idx + w * k + j);
      return reinterpret_cast<uint8_t*>(route.dst[__ldg(route.g_rank + g)]) + (pos + __ldg(route.g_delta + g)) * row_bytes;
    };
    uint8_t* dst[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) dst[j] = j < k ? dest(j) : nullptr;
    if ((row_bytes & 15) == 0) {
      const int64_t n16 = row_bytes >> 4;
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      for (int64_t c = lane; c < n16; c += 32 * 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c + u * 32 < n16) v[u] = __ldg(s4 + c + u * 32);
        for (int j = 0; j < k; ++j) {
          uint4* d4 = reinterpret_cast<uint4*>(j < 8 ? dst[j] : dest(j));
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (c + u * 32 < n16) d4[c + u * 32] = v[u];
        }
      }
    } else {
      for (int64_t c = lane; c < row_bytes; c += 32) {
        const uint8_t v = src[c];
        for (int j = 0; j < k; ++j) (j < 8 ? dst[j] : dest(j))[c] = v;
      }
    }
    return;
  }
  if (p.align <= 1) return;
  const int64_t row = pad_row(p, w - p.n_b);
  if (row < 0) return;
  uint8_t* d = xs + row * row_bytes;
  if ((row_bytes & 15) == 0) {
    uint4* d4 = reinterpret_cast<uint4*>(d);
    for (int64_t c = lane; c < (row_bytes >> 4); c += 32) d4[c] = make_uint4(0, 0, 0, 0);
  } else {
    for (int64_t c = lane; c < row_bytes; c += 32) d[c] = 0;
  }
}

// ----------------------------------------------------------- gather_combine
template <typename T, typename S>
__global__ void gather_combine_kernel(const T* __restrict__ ys, int64_t d, fmoe_plan p,
                                      const S* __restrict__ w, T* __restrict__ y) {
  pdl_wait();
  using A = AccOf<T>;
  constexpr int V = Vec<T>::N;
  const int64_t i = warp_id_global();
  const int lane = threadIdx.x & 31;
  if (i >= p.n_b) return;
  const int k = (int)p.k;
  if ((d % V) == 0) {
    const int64_t nv = d / V;
    for (int64_t c = lane; c < nv; c += 32) {
      A acc[V];
#pragma unroll
      for (int u = 0; u < V; ++u) acc[u] = A(0);
      for (int j = 0; j < k; ++j) {
        const int64_t pos = __ldg(p.inverse_pos + i * k + j);
        const A wt = (A)__ldg(w + i * k + j);
        A yv[V];
        unpack16<T, A>(__ldg(reinterpret_cast<const uint4*>(ys + pos * d) + c), yv);
#pragma unroll
        for (int u = 0; u < V; ++u) acc[u] = fma(wt, yv[u], acc[u]);
      }
      reinterpret_cast<uint4*>(y + i * d)[c] = pack16<T, A>(acc);
    }
  } else {
    for (int64_t c = lane; c < d; c += 32) {
      A acc = A(0);
      for (int j = 0; j < k; ++j) {
        const int64_t pos = __ldg(p.inverse_pos + i * k + j);
        acc = fma((A)__ldg(w + i * k + j), (A)to_f(ys[pos * d + c]), acc);
      }
      if constexpr (std::is_same<T, double>::value)
        y[i * d + c] = acc;
      else
        y[i * d + c] = from_f<T>((float)acc);
    }
  }
}

// ---------------------------------------------------------- scatter_backward
// KM: slots held in registers by the fast path (k <= KM); the k <= 2 instance
// needs half the registers of KM = 4 (more warps per SM)
template <typename T, int KM = 4>
__global__ void scatter_bwd_kernel(const T* __restrict__ d_xs, int64_t d, fmoe_plan p,
                                   const T* __restrict__ addend, T* __restrict__ dx) {
  pdl_wait();  // launched right behind the gate d_x GEMM (scatter_bwd below)
  using A = AccOf<T>;
  constexpr int V = Vec<T>::N;
  const int64_t i = warp_id_global();
  const int lane = threadIdx.x & 31;
  if (i >= p.n_b) return;
  const int k = (int)p.k;
  if ((d % V) == 0 && k <= KM) {
    // every slot's rows (and the addend) in flight together; adds in slot
    // order then the addend, as below
    constexpr int U = 4;
    const int64_t nv = d / V;
    const T* src[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) src[j] = j < k ? d_xs + (int64_t)__ldg(p.inverse_pos + i * k + j) * d : d_xs;
    for (int64_t c0 = lane; c0 < nv; c0 += 32 * U) {
      uint4 raw[KM][U], ad[U];
#pragma unroll
      for (int j = 0; j < KM; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j < k && c0 + 32 * u < nv) raw[j][u] = __ldg(reinterpret_cast<const uint4*>(src[j]) + c0 + 32 * u);
      if (addend)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + 32 * u < nv) ad[u] = __ldg(reinterpret_cast<const uint4*>(addend + i * d) + c0 + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (c0 + 32 * u >= nv) continue;
        A acc[V];
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = A(0);
#pragma unroll
        for (int j = 0; j < KM; ++j) {
          if (j >= k) break;
          A g[V];
          unpack16<T, A>(raw[j][u], g);
#pragma unroll
          for (int e = 0; e < V; ++e) acc[e] += g[e];
        }
        if (addend) {
          A g[V];
          unpack16<T, A>(ad[u], g);
#pragma unroll
          for (int e = 0; e < V; ++e) acc[e] += g[e];
        }
        reinterpret_cast<uint4*>(dx + i * d)[c0 + 32 * u] = pack16<T, A>(acc);
      }
    }
    return;
  }
  if ((d % V) == 0) {
    const int64_t nv = d / V;
#pragma unroll 4
    for (int64_t c = lane; c < nv; c += 32) {
      A acc[V];
#pragma unroll
      for (int u = 0; u < V; ++u) acc[u] = A(0);
      for (int j = 0; j < k; ++j) {
        const int64_t pos = __ldg(p.inverse_pos + i * k + j);
        A g[V];
        unpack16<T, A>(__ldg(reinterpret_cast<const uint4*>(d_xs + pos * d) + c), g);
#pragma unroll
        for (int u = 0; u < V; ++u) acc[u] += g[u];
      }
      if (addend) {  // d_x += gate.d_x (moe_layer.cpp:140)
        A g[V];
        unpack16<T, A>(__ldg(reinterpret_cast<const uint4*>(addend + i * d) + c), g);
#pragma unroll
        for (int u = 0; u < V; ++u) acc[u] += g[u];
      }
      reinterpret_cast<uint4*>(dx + i * d)[c] = pack16<T, A>(acc);
    }
  } else {
    for (int64_t c = lane; c < d; c += 32) {
      A acc = A(0);
      for (int j = 0; j < k; ++j) acc += (A)to_f(d_xs[(int64_t)__ldg(p.inverse_pos + i * k + j) * d + c]);
      if (addend) acc += (A)to_f(addend[i * d + c]);
      if constexpr (std::is_same<T, double>::value)
        dx[i * d + c] = acc;
      else
        dx[i * d + c] = from_f<T>((float)acc);
    }
  }
}

// ---------------------------------------------------- gather_combine_backward
// In-order dot product as the reference build computes it (see
// oracle/fmoe_oracle.c dot_ref): paired products rounded and added in
// order, a final odd term fused.
template <typename A, typename T>
__device__ __forceinline__ A dot_ref_seq(const T* a, const T* b, int64_t n) {
  A dot = A(0);
  const int64_t paired = n & ~int64_t(1);
  for (int64_t c = 0; c < paired; ++c) {
    const A prod = __dmul_rn((A)to_f(a[c]), (A)to_f(b[c]));
    dot = __dadd_rn(dot, prod);
  }
  if (n & 1) dot = fma((A)to_f(a[paired]), (A)to_f(b[paired]), dot);
  return dot;
}

// 4 blocks (32 warps) per SM: <= 64 registers keeps more token rows in flight
// (A/B: gather_combine_bwd 156 -> 141 us at cfg2 against the unbounded 80-register build)
#ifndef FMOE_GCB_MINB
#define FMOE_GCB_MINB 4
#endif
template <typename T, typename S>
__global__ void __launch_bounds__(256, FMOE_GCB_MINB) gcb_kernel(const T* __restrict__ dy, const T* __restrict__ ys, int64_t d, fmoe_plan p,
                           const S* __restrict__ w, T* __restrict__ d_ys, S* __restrict__ d_w,
                           const float* __restrict__ scores, const int32_t* __restrict__ topk_idx,
                           __nv_bfloat16* __restrict__ dz, ScatterRoute route) {
  pdl_wait();
  using A = AccOf<T>;
  constexpr int V = Vec<T>::N;
  const int64_t i = warp_id_global();
  const int lane = threadIdx.x & 31;
  const int k = (int)p.k;
  if (i >= p.n_b) {
    if (p.align <= 1 || d_ys == nullptr) return;
    const int64_t row = pad_row(p, i - p.n_b);
    if (row < 0) return;
    if ((d % V) == 0) {
      uint4* d4 = reinterpret_cast<uint4*>(d_ys + row * d);
      for (int64_t c = lane; c < d / V; c += 32) d4[c] = make_uint4(0, 0, 0, 0);
    } else {
      for (int64_t c = lane; c < d; c += 32) d_ys[row * d + c] = T(0);
    }
    return;
  }
  const T* dyr = dy + i * d;
  // d_ys == NULL without a route: the rows are pushed by ep_push_kernel (the
  // overlapped exchange); only d_w and the gate Jacobian are produced here
  const bool write_dys = d_ys != nullptr || route.idx != nullptr;
  float dw_f[8];
  if constexpr (!std::is_same<T, double>::value) {
    if ((d % V) == 0 && k <= 2) {
      // fp32-accumulating fast path: the token's d_y slice is loaded once and
      // every slot's ys loads are in flight together (same per-lane order of
      // the dot products as the generic loop below, so the same bits)
      constexpr int U = 4;
      const int64_t nv = d / V;
      // gate Jacobian operands (E <= 64) fetched now, in flight with the rows
      const int E = (int)p.n_experts;
      const bool pre = dz != nullptr && E <= 64;
      float s_pre[2] = {0.f, 0.f};
      int ix_pre[2] = {0, 0};
      if (pre) {
        const float* s = scores + i * E;
        if (lane < E) s_pre[0] = __ldg(s + lane);
        if (lane + 32 < E) s_pre[1] = __ldg(s + lane + 32);
        for (int j = 0; j < k; ++j) ix_pre[j] = __ldg(topk_idx + i * k + j);
      }
      T* dr[2];
      const T* yr[2];
      A wt[2], part[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j >= k) {
          dr[j] = d_ys;
          yr[j] = ys;
          wt[j] = A(0);
          part[j] = A(0);
          continue;
        }
        const int64_t pos = __ldg(p.inverse_pos + i * k + j);
        wt[j] = (A)__ldg(w + i * k + j);
        dr[j] = d_ys + pos * d;
        if (route.idx) {
          const int g = __ldg(route.idx + i * k + j);
          dr[j] = reinterpret_cast<T*>(route.dst[__ldg(route.g_rank + g)]) + (pos + __ldg(route.g_delta + g)) * d;
        }
        yr[j] = ys + pos * d;
        part[j] = A(0);
      }
      for (int64_t c0 = lane; c0 < nv; c0 += 32 * U) {
        uint4 gv[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (c0 + 32 * u < nv) gv[u] = __ldg(reinterpret_cast<const uint4*>(dyr) + c0 + 32 * u);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j >= k) break;
          uint4 yv4[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (c0 + 32 * u < nv) yv4[u] = __ldg(reinterpret_cast<const uint4*>(yr[j]) + c0 + 32 * u);
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (c0 + 32 * u < nv) {
              A g[V], yv[V], o[V];
              unpack16<T, A>(gv[u], g);
              unpack16<T, A>(yv4[u], yv);
#pragma unroll
              for (int e = 0; e < V; ++e) {
                o[e] = wt[j] * g[e];
                part[j] = fma(g[e], yv[e], part[j]);
              }
              if (write_dys) reinterpret_cast<uint4*>(dr[j])[c0 + 32 * u] = pack16<T, A>(o);
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j >= k) break;
        A dot = part[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (lane == 0) d_w[i * k + j] = (S)dot;
        dw_f[j] = (float)dot;
      }
      if (pre) {  // the general tail below, from registers (same operations, same bits)
        float dot = 0.f;
        for (int j = 0; j < k; ++j) {
          const int ix = ix_pre[j];
          const float sx = __shfl_sync(0xffffffffu, (ix >> 5) ? s_pre[1] : s_pre[0], ix & 31);
          dot = fmaf(dw_f[j], sx, dot);
        }
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int e = lane + 32 * h2;
          if (e >= E) break;
          float dse = 0.f;
          for (int j = 0; j < k; ++j)
            if (ix_pre[j] == e) dse += dw_f[j];
          dz[i * E + e] = __float2bfloat16_rn(s_pre[h2] * (dse - dot));
        }
        return;
      }
      goto gate_jacobian;
    }
  }
  for (int j = 0; j < k; ++j) {
    const int64_t pos = __ldg(p.inverse_pos + i * k + j);
    const A wt = (A)__ldg(w + i * k + j);
    T* dr = d_ys + pos * d;
    if (route.idx) {  // d_ys rows go straight to the expert ranks (backward global_scatter)
      const int g = __ldg(route.idx + i * k + j);
      dr = reinterpret_cast<T*>(route.dst[__ldg(route.g_rank + g)]) + (pos + __ldg(route.g_delta + g)) * d;
    }
    const T* yr = ys + pos * d;
    A part = A(0);
    if ((d % V) == 0) {
      const int64_t nv = d / V;
      for (int64_t c = lane; c < nv; c += 32) {
        A g[V], yv[V], o[V];
        unpack16<T, A>(__ldg(reinterpret_cast<const uint4*>(dyr) + c), g);
        unpack16<T, A>(__ldg(reinterpret_cast<const uint4*>(yr) + c), yv);
#pragma unroll
        for (int u = 0; u < V; ++u) {
          if constexpr (std::is_same<T, double>::value)
            o[u] = __dmul_rn(wt, g[u]);
          else
            o[u] = wt * g[u];
          part = fma(g[u], yv[u], part);
        }
        if (write_dys) reinterpret_cast<uint4*>(dr)[c] = pack16<T, A>(o);
      }
    } else {
      for (int64_t c = lane; c < d; c += 32) {
        const A g = (A)to_f(dyr[c]);
        if (write_dys) {
          if constexpr (std::is_same<T, double>::value)
            dr[c] = __dmul_rn(wt, g);
          else
            dr[c] = from_f<T>((float)(wt * g));
        }
        part = fma(g, (A)to_f(yr[c]), part);
      }
    }
    A dot;
    if constexpr (std::is_same<T, double>::value) {
      dot = lane == 0 ? dot_ref_seq<A>(dyr, yr, d) : A(0);  // parity: reference order
      (void)part;
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      dot = part;
    }
    if (lane == 0) d_w[i * k + j] = (S)dot;
    if (j < 8) dw_f[j] = (float)dot;
  }
gate_jacobian:
  if (dz != nullptr) {
    // Softmax Jacobian (gate.cpp:44-59) fused: ds is k-sparse.
    const int E = (int)p.n_experts;
    const float* s = scores + i * E;
    int ix[8];
    float dot = 0.f;
    for (int j = 0; j < k && j < 8; ++j) {
      ix[j] = __ldg(topk_idx + i * k + j);
      dot = fmaf(dw_f[j], __ldg(s + ix[j]), dot);
    }
    for (int e = lane; e < E; e += 32) {
      float dse = 0.f;
      for (int j = 0; j < k && j < 8; ++j)
        if (ix[j] == e) dse += dw_f[j];
      dz[i * E + e] = __float2bfloat16_rn(__ldg(s + e) * (dse - dot));
    }
  }
}

// --------------------------------------------------------------- colsum
template <typename T, typename O>
__global__ void block_colsum_kernel(const T* __restrict__ src, int64_t n_cols,
                                    const int32_t* __restrict__ offsets,
                                    const int32_t* __restrict__ counts, O* __restrict__ out) {
  const int g = blockIdx.y;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cols) return;
  const int64_t r0 = __ldg(offsets + g), n = __ldg(counts + g);
  O acc = O(0);
  const T* p = src + r0 * n_cols + c;
  int64_t r = 0;
  for (; r + 8 <= n; r += 8) {
    T v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = p[(r + u) * n_cols];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += (O)to_f(v[u]);
  }
  for (; r < n; ++r) acc += (O)to_f(p[r * n_cols]);
  out[(int64_t)g * n_cols + c] = acc;
}

// ------------------------------------------------- tile column sums (bf16)
// part[t][c] = sum of the 128 rows of tile t (fp32), rows in order.  One block
// per tile; a thread owns 8 columns (one 16-byte vector per row) and keeps 8
// rows of loads in flight, so the pass streams d_ys at HBM rate.
__global__ void __launch_bounds__(256) tile_colsum_kernel(const __nv_bfloat16* __restrict__ src, int64_t n_cols,
                                                          const int32_t* __restrict__ n_tiles, float* __restrict__ part) {
  pdl_wait();
  const int64_t t = blockIdx.x;
  if (t >= __ldg(n_tiles)) return;
  const int64_t nv = n_cols / 8;
  for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
    const uint4* p = reinterpret_cast<const uint4*>(src + t * 128 * n_cols) + v;
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    for (int r = 0; r < 128; r += 8) {
      uint4 u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) u[q] = __ldg(p + (r + q) * nv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t w[4] = {u[q].x, u[q].y, u[q].z, u[q].w};
#pragma unroll
        for (int z = 0; z < 4; ++z) {
          acc[2 * z] += __uint_as_float(w[z] << 16);
          acc[2 * z + 1] += __uint_as_float(w[z] & 0xffff0000u);
        }
      }
    }
    float4* o = reinterpret_cast<float4*>(part + t * n_cols + v * 8);
    o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// out[e][c] = sum over expert e's tiles, in tile order (deterministic).  Two
// partial sets in one launch: column blocks [0, nb1) reduce part1 (n1
// columns), the rest part2 (n2 columns); eight tiles' loads in flight.
__global__ void reduce_tile_partials_kernel(const float* __restrict__ part1, int64_t n1, float* __restrict__ out1,
                                            const float* __restrict__ part2, int64_t n2, float* __restrict__ out2,
                                            const int32_t* __restrict__ offsets) {
  pdl_wait();
  const int e = blockIdx.y;
  const int64_t nb1 = (n1 + blockDim.x - 1) / blockDim.x;
  const bool first = blockIdx.x < nb1;
  const float* part = first ? part1 : part2;
  const int64_t n = first ? n1 : n2;
  float* out = first ? out1 : out2;
  const int64_t c = (int64_t)(first ? blockIdx.x : blockIdx.x - nb1) * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int t0 = __ldg(offsets + e) / 128, t1 = __ldg(offsets + e + 1) / 128;
  float s = 0.f;
  int t = t0;
  for (; t + 8 <= t1; t += 8) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = part[(int64_t)(t + j) * n + c];
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  for (; t < t1; ++t) s += part[(int64_t)t * n + c];
  out[(int64_t)e * n + c] = s;
}

// order[rank] = group, ranked by decreasing row count (offsets[g+1] -
// offsets[g]), ties by index: O(G^2) comparisons in one block.
__global__ void order_groups_kernel(const int32_t* __restrict__ offsets, int G, int32_t* __restrict__ order) {
  pdl_wait();
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const int c = offsets[g + 1] - offsets[g];
    int rank = 0;
    for (int h = 0; h < G; ++h) {
      const int ch = offsets[h + 1] - offsets[h];
      rank += (ch > c) || (ch == c && h < g);
    }
    order[rank] = g;
  }
}

}  // namespace

void order_groups_desc(Ctx* ctx, const int32_t* offsets, int64_t groups, int32_t* order) {
  if (groups <= 0) return;
  CK(launch_pdl(order_groups_kernel, dim3(1), dim3(1024), 0, ctx->stream, offsets, (int)groups, order));
  CK_LAUNCH(ctx);
}

void tile_colsum(Ctx* ctx, const __nv_bfloat16* src, int64_t n_cols, const int32_t* n_tiles,
                 int64_t max_tiles, float* part) {
  if (max_tiles == 0 || n_cols == 0) return;
  if (n_cols % 8) shape_error("tile_colsum: columns must be a multiple of 8");
  const int threads = (int)std::min<int64_t>(256, ceil_div(n_cols / 8, 32) * 32);
  CK(launch_pdl(tile_colsum_kernel, dim3((unsigned)max_tiles), dim3(threads), 0, ctx->stream, src, n_cols, n_tiles,
                part));
  CK_LAUNCH(ctx);
}

void reduce_tile_partials(Ctx* ctx, const float* part, int64_t n_cols, const int32_t* offsets,
                          int64_t n_blocks, float* out, const float* part2, int64_t n_cols2, float* out2) {
  if (n_blocks == 0 || (n_cols == 0 && n_cols2 == 0)) return;
  if (!part2) n_cols2 = 0;
  dim3 grid((unsigned)(ceil_div(n_cols, 256) + ceil_div(n_cols2, 256)), (unsigned)n_blocks);
  CK(launch_pdl(reduce_tile_partials_kernel, grid, dim3(256), 0, ctx->stream, part, n_cols, out,
                (const float*)part2, n_cols2, out2, offsets));
  CK_LAUNCH(ctx);
}

void scatter(Ctx* ctx, fmoe_dtype t, const void* x, int64_t d, const fmoe_plan& p, void* xs,
             const ScatterRoute* route) {
  const int64_t warps = p.n_b + (p.align > 1 ? p.n_experts * p.align : 0);
  if (warps == 0) return;
  const unsigned grid = (unsigned)ceil_div(warps * 32, 256);
  CK(launch_pdl(scatter_kernel, dim3(grid), dim3(256), 0, ctx->stream, reinterpret_cast<const uint8_t*>(x),
                d * (int64_t)dtype_size(t), p, reinterpret_cast<uint8_t*>(xs), route ? *route : ScatterRoute{}));
  CK_LAUNCH(ctx);
}

void gather_combine(Ctx* ctx, fmoe_dtype t, const void* ys, int64_t d, const fmoe_plan& p,
                    const void* w, void* y) {
  if (p.n_b == 0) return;
  const unsigned grid = (unsigned)ceil_div(p.n_b * 32, 256);
  dispatch_dtype(t, [&](auto* tag) {
    using T = std::remove_pointer_t<decltype(tag)>;
    using S = typename ScoreOf<T>::type;
    CK(launch_pdl(gather_combine_kernel<T, S>, dim3(grid), dim3(256), 0, ctx->stream, reinterpret_cast<const T*>(ys),
                  d, p, reinterpret_cast<const S*>(w), reinterpret_cast<T*>(y)));
  });
  CK_LAUNCH(ctx);
}

void scatter_bwd(Ctx* ctx, fmoe_dtype t, const void* d_xs, int64_t d, const fmoe_plan& p, void* dx,
                 const void* addend) {
  if (p.n_b == 0) return;
  const unsigned grid = (unsigned)ceil_div(p.n_b * 32, 256);
  dispatch_dtype(t, [&](auto* tag) {
    using T = std::remove_pointer_t<decltype(tag)>;
    if (p.k <= 2)
      CK(launch_pdl(scatter_bwd_kernel<T, 2>, dim3(grid), dim3(256), 0, ctx->stream, reinterpret_cast<const T*>(d_xs),
                    d, p, reinterpret_cast<const T*>(addend), reinterpret_cast<T*>(dx)));
    else
      CK(launch_pdl(scatter_bwd_kernel<T, 4>, dim3(grid), dim3(256), 0, ctx->stream, reinterpret_cast<const T*>(d_xs),
                    d, p, reinterpret_cast<const T*>(addend), reinterpret_cast<T*>(dx)));
  });
  CK_LAUNCH(ctx);
}

void gather_combine_bwd(Ctx* ctx, fmoe_dtype t, const void* dy, const void* ys, int64_t d,
                        const fmoe_plan& p, const void* w, void* d_ys, void* d_w,
                        const void* scores, const int32_t* topk_idx, __nv_bfloat16* dz,
                        const ScatterRoute* route) {
  const int64_t warps = p.n_b + (p.align > 1 ? p.n_experts * p.align : 0);
  if (warps == 0) return;
  if (dz && p.k > 8) shape_error("fused gate backward supports k <= 8");
  const unsigned grid = (unsigned)ceil_div(warps * 32, 256);
  dispatch_dtype(t, [&](auto* tag) {
    using T = std::remove_pointer_t<decltype(tag)>;
    using S = typename ScoreOf<T>::type;
    CK(launch_pdl(gcb_kernel<T, S>, dim3(grid), dim3(256), 0, ctx->stream, reinterpret_cast<const T*>(dy),
                  reinterpret_cast<const T*>(ys), d, p, reinterpret_cast<const S*>(w), reinterpret_cast<T*>(d_ys),
                  reinterpret_cast<S*>(d_w), reinterpret_cast<const float*>(scores), topk_idx, dz,
                  route ? *route : ScatterRoute{}));
  });
  CK_LAUNCH(ctx);
}

void block_colsum(Ctx* ctx, fmoe_dtype t, const void* src, int64_t n_cols, const int32_t* offsets,
                  const int32_t* counts, int64_t n_blocks, void* out) {
  if (n_blocks == 0 || n_cols == 0) return;
  dim3 grid((unsigned)ceil_div(n_cols, 128), (unsigned)n_blocks);
  dispatch_dtype(t, [&](auto* tag) {
    using T = std::remove_pointer_t<decltype(tag)>;
    using O = typename ScoreOf<T>::type;  // f64 -> f64, else f32
    block_colsum_kernel<T, O><<<grid, 128, 0, ctx->stream>>>(reinterpret_cast<const T*>(src), n_cols,
                                                            offsets, counts, reinterpret_cast<O*>(out));
  });
  CK_LAUNCH(ctx);
}

}  // namespace fmoe_b200
