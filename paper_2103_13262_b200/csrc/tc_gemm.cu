// tc_gemm.cu -- see tc_gemm.cuh for the design.
#include <cuda.h>

#include <mutex>

#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace fmoe_b200 {
namespace tc {

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;          // 16 KiB
  static constexpr int B_BYTES = BN * BK * 2;          // 8/16/32 KiB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (196 * 1024) / STAGE_BYTES > 8 ? 8 : (196 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;             // two fp32 accumulators
  static constexpr int COLSUM_BYTES = 4 * BN * 4;      // per-warp column sums of one tile
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + COLSUM_BYTES;
};

// Named barrier among the 4 epilogue warps (ids 1.. are free; 0 = __syncthreads).
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// After the call lane L holds sum over the warp's 32 lanes of v[L] (31 shuffles).
__device__ __forceinline__ float warp_transpose_sum(float (&v)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const float send = upper ? v[i] : v[i + o];
      const float keep = upper ? v[i + o] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0];
}

// K-major / MN-major canonical SW128 layouts (cute UMMA::make_umma_desc):
//   K-major : 8-row x 128 B atoms, SBO = 1024 (next 8 rows), LBO unused (=16 B)
//   MN-major: 64-element x 8-k-row atoms; LBO = next 64 MN elements (one TMA
//             box of 64 k-rows = 8 KiB), SBO = 1024 (next 8 k-rows)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, bool mn) {
  const uint32_t lbo = mn ? 8192u : 16u;
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: D f32, A/B bf16, M=128, N=BN.
template <int BN, bool A_MN, bool B_MN>
__device__ __forceinline__ constexpr uint32_t idesc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

struct Tile {
  int g, m0, n0, kbeg, nkb;
};

template <int BN>
__device__ __forceinline__ int n_tiles_n(const Params& p) {
  return (p.N + BN - 1) / BN;
}

template <int BN>
__device__ __forceinline__ int total_tiles(const Params& p) {
  const int nn = n_tiles_n<BN>(p);
  if (p.mode == RAGGED_M) {
    const int nm = p.n_mtiles ? *p.n_mtiles : (p.M + BM - 1) / BM;
    return nm * nn;
  }
  return p.n_groups * ((p.M + BM - 1) / BM) * nn;
}

template <int BN>
__device__ __forceinline__ Tile decode(const Params& p, int t) {
  Tile r;
  const int nn = n_tiles_n<BN>(p);
  if (p.mode == RAGGED_M) {
    const int mt = t / nn;
    r.n0 = (t - mt * nn) * BN;
    r.m0 = mt * BM;
    r.g = p.tile_group ? __ldg(p.tile_group + mt) : 0;
    r.kbeg = 0;
    r.nkb = (p.K + BK - 1) / BK;
  } else {
    const int nm = (p.M + BM - 1) / BM;
    const int per = nm * nn;
    r.g = t / per;
    const int rem = t - r.g * per;
    const int mt = rem / nn;
    r.m0 = mt * BM;
    r.n0 = (rem - mt * nn) * BN;
    r.kbeg = __ldg(p.k_offsets + r.g);
    const int kend = __ldg(p.k_offsets + r.g + 1);
    r.nkb = (kend - r.kbeg + BK - 1) / BK;
  }
  return r;
}

// ------------------------------------------------------------- epilogues
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int BN>
__device__ __forceinline__ void epi_store_chunk(const Params& p, const Tile& tl, int row, int c0,
                                                float (&v)[32]) {
  // row: absolute row in the output tile space; c0: absolute column of v[0]
  if (p.epi == EPI_F32) {
    float* out = reinterpret_cast<float*>(p.C) + (int64_t)tl.g * p.c_group_stride +
                 (int64_t)row * p.ldc + c0;
    if (row >= p.M) return;
    if (c0 + 32 <= p.N) {
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(out + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
      for (int i = 0; i < 32; ++i)
        if (c0 + i < p.N) out[i] = v[i];
    }
    return;
  }
  // bf16 outputs (RAGGED_M row space)
  if (row >= p.M) return;
  if (p.epi == EPI_BF16) {
    if (p.bias) {
      const float* b = p.bias + (int64_t)tl.g * p.bias_group_stride + c0;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 bb = (c0 + i + 4 <= p.N) ? __ldg(reinterpret_cast<const float4*>(b + i))
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
        v[i] += bb.x; v[i + 1] += bb.y; v[i + 2] += bb.z; v[i + 3] += bb.w;
      }
    }
    if (p.relu) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = v[i] < 0.f ? 0.f : v[i];
    }
  } else if (p.epi == EPI_MASK_BF16) {
    const uint4* m = reinterpret_cast<const uint4*>(p.mask + (int64_t)row * p.ldm + c0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 mv = __ldg(m + q);
      const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mv);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[q * 8 + i] = __bfloat162float(mb[i]) > 0.f ? v[q * 8 + i] : 0.f;
    }
  } else if (p.epi == EPI_GATE_DX) {
    float s[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) s[i] = 0.f;
    for (int j = 0; j < p.gk; ++j) {
      const int pos = __ldg(p.inverse_pos + (int64_t)row * p.gk + j);
      const uint4* src = reinterpret_cast<const uint4*>(p.gather_src + (int64_t)pos * p.N + c0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 gv = __ldg(src + q);
        const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&gv);
#pragma unroll
        for (int i = 0; i < 8; ++i) s[q * 8 + i] += __bfloat162float(gb[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = s[i] + v[i];
  }
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.C) + (int64_t)row * p.ldc + c0;
  uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    o4[q] = make_uint4(pack_bf16(v[q * 8 + 0], v[q * 8 + 1]), pack_bf16(v[q * 8 + 2], v[q * 8 + 3]),
                       pack_bf16(v[q * 8 + 4], v[q * 8 + 5]), pack_bf16(v[q * 8 + 6], v[q * 8 + 7]));
}

__device__ __forceinline__ void load_chunk(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  tmem_ld_32x32b_x32(taddr, r);
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Gate epilogue: the thread owns one token row and all E = N logits.
// softmax_rows (matrix.cpp:155-170): max, exp(l - max), sequential sum, divide;
// topk_rows (matrix.cpp:172-189): descending, ties keep the lower expert.
template <int BN>
__device__ __forceinline__ void epi_gate(const Params& p, uint32_t tbase, int row) {
  constexpr int KMAX = 8;
  const int E = p.N;
  float mx = -INFINITY;
  for (int c = 0; c < BN / 32; ++c) {
    if (c * 32 >= E) break;
    float v[32];
    load_chunk(tbase + c * 32, v);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (c * 32 + i < E) mx = fmaxf(mx, v[i]);
  }
  float sum = 0.f;
  for (int c = 0; c < BN / 32; ++c) {
    if (c * 32 >= E) break;
    float v[32];
    load_chunk(tbase + c * 32, v);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (c * 32 + i < E) sum += expf(v[i] - mx);
  }
  float tv[KMAX];
  int ti[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    tv[j] = -INFINITY;
    ti[j] = -1;
  }
  const bool valid = row < p.M;
  const int k = p.topk;
  for (int c = 0; c < BN / 32; ++c) {
    if (c * 32 >= E) break;
    float v[32];
    load_chunk(tbase + c * 32, v);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int col = c * 32 + i;
      if (col < E) {
        const float s = __fdiv_rn(expf(v[i] - mx), sum);
        if (valid) p.scores[(int64_t)row * E + col] = s;
        // insertion into the sorted top-k list (strict > keeps lower index first)
        float cs = s;
        int ci = col;
        bool carry = false;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
          if (j < k) {
            const bool take = carry || (cs > tv[j]);
            if (take) {
              const float tf = tv[j];
              const int tix = ti[j];
              tv[j] = cs;
              ti[j] = ci;
              cs = tf;
              ci = tix;
              carry = true;
            }
          }
        }
      }
    }
  }
  if (valid && k > 0) {
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < k) {
        p.topk_idx[(int64_t)row * k + j] = ti[j];
        p.topk_val[(int64_t)row * k + j] = tv[j];
      }
  }
}

// ------------------------------------------------------------------ kernel
template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const Params p) {
  using C = Cfg<BN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + STAGES * C::B_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* colsum_smem = reinterpret_cast<float*>(smem + STAGES * C::STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(full + s), 1);
      mbar_init(smem_u32(empty + s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(tfull + a), 1);
      mbar_init(smem_u32(tempty + a), 8);  // one arrive per epilogue warp
    }
    fence_mbarrier_init();
  }
  if (warp == 2) {
    tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total = total_tiles<BN>(p);

  if (warp == 0) {
    if (lane == 0) {
      // ======================= TMA producer =======================
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const Tile tl = decode<BN>(p, t);
        const int brow = (p.mode == RAGGED_M) ? tl.g * p.b_group_rows : tl.kbeg;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          mbar_wait(smem_u32(empty + stage), phase ^ 1);
          const uint32_t fb = smem_u32(full + stage);
          mbar_arrive_expect_tx(fb, C::STAGE_BYTES);
          const uint32_t a_dst = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_dst = smem_u32(sB + stage * C::B_BYTES);
          if (!A_MN) {
            tma_load_2d(a_dst, &tmA, fb, kb * BK, tl.m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(a_dst + j * 8192, &tmA, fb, tl.m0 + 64 * j, tl.kbeg + kb * BK);
          }
          if (!B_MN) {
            tma_load_2d(b_dst, &tmB, fb, kb * BK, brow + tl.n0);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(b_dst + j * 8192, &tmB, fb, tl.n0 + 64 * j, brow + kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ======================= MMA issuer =========================
      constexpr uint32_t ID = idesc<BN, A_MN, B_MN>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const Tile tl = decode<BN>(p, t);
        if (tl.nkb == 0) continue;
        mbar_wait(smem_u32(tempty + acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          mbar_wait(smem_u32(full + stage), phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = sdesc(a_addr + (A_MN ? k * 2048 : k * 32), A_MN);
            const uint64_t bd = sdesc(b_addr + (B_MN ? k * 2048 : k * 32), B_MN);
            tc_mma_f16(d_tmem, ad, bd, ID, (kb | k) != 0);
          }
          tc_commit(smem_u32(empty + stage));
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(smem_u32(tfull + acc));
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ========================= epilogue ===========================
    // 8 warps: warp w reads TMEM lanes 32*(w%4).. (the hardware lane quarter
    // of its sub-partition) and half (w-4)/4 of the tile's column chunks.
    const int q = warp & 3;
    const int ew = warp - 4;  // 0..7
    constexpr int NC = BN / 32;
    const int c_lo = (ew >> 2) * (NC / 2), c_hi = c_lo + NC / 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const Tile tl = decode<BN>(p, t);
      const int row = tl.m0 + q * 32 + lane;
      if (tl.nkb == 0) {
        // empty K range (expert without tokens): gradient is exactly zero
        if (p.epi == EPI_F32) {
          for (int c = c_lo; c < c_hi; ++c) {
            float z[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) z[i] = 0.f;
            if (tl.n0 + c * 32 < p.N) epi_store_chunk<BN>(p, tl, row, tl.n0 + c * 32, z);
          }
        }
        continue;
      }
      mbar_wait(smem_u32(tfull + acc), acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (p.epi == EPI_GATE) {
        if (ew < 4) epi_gate<BN>(p, tbase, row);  // one thread owns a whole row of logits
      } else {
        for (int c = c_lo; c < c_hi; ++c) {
          if (tl.n0 + c * 32 >= p.N) break;
          float v[32];
          load_chunk(tbase + c * 32, v);
          epi_store_chunk<BN>(p, tl, row, tl.n0 + c * 32, v);
          if (p.colsum_part) {  // column sums of the final fp32 values of this tile
            if (row >= p.M) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.f;
            }
            colsum_smem[q * BN + c * 32 + lane] = warp_transpose_sum(v, lane);
          }
        }
        if (p.colsum_part) {
          epi_bar();
          for (int col = ew * 32 + lane; col < BN; col += 256)
            if (tl.n0 + col < p.N)
              p.colsum_part[(int64_t)(tl.m0 / BM) * p.N + tl.n0 + col] =
                  colsum_smem[col] + colsum_smem[BN + col] + colsum_smem[2 * BN + col] + colsum_smem[3 * BN + col];
          epi_bar();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(tempty + acc));
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------- host
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) throw Error(FMOE_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}
}  // namespace

CUtensorMap make_tmap(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                      uint32_t box_inner, uint32_t box_outer) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                 strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(FMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) +
                                   ") inner=" + std::to_string(inner) + " outer=" + std::to_string(outer));
  return m;
}

template <int BN, bool A_MN, bool B_MN>
static void launch_t(Ctx* ctx, const CUtensorMap& ta, const CUtensorMap& tb, const Params& p,
                     int64_t max_tiles) {
  auto kern = tc_gemm_kernel<BN, A_MN, B_MN>;
  static bool attr_set[8] = {};
  const int dev = ctx->device & 7;
  if (!attr_set[dev]) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
    attr_set[dev] = true;
  }
  int64_t grid = ctx->num_sms;
  if (max_tiles < grid) grid = max_tiles;
  if (grid < 1) return;
  kern<<<(unsigned)grid, NUM_THREADS, Cfg<BN>::SMEM, ctx->stream>>>(ta, tb, p);
  CK_LAUNCH(ctx);
}

void launch(Ctx* ctx, int bn, bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb,
            const Params& p, int64_t max_tiles) {
#define FMOE_TC_CASE(BN_, AM, BM_)                          \
  if (bn == BN_ && a_mn == AM && b_mn == BM_) {             \
    launch_t<BN_, AM, BM_>(ctx, ta, tb, p, max_tiles);      \
    return;                                                 \
  }
  FMOE_TC_CASE(256, false, true)   // expert fc1/fc2 forward
  FMOE_TC_CASE(256, false, false)  // dgrad, gate dx
  FMOE_TC_CASE(256, true, true)    // weight gradients
  FMOE_TC_CASE(128, false, true)
  FMOE_TC_CASE(128, false, false)
  FMOE_TC_CASE(128, true, true)
  FMOE_TC_CASE(64, false, true)    // gate logits (E <= 64), gate dWg partials
  FMOE_TC_CASE(64, false, false)
  FMOE_TC_CASE(64, true, true)
#undef FMOE_TC_CASE
  shape_error("tc gemm: unsupported tile configuration");
}

}  // namespace tc
}  // namespace fmoe_b200
