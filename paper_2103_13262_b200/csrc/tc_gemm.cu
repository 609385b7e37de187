// tc_gemm.cu -- see tc_gemm.cuh for the design.
#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "ptx.cuh"
#include "tc_gemm.cuh"

namespace fmoe_b200 {
namespace tc {

// CG = CTAs per MMA (cta_group): 1 -> 128 x BN tiles per CTA; 2 -> 256 x BN tiles
// per CTA pair, each CTA holding its 128 rows of A and BN/2 rows of B.
template <int BN, int CG = 1, int EPI = EPI_F32>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;          // 16 KiB: this CTA's 128 rows
  static constexpr int B_BYTES = (BN / CG) * BK * 2;   // this CTA's share of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;             // two fp32 accumulators
  static constexpr bool F32OUT = EPI == EPI_F32 || EPI == EPI_F32X;  // fp32 output tiles
  static constexpr int COLSUM_BYTES = F32OUT ? 0 : 4 * BN * 4;  // per-warp column sums of one tile
  // outputs leave through TMA stores from per-warp staging tiles of 32 rows x
  // 64 B (64B swizzle): 32 bf16 columns, or 16 fp32 columns (a 32-column fp32
  // chunk is stored as two halves).  One tile per warp keeps 6 pipeline
  // stages in shared memory.
  static constexpr bool TMA_STORE = EPI == EPI_BF16 || EPI == EPI_MASK_BF16 || F32OUT;
#ifndef FMOE_TC_F32_ROW_BYTES
#define FMOE_TC_F32_ROW_BYTES 64  // fp32 staging rows: 64 B (16 columns, two stores per chunk); 128 B
                                  // (one 32-column store) measured 5% slower weight gradients
#endif
  static constexpr int OUT_ROW_BYTES = F32OUT ? FMOE_TC_F32_ROW_BYTES : 64;
#ifndef FMOE_TC_BF16_NBUF
#define FMOE_TC_BF16_NBUF 1  // staging tiles per epilogue warp for bf16 outputs (A/B: 2 tiles cost a
                             // pipeline stage or the 227 KB plan; both measured slower overall)
#endif
#ifndef FMOE_TC_F32_NBUF
#define FMOE_TC_F32_NBUF 1  // staging tiles per epilogue warp for fp32 (weight-gradient) outputs
#endif
  static constexpr int NBUF = F32OUT ? FMOE_TC_F32_NBUF : FMOE_TC_BF16_NBUF;
  static constexpr int TILE_BYTES = 32 * OUT_ROW_BYTES;
  // gate (E <= 64): each epilogue lane stages its row of scores (padded to
  // avoid bank conflicts) and stores it as one contiguous bulk copy
  static constexpr bool GATE_STAGE = EPI == EPI_GATE && BN == 64;
  static constexpr int GATE_ROW_BYTES = BN * 4 + 16;
  static constexpr int STORE_BYTES = TMA_STORE ? 8 * NBUF * TILE_BYTES : GATE_STAGE ? 8 * 32 * GATE_ROW_BYTES : 0;
  // bf16 epilogues stage the bias of each warp's 128-column slice of the tile
  static constexpr int BIAS_BYTES = EPI == EPI_BF16 ? 8 * (BN / 2) * 4 : 0;
#ifndef FMOE_TC_SMEM_KB
#define FMOE_TC_SMEM_KB 200  // per-CTA shared memory the GEMM plans for: 5 stages (227 -> 6 stages
                             // measured equal in time with ~25% more DRAM traffic)
#endif
#ifndef FMOE_TC_F32_SMEM_KB
#define FMOE_TC_F32_SMEM_KB FMOE_TC_SMEM_KB
#endif
  static constexpr int BUDGET = (GATE_STAGE ? 224 : F32OUT ? FMOE_TC_F32_SMEM_KB : FMOE_TC_SMEM_KB) * 1024 -
                                1280 /*align + barriers*/ - STORE_BYTES - COLSUM_BYTES - BIAS_BYTES;
  static constexpr int STAGES = BUDGET / STAGE_BYTES > 8 ? 8 : BUDGET / STAGE_BYTES;
  static constexpr int SMEM =
      STAGES * STAGE_BYTES + STORE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + COLSUM_BYTES + BIAS_BYTES;
  static_assert(SMEM <= 227 * 1024, "tc_gemm: shared memory over the sm_100 per-CTA limit");
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

// Instruction descriptor, kind::f16: D f32, A/B bf16, M=128*CG, N=BN.
template <int BN, bool A_MN, bool B_MN, int CG>
__device__ __forceinline__ constexpr uint32_t idesc() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((BM * CG) >> 4) << 24);
}

struct Tile {
  int g, m0, n0, kbeg, nkb;  // m0: first row of the (pair) tile; nkb: k-blocks of all phases
  int kpp;                   // k-blocks per phase (bf16x3: nkb = 3 * kpp)
  int lo, hi;                // RAGGED_M: rows the epilogue owns (row_split chunks overlap)
};

template <int BN>
__device__ __forceinline__ int n_tiles_n(const Params& p) {
  return (p.N + BN - 1) / BN;
}

// Tile rows = BM*CG.  RAGGED_M row tiles are counted in 128-row units by the
// plan (n_mtiles, tile_group); with CG=2 the plan aligns expert blocks to 256.
template <int BN, int CG>
__device__ __forceinline__ int total_tiles(const Params& p) {
  const int nn = n_tiles_n<BN>(p);
  if (p.mode == RAGGED_M) {
    if (p.row_split) return p.row_split * p.row_chunks;
    const int nm = p.n_mtiles ? (*p.n_mtiles + CG - 1) / CG : (p.M + BM * CG - 1) / (BM * CG);
    return nm * nn;
  }
  return p.n_groups * ((p.M + BM * CG - 1) / (BM * CG)) * nn;
}

template <int BN, int CG, bool SPLIT = false>
__device__ __forceinline__ Tile decode(const Params& p, int t) {
  Tile r;
  const int nn = n_tiles_n<BN>(p);
  if (p.mode == RAGGED_M && p.row_split) {  // balanced row ranges (CG = 1, N <= BN)
    const int S = p.row_split, slot = t % S, c = t / S;
    const int rb = (int)((int64_t)slot * p.M / S), re = (int)((int64_t)(slot + 1) * p.M / S);
    const int start = rb + c * BM;
    r.m0 = re - rb >= BM ? min(start, re - BM) : rb;
    r.lo = start;
    r.hi = min(re, r.m0 + BM);
    r.n0 = 0;
    r.g = 0;
    r.kbeg = 0;
    r.kpp = start < re ? (p.K + BK - 1) / BK : 0;
  } else if (p.mode == RAGGED_M) {
    const int mt0 = t / nn;
    r.n0 = (t - mt0 * nn) * BN;
    const int mt = p.mtile_order ? __ldg(p.mtile_order + mt0) : mt0;
    r.m0 = mt * BM * CG;
    r.g = p.tile_group ? __ldg(p.tile_group + mt * CG) : 0;
    r.kbeg = 0;
    r.kpp = (p.K + BK - 1) / BK;
    r.lo = r.m0;
    r.hi = p.M;
  } else {
    const int nm = (p.M + BM * CG - 1) / (BM * CG);
    const int per = nm * nn;
    const int gs = t / per;
    r.g = p.group_order ? __ldg(p.group_order + gs) : gs;
    const int rem = t - gs * per;
    const int mt = rem / nn;
    r.m0 = mt * BM * CG;
    r.n0 = (rem - mt * nn) * BN;
    int kend;
    if (p.k_offsets) {
      r.kbeg = __ldg(p.k_offsets + r.g);
      kend = __ldg(p.k_offsets + r.g + 1);
    } else {  // uniform splits (gate d_wg)
      r.kbeg = r.g * p.k_split;
      kend = min(p.K, r.kbeg + p.k_split);
    }
    r.kpp = (kend - r.kbeg + BK - 1) / BK;
  }
  r.nkb = (SPLIT && p.phases > 1) ? r.kpp * p.phases : r.kpp;  // split passes: fp32-output kernels only
  return r;
}

// Tile of iteration `it` of the persistent CTA (pair) `slot` out of `nslots`:
// round-robin, or for group-ordered RAGGED_K a snake over the slots (rounds
// alternate direction) so the heaviest tiles, dealt first, spread evenly.
// Returns -1 when the iteration has no tile; iterations end at `total`.
__device__ __forceinline__ int tile_at(const Params& p, int it, int slot, int nslots) {
  if (!p.group_order) return it * nslots + slot;
  return it * nslots + ((it & 1) ? nslots - 1 - slot : slot);
}

// ------------------------------------------------------------- epilogues
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Relu bitmap word of (row, 32-column chunk at c0), laid out so the 32 rows a
// warp drains form one contiguous 128-byte line: [row/32][c0/32][row%32].
__device__ __forceinline__ int64_t relu_bits_index(int row, int c0, int n) {
  return (((int64_t)(row >> 5) * (n >> 5) + (c0 >> 5)) << 5) + (row & 31);
}

template <int BN, int EPI>
__device__ __forceinline__ void epi_store_chunk(const Params& p, const Tile& tl, int row, int c0,
                                                float (&v)[32], uint32_t bits = 0,
                                                uint32_t stage_addr = 0) {
  // row: absolute row in the output tile space; c0: absolute column of v[0]
  if constexpr (EPI == EPI_F32 || EPI == EPI_F32X) {
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
  // bf16 outputs (RAGGED_M row space).  With a TMA-store staging tile every
  // lane still writes its (dummy) row; the tensor map clips rows >= M.
  if (row >= p.M) {
    if (!stage_addr) return;
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.f;
  } else if constexpr (EPI == EPI_BF16) {
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
      if (p.relu_bits_out) {
        uint32_t b = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) b |= (v[i] > 0.f ? 1u : 0u) << i;
        p.relu_bits_out[relu_bits_index(row, c0, p.N)] = b;
      }
    }
  } else if constexpr (EPI == EPI_MASK_BF16) {
    if (p.relu_bits) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = ((bits >> i) & 1u) ? v[i] : 0.f;
    } else {
    const uint4* m = reinterpret_cast<const uint4*>(p.mask + (int64_t)row * p.ldm + c0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 mv = __ldg(m + q);
      const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mv);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[q * 8 + i] = __bfloat162float(mb[i]) > 0.f ? v[q * 8 + i] : 0.f;
    }
    }
  } else if constexpr (EPI == EPI_GATE_DX) {
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
  if (stage_addr) {
    // 32 rows x 64 B staging tile in the TMA SWIZZLE_64B layout: 16-byte chunk
    // j of row r sits at r*64 + ((j ^ ((r >> 1) & 3)) << 4)
    const uint32_t r = threadIdx.x & 31;
    const uint32_t base = stage_addr + r * 64;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t a = base + (((uint32_t)q ^ ((r >> 1) & 3u)) << 4);
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                   "r"(pack_bf16(v[q * 8 + 0], v[q * 8 + 1])), "r"(pack_bf16(v[q * 8 + 2], v[q * 8 + 3])),
                   "r"(pack_bf16(v[q * 8 + 4], v[q * 8 + 5])), "r"(pack_bf16(v[q * 8 + 6], v[q * 8 + 7]))
                   : "memory");
    }
    return;
  }
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(p.C) + (int64_t)row * p.ldc + c0;
  if (p.route_out) {  // fused global_gather: the row goes home over NVLink
    const int W = p.route_world;
    out = nullptr;
    for (int s = 0; s < W; ++s) {
      const int start = __ldg(p.route_start + tl.g * W + s);
      if ((unsigned)(row - start) < (unsigned)__ldg(p.route_rows + tl.g * W + s)) {
        out = reinterpret_cast<__nv_bfloat16*>(p.route_out[s]) +
              (int64_t)(__ldg(p.route_dst + tl.g * W + s) + row - start) * p.ldc + c0;
        break;
      }
    }
    if (!out) return;  // pad row
  }
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

// Gate epilogue for E <= 64 (BN = 64): the row's logits stay in registers, so
// each exp is computed once; scores leave as 16-byte stores; top-2 (the
// common case) is a two-slot insertion.  Same arithmetic as epi_gate below:
// max, exp(l - max), sequential sum, correctly rounded division, descending
// selection with ties to the lower expert (matrix.cpp:155-189).
__device__ __forceinline__ void epi_gate64(const Params& p, uint32_t tbase, int row, bool valid, uint32_t stage_row) {
  const int E = p.N;
  float ev[64];
  {
    uint32_t r0[32], r1[32];
    tmem_ld_issue(tbase, r0);
    if (E > 32) tmem_ld_issue(tbase + 32, r1);
    tmem_ld_wait(r0);
    if (E > 32) tmem_ld_wait(r1);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      ev[i] = __uint_as_float(r0[i]);
      ev[32 + i] = E > 32 ? __uint_as_float(r1[i]) : 0.f;
    }
  }
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < 64; ++i)
    if (i < E) mx = fmaxf(mx, ev[i]);
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < 64; ++i)
    if (i < E) {
      ev[i] = __expf(ev[i] - mx);  // ex2.approx: a few ulp, inside the bf16 path's 1e-5 score bound
      sum += ev[i];
    }
  const float rs = __frcp_rn(sum);
#pragma unroll
  for (int i = 0; i < 64; ++i) ev[i] = ev[i] * rs;
  const int k = p.topk;
  if (valid && stage_row) {
    // the row through shared memory, then one contiguous bulk store (a warp's
    // direct float4 stores would each touch 32 rows)
    bulk_wait_read<0>();  // this lane's previous row has left the staging slot
#pragma unroll
    for (int i = 0; i < 64; i += 4)
      if (i < E)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stage_row + i * 4), "f"(ev[i]), "f"(ev[i + 1]),
                     "f"(ev[i + 2]), "f"(ev[i + 3])
                     : "memory");
    fence_proxy_async_smem();
    bulk_store_1d(p.scores + (int64_t)row * E, stage_row, (uint32_t)E * 4);
  } else if (valid) {
    float* srow = p.scores + (int64_t)row * E;
    if (E == 64) {
#pragma unroll
      for (int i = 0; i < 64; i += 4)
        *reinterpret_cast<float4*>(srow + i) = make_float4(ev[i], ev[i + 1], ev[i + 2], ev[i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (i < E) srow[i] = ev[i];
    }
  }
  if (!valid || k <= 0) return;
  if (k == 2) {
    float v0 = -INFINITY, v1 = -INFINITY;
    int i0 = -1, i1 = -1;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      if (i < E) {
        const float s = ev[i];
        // an empty slot takes any value, so a NaN row (every score NaN, the
        // reference's stable sort leaves it in column order) still selects
        // valid experts 0, 1 with NaN scores instead of leaving -1
        if (s > v0 || i0 < 0) {
          v1 = v0; i1 = i0; v0 = s; i0 = i;
        } else if (s > v1 || i1 < 0) {
          v1 = s; i1 = i;
        }
      }
    }
    p.topk_idx[(int64_t)row * 2] = i0;
    p.topk_idx[(int64_t)row * 2 + 1] = i1;
    p.topk_val[(int64_t)row * 2] = v0;
    p.topk_val[(int64_t)row * 2 + 1] = v1;
    return;
  }
  constexpr int KMAX = 8;
  float tv[KMAX];
  int ti[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    tv[j] = -INFINITY;
    ti[j] = -1;
  }
#pragma unroll
  for (int i = 0; i < 64; ++i) {
    if (i < E) {
      float cs = ev[i];
      int ci = i;
      bool carry = false;
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        if (j < k) {
          const bool take = carry || (cs > tv[j]) || ti[j] < 0;  // empty slots take NaN too
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
#pragma unroll
  for (int j = 0; j < KMAX; ++j)
    if (j < k) {
      p.topk_idx[(int64_t)row * k + j] = ti[j];
      p.topk_val[(int64_t)row * k + j] = tv[j];
    }
}

// Gate epilogue: the thread owns one token row and all E = N logits.
// softmax_rows (matrix.cpp:155-170): max, exp(l - max), sequential sum, divide;
// topk_rows (matrix.cpp:172-189): descending, ties keep the lower expert.
template <int BN>
__device__ __forceinline__ void epi_gate(const Params& p, uint32_t tbase, int row, bool valid) {
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
            const bool take = carry || (cs > tv[j]) || ti[j] < 0;  // empty slots take NaN too
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

// Lean drain of one tile for the bf16 expert GEMMs (every row valid, N a
// multiple of BN, TMA-store output): the transforms are selected at compile
// time so a 32-column chunk costs ~one instruction per value per transform.
//   BIAS  += bias (staged in shared memory once per tile)
//   RELU  max(v, 0) and, when p.relu_bits_out, its bitmap (bit = v > 0)
//   MASK  v * bit of p.relu_bits (relu_backward, strict >)
//   COLSUM per-column sums of the final values into colsum_smem
template <int BN, int NBUF, bool BIAS, bool RELU, bool MASK, bool COLSUM>
__device__ __forceinline__ void drain_bf16(const Params& p, const Tile& tl, const CUtensorMap* tmC, uint32_t tbase,
                                           int c_lo, int row, int out_row, uint32_t stage_base, uint32_t& sbuf,
                                           const float* bias_s, float* colsum_smem, int q, int lane) {
  constexpr int CPW = BN / 64;
  constexpr uint32_t TILE_BYTES = 32 * 64;
  uint32_t mbits[CPW];
  if constexpr (MASK) {
#pragma unroll
    for (int i = 0; i < CPW; ++i) mbits[i] = __ldg(p.relu_bits + relu_bits_index(row, tl.n0 + (c_lo + i) * 32, p.N));
  }
  uint32_t buf[2][32];
  tmem_ld_issue(tbase + c_lo * 32, buf[0]);
#pragma unroll
  for (int i = 0; i < CPW; ++i) {
    const int c = c_lo + i;
    tmem_ld_wait(buf[i & 1]);
    if (i + 1 < CPW) tmem_ld_issue(tbase + (c + 1) * 32, buf[(i + 1) & 1]);
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(buf[i & 1][j]);
    if constexpr (BIAS) {
      const float4* b4 = reinterpret_cast<const float4*>(bias_s + i * 32);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 bb = b4[j];
        v[4 * j] += bb.x; v[4 * j + 1] += bb.y; v[4 * j + 2] += bb.z; v[4 * j + 3] += bb.w;
      }
    }
    if constexpr (RELU) {
      uint32_t bits = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        // relu on the bit pattern: every negative float (-0 included) is a
        // negative int, so max(bits, 0) is +0 for them and v otherwise; the
        // mask bit is min(bits, 1) (v > 0 <=> nonzero bits)
        const int xi = max(__float_as_int(v[j]), 0);
        v[j] = __int_as_float(xi);
        bits += min((uint32_t)xi, 1u) << j;
      }
      if (p.relu_bits_out) p.relu_bits_out[relu_bits_index(row, tl.n0 + c * 32, p.N)] = bits;
    }
    if constexpr (MASK) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = ((mbits[i] >> j) & 1u) ? v[j] : 0.f;
    }
    const uint32_t stage = stage_base + sbuf * TILE_BYTES;
    if (lane == 0) bulk_wait_read<NBUF - 1>();
    __syncwarp();
    {
      const uint32_t r = (uint32_t)lane;
      const uint32_t base = stage + r * 64;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const uint32_t a = base + (((uint32_t)qq ^ ((r >> 1) & 3u)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a),
                     "r"(pack_bf16(v[qq * 8 + 0], v[qq * 8 + 1])), "r"(pack_bf16(v[qq * 8 + 2], v[qq * 8 + 3])),
                     "r"(pack_bf16(v[qq * 8 + 4], v[qq * 8 + 5])), "r"(pack_bf16(v[qq * 8 + 6], v[qq * 8 + 7]))
                     : "memory");
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    tma_store_commit_warp(tmC, stage, tl.n0 + c * 32, out_row);
    sbuf = (sbuf + 1) % NBUF;
    if constexpr (COLSUM) colsum_smem[q * BN + c * 32 + lane] = warp_transpose_sum(v, lane);
  }
}

// Overlapped expert-parallel exchange: block until every chunk (expert g,
// source s) that intersects rows [r0, r0 + BM) has been published by its
// sender (see Params::arrive_flags).  Lane 0 polls the local flag words with
// acquire loads; the proxy fence then orders the TMA (async proxy) reads of
// those rows after the observed release.
__device__ __forceinline__ void wait_rows_arrived(const Params& p, int g, int r0, int lane) {
  if (lane == 0) {
    const int W = p.arrive_W, C = p.arrive_C;
    for (int s = 0; s < W; ++s) {
      const int c = g * W + s;
      const int st = __ldg(p.arrive_rt + c), nr = __ldg(p.arrive_rt + C + c);
      if (nr <= 0 || st >= r0 + BM || st + nr <= r0) continue;
      const uint32_t* f = p.arrive_flags + c;
      while (true) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int32_t)(v - p.arrive_epoch) >= 0) break;
        __nanosleep(128);
      }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncwarp();
}

// ------------------------------------------------------------------ kernel
template <int BN, bool A_MN, bool B_MN, int CG, int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ SplitMaps tmS,
                   const Params p) {
  using C = Cfg<BN, CG, EPI>;
  constexpr int STAGES = C::STAGES;
  // CTA pair (CG=2): rank 0 (leader) issues the MMAs for both CTAs; both
  // CTAs load their halves by TMA and drain their own TMEM rows.
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const int t0 = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int tstep = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sOut = smem + STAGES * C::STAGE_BYTES;  // TMA-store staging (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + C::STORE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* colsum_smem = reinterpret_cast<float*>(sOut + C::STORE_BYTES + 256);
  float* bias_smem = reinterpret_cast<float*>(sOut + C::STORE_BYTES + 256 + C::COLSUM_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (p.probe && blockIdx.x == 0 && threadIdx.x == 0) {
    p.probe[0] = clock64();
    p.probe[1] = globaltimer_ns();
  }

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (C::F32OUT && p.phases > 1) {
      prefetch_tmap(&tmS.a1);
      prefetch_tmap(&tmS.a2);
      prefetch_tmap(&tmS.b1);
      prefetch_tmap(&tmS.b2);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(full + s), 1);
      mbar_init(smem_u32(empty + s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(tfull + a), 1);
      // one arrive per epilogue warp of the pair (the gate epilogue's two warp
      // groups take alternate tiles: 4 arrivals)
      mbar_init(smem_u32(tempty + a), (EPI == EPI_GATE ? 4 : 8) * CG);
    }
    fence_mbarrier_init();
  }
  if (warp == 2) {
    if (CG == 2) {
      tmem_alloc_pair(smem_u32(tmem_slot), C::TMEM_COLS);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  // programmatic dependent launch: barrier init, TMEM allocation and the
  // tensor-map prefetch above overlap the previous kernel's tail; nothing
  // below touches global memory before it completes
  pdl_wait();
  const uint32_t tmem_base = *tmem_slot;
  const int total = total_tiles<BN, CG>(p);
  const int row_off = (int)rank * BM;             // this CTA's rows inside a pair tile
  const int n_off = (int)rank * (BN / CG);        // this CTA's B rows (N) inside the tile

  if (warp == 0) {
#ifndef FMOE_TC_TMA_WARP
#define FMOE_TC_TMA_WARP 1  // the whole warp runs the producer loop, one elected lane issues
#endif
    if (FMOE_TC_TMA_WARP || lane == 0) {
      // ======================= TMA producer =======================
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0; it * tstep < total; ++it) {
        const int t = tile_at(p, it, t0, tstep);
        if (t >= total) continue;
        const Tile tl = decode<BN, CG, C::F32OUT>(p, t);
        const int brow = (p.mode == RAGGED_M) ? tl.g * p.b_group_rows : tl.kbeg;
        if (p.arrive_flags && tl.nkb > 0) wait_rows_arrived(p, tl.g, tl.m0 + row_off, lane);
        // gathered K-major A: this lane's 4 source rows of the tile, for all its k-blocks
        int4 grow = make_int4(0, 0, 0, 0);
        if (!A_MN && p.gather_rows && tl.nkb > 0)
          grow = __ldg(reinterpret_cast<const int4*>(p.gather_rows + tl.m0 + row_off) + lane);
        // split (bf16x6) passes: kb restarts at 0 for every pass, whose A / B
        // planes come from sel_a / sel_b
        int ph = 0;
        for (int kb = 0, kbt = 0; kbt < tl.nkb; ++kbt) {
          const CUtensorMap* mA = &tmA;
          const CUtensorMap* mB = &tmB;
          if constexpr (C::F32OUT) {
            if (tl.kpp != tl.nkb) {
              const uint32_t pa = (p.sel_a >> (4 * ph)) & 3u, pb = (p.sel_b >> (4 * ph)) & 3u;
              mA = pa == 0 ? &tmA : pa == 1 ? &tmS.a1 : &tmS.a2;
              mB = pb == 0 ? &tmB : pb == 1 ? &tmS.b1 : &tmS.b2;
            }
          }
          mbar_wait(smem_u32(empty + stage), phase ^ 1);
          const uint32_t fb = smem_u32(full + stage);
          if (rank == 0) {
            if (FMOE_TC_TMA_WARP)
              mbar_arrive_expect_tx_warp(fb, CG * C::STAGE_BYTES);
            else
              mbar_arrive_expect_tx(fb, CG * C::STAGE_BYTES);
          }
          const uint32_t a_dst = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_dst = smem_u32(sB + stage * C::B_BYTES);
          auto load = [&](uint32_t dst, const CUtensorMap* m, int c0, int c1) {
            if (FMOE_TC_TMA_WARP)
              tma_load_2d_warp<CG>(dst, m, fb, c0, c1);
            else if (CG == 2)
              tma_load_2d_pair(dst, m, fb, c0, c1);
            else
              tma_load_2d(dst, m, fb, c0, c1);
          };
          if (p.gather_rows) {
            // TMA gather4: K-major A (RAGGED_M) -- lane l brings tile rows 4l..4l+3
            // of this k-block; MN-major A (RAGGED_K) -- lane l brings K-rows
            // 4(l%16).. of the k-block into M box l/16
            int4 r;
            if (!A_MN) {
              r = grow;
            } else {
              r = __ldg(reinterpret_cast<const int4*>(p.gather_rows + tl.kbeg + kb * BK) + (lane & 15));
            }
            r.x = r.x < 0 ? p.gather_oob : r.x;
            r.y = r.y < 0 ? p.gather_oob : r.y;
            r.z = r.z < 0 ? p.gather_oob : r.z;
            r.w = r.w < 0 ? p.gather_oob : r.w;
            if (!A_MN)
              tma_gather4<CG>(a_dst + lane * 512, mA, fb, kb * BK, r);
            else
              tma_gather4<CG>(a_dst + (lane >> 4) * 8192 + (lane & 15) * 512, mA, fb,
                              tl.m0 + row_off + 64 * (lane >> 4), r);
          } else if (!A_MN) {
            load(a_dst, mA, kb * BK, tl.m0 + row_off);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              load(a_dst + j * 8192, mA, tl.m0 + row_off + 64 * j, tl.kbeg + kb * BK);
          }
          if (!B_MN) {
            load(b_dst, mB, kb * BK, brow + tl.n0 + n_off);
          } else {
#pragma unroll
            for (int j = 0; j < BN / CG / 64; ++j)
              load(b_dst + j * 8192, mB, tl.n0 + n_off + 64 * j, brow + kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (++kb == tl.kpp) {
            kb = 0;
            ++ph;
          }
        }
      }
    }
  } else if (warp == 1) {
#ifndef FMOE_TC_MMA_WARP
#define FMOE_TC_MMA_WARP 3  // 3: whole warp, one elected lane issues each k-block (4 MMAs + commit) in one asm; 1: per MMA; 0: lane 0 only
#endif
    if (rank == 0 && (FMOE_TC_MMA_WARP || lane == 0)) {
      // ======================= MMA issuer =========================
      constexpr uint32_t ID = idesc<BN, A_MN, B_MN, CG>();
      // descriptors: constant fields + the 16-byte start address (bits 0..13;
      // stage bases are 1 KiB aligned and below 228 KiB, so adding the k
      // offsets never carries out of the field)
      const uint64_t da0 = sdesc(smem_u32(sA), A_MN), db0 = sdesc(smem_u32(sB), B_MN);
      constexpr uint32_t KA = A_MN ? 2048 / 16 : 32 / 16, KB = B_MN ? 2048 / 16 : 32 / 16;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int it = 0; it * tstep < total; ++it) {
        const int t = tile_at(p, it, t0, tstep);
        if (t >= total) continue;
        const Tile tl = decode<BN, CG, C::F32OUT>(p, t);
        if (tl.nkb == 0) continue;
        mbar_wait(smem_u32(tempty + acc), acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          mbar_wait(smem_u32(full + stage), phase);
          tc_fence_after();
          const uint64_t ad = da0 + (uint64_t)(stage * (C::A_BYTES / 16));
          const uint64_t bd = db0 + (uint64_t)(stage * (C::B_BYTES / 16));
          if constexpr (FMOE_TC_MMA_WARP == 3) {
            static_assert(BK / 16 == 4, "k-block issue form assumes BK = 64");
            // 4 x K=16 and the commit that frees the stage (in both CTAs of a pair)
            tc_mma_kblock_warp<CG, KA, KB>(d_tmem, (uint32_t)ad, (uint32_t)(da0 >> 32), (uint32_t)bd,
                                           (uint32_t)(db0 >> 32), ID, kb != 0, smem_u32(empty + stage));
          } else {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              if (FMOE_TC_MMA_WARP)
                tc_mma_f16_warp<CG>(d_tmem, ad + k * KA, bd + k * KB, ID, (kb | k) != 0);
              else if (CG == 2)
                tc_mma_f16_pair(d_tmem, ad + k * KA, bd + k * KB, ID, (kb | k) != 0);
              else
                tc_mma_f16(d_tmem, ad + k * KA, bd + k * KB, ID, (kb | k) != 0);
            }
            if (FMOE_TC_MMA_WARP)
              tc_commit_warp<CG>(smem_u32(empty + stage));
            else if (CG == 2)
              tc_commit_pair(smem_u32(empty + stage));
            else
              tc_commit(smem_u32(empty + stage));
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (FMOE_TC_MMA_WARP)
          tc_commit_warp<CG>(smem_u32(tfull + acc));
        else if (CG == 2)
          tc_commit_pair(smem_u32(tfull + acc));
        else
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
    uint32_t sbuf = 0;  // TMA-store staging tile in use (per warp, double-buffered)
    for (int it = 0; it * tstep < total; ++it) {
      const int t = tile_at(p, it, t0, tstep);
      if (t >= total) continue;
      const Tile tl = decode<BN, CG, C::F32OUT>(p, t);
      const int row = tl.m0 + row_off + q * 32 + lane;
      if (tl.nkb == 0) {
        // empty K range (expert without tokens): gradient is exactly zero
        if constexpr (EPI == EPI_F32) {
          for (int c = c_lo; c < c_hi; ++c) {
            float z[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) z[i] = 0.f;
            if (tl.n0 + c * 32 < p.N) epi_store_chunk<BN, EPI>(p, tl, row, tl.n0 + c * 32, z);
          }
        }
        continue;
      }
      if constexpr (EPI == EPI_GATE) {
        // one thread owns a whole row of logits; the two warp groups drain
        // alternate tiles (accumulators) so two tiles' softmax run at once
        if ((ew >> 2) == acc) {
          mbar_wait(smem_u32(tfull + acc), acc_phase);
          tc_fence_after();
          const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
          const bool valid = row >= tl.lo && row < tl.hi;
          if constexpr (BN == 64)
            epi_gate64(p, tb, row, valid,
                       C::GATE_STAGE ? smem_u32(sOut) + (uint32_t)((ew * 32 + lane) * C::GATE_ROW_BYTES) : 0u);
          else
            epi_gate<BN>(p, tb, row, valid);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(tempty + acc));
        }
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        continue;
      }
      mbar_wait(smem_u32(tfull + acc), acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if constexpr (EPI == EPI_GATE) {
      } else if (EPI == EPI_GATE_DX && p.gk <= 2) {
        // scatter_backward gather fused with the gate d_x: the row's k source
        // positions are read once per tile and both source rows of a chunk are
        // requested before the TMEM load, so each chunk costs one memory latency.
        int pos0 = 0, pos1 = 0;
        if (row < p.M) {
          pos0 = __ldg(p.inverse_pos + (int64_t)row * p.gk);
          pos1 = p.gk > 1 ? __ldg(p.inverse_pos + (int64_t)row * p.gk + 1) : pos0;
        }
        for (int c = c_lo; c < c_hi; ++c) {
          const int c0 = tl.n0 + c * 32;
          if (c0 >= p.N) break;
          uint4 ga[4], gb[4];
          if (row < p.M) {
            const uint4* sa = reinterpret_cast<const uint4*>(p.gather_src + (int64_t)pos0 * p.N + c0);
            const uint4* sb = reinterpret_cast<const uint4*>(p.gather_src + (int64_t)pos1 * p.N + c0);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              ga[q4] = __ldg(sa + q4);
              gb[q4] = p.gk > 1 ? __ldg(sb + q4) : make_uint4(0, 0, 0, 0);
            }
          }
          float v[32];
          load_chunk(tbase + c * 32, v);
          if (row < p.M) {
            uint4 o[4];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const __nv_bfloat16* a8 = reinterpret_cast<const __nv_bfloat16*>(&ga[q4]);
              const __nv_bfloat16* b8 = reinterpret_cast<const __nv_bfloat16*>(&gb[q4]);
              float s[8];
#pragma unroll
              for (int i = 0; i < 8; ++i)  // (d_xs[pos0] + d_xs[pos1]) + gate d_x, slot order
                s[i] = (__bfloat162float(a8[i]) + __bfloat162float(b8[i])) + v[q4 * 8 + i];
              o[q4] = make_uint4(pack_bf16(s[0], s[1]), pack_bf16(s[2], s[3]), pack_bf16(s[4], s[5]),
                                 pack_bf16(s[6], s[7]));
            }
            uint4* out = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.C) + (int64_t)row * p.ldc + c0);
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) out[q4] = o[q4];
          }
        }
      } else if ((EPI == EPI_BF16 || EPI == EPI_MASK_BF16) && C::TMA_STORE && p.tma_out && (p.N % BN) == 0 &&
                 tl.m0 + BM * CG <= p.M && (EPI != EPI_MASK_BF16 || p.relu_bits) &&
                 (EPI != EPI_BF16 || p.relu || !p.relu_bits_out)) {
        // fast path (the expert GEMMs): compile-time transforms, see drain_bf16
        const uint32_t stage_base = smem_u32(sOut) + (uint32_t)(ew * C::NBUF * C::TILE_BYTES);
        const int out_row = tl.m0 + row_off + q * 32;
        float* bias_s = bias_smem + ew * (BN / 2);
        if constexpr (EPI == EPI_BF16) {
          if (p.bias) {  // this warp's 128 bias columns -> shared memory, once per tile
            const float4 bb = __ldg(reinterpret_cast<const float4*>(p.bias + (int64_t)tl.g * p.bias_group_stride +
                                                                   tl.n0 + c_lo * 32) + lane);
            reinterpret_cast<float4*>(bias_s)[lane] = bb;
            __syncwarp();
            if (p.relu)
              drain_bf16<BN, C::NBUF, true, true, false, false>(p, tl, &tmC, tbase, c_lo, row, out_row, stage_base,
                                                                sbuf, bias_s, colsum_smem, q, lane);
            else
              drain_bf16<BN, C::NBUF, true, false, false, false>(p, tl, &tmC, tbase, c_lo, row, out_row, stage_base,
                                                                 sbuf, bias_s, colsum_smem, q, lane);
          } else if (p.relu) {
            drain_bf16<BN, C::NBUF, false, true, false, false>(p, tl, &tmC, tbase, c_lo, row, out_row, stage_base,
                                                               sbuf, bias_s, colsum_smem, q, lane);
          } else {
            drain_bf16<BN, C::NBUF, false, false, false, false>(p, tl, &tmC, tbase, c_lo, row, out_row, stage_base,
                                                                sbuf, bias_s, colsum_smem, q, lane);
          }
        } else {
          if (p.colsum_part)
            drain_bf16<BN, C::NBUF, false, false, true, true>(p, tl, &tmC, tbase, c_lo, row, out_row, stage_base,
                                                              sbuf, bias_s, colsum_smem, q, lane);
          else
            drain_bf16<BN, C::NBUF, false, false, true, false>(p, tl, &tmC, tbase, c_lo, row, out_row, stage_base,
                                                               sbuf, bias_s, colsum_smem, q, lane);
        }
        if (p.colsum_part) {
          epi_bar();
          for (int col = ew * 32 + lane; col < BN; col += 256)
            p.colsum_part[(int64_t)((tl.m0 + row_off) / BM) * p.N + tl.n0 + col] =
                colsum_smem[col] + colsum_smem[BN + col] + colsum_smem[2 * BN + col] + colsum_smem[3 * BN + col];
          epi_bar();
        }
      } else {
        // Software-pipelined drain: the TMEM load of chunk i+1 is in flight
        // while chunk i is transformed and stored; relu bitmaps are fetched
        // up front.
        constexpr int CPW = NC / 2;
        uint32_t mbits[CPW];
#pragma unroll
        for (int i = 0; i < CPW; ++i) {
          const int c0 = tl.n0 + (c_lo + i) * 32;
          mbits[i] = (p.relu_bits && row < p.M && c0 < p.N)
                         ? __ldg(p.relu_bits + relu_bits_index(row, c0, p.N))
                         : 0u;
        }
        uint32_t buf[2][32];
        if (tl.n0 + c_lo * 32 < p.N) tmem_ld_issue(tbase + c_lo * 32, buf[0]);
#pragma unroll
        for (int i = 0; i < CPW; ++i) {
          const int c = c_lo + i;
          if (tl.n0 + c * 32 < p.N) {
            tmem_ld_wait(buf[i & 1]);
            if (i + 1 < CPW && tl.n0 + (c + 1) * 32 < p.N) tmem_ld_issue(tbase + (c + 1) * 32, buf[(i + 1) & 1]);
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(buf[i & 1][j]);
            if constexpr (EPI == EPI_F32X) {
              // fp32 expert outputs (FMOE_F32): dot product, then the rounded
              // bias add, relu keeping -0.0, strict > 0 mask -- the SIMT
              // kernel's order (gemm_simt.cu, matrix.cpp:128-153)
              const int c0 = tl.n0 + c * 32;
              if (row < p.M) {
                if (p.bias) {
                  const float* bb = p.bias + (int64_t)tl.g * p.bias_group_stride + c0;
#pragma unroll
                  for (int j = 0; j < 32; ++j)
                    if (c0 + j < p.N) v[j] = v[j] + __ldg(bb + j);
                }
                if (p.relu) {
#pragma unroll
                  for (int j = 0; j < 32; ++j) v[j] = v[j] < 0.f ? 0.f : v[j];
                }
                if (p.maskf) {
                  const float* mr = p.maskf + (int64_t)row * p.ldm + c0;
#pragma unroll
                  for (int j = 0; j < 32; ++j)
                    if (c0 + j < p.N) v[j] = __ldg(mr + j) > 0.f ? v[j] : 0.f;
                }
              }
            }
#ifdef FMOE_TC_F32_NOSTORE  // experiment: drain TMEM but store nothing (mainloop-bound speed)
            if constexpr (EPI == EPI_F32) continue;
#endif
            if constexpr (C::F32OUT) {
              if (p.tma_out) {
                // fp32 staging (rows >= M staged as zeros, clipped by the tensor map):
                //  64 B rows: two 16-column halves, 64B swizzle (16-byte chunk j of row r
                //             at r*64 + ((j ^ ((r >> 1) & 3)) << 4))
                // 128 B rows: one 32-column tile, 128B swizzle (chunk j at r*128 + ((j ^ (r & 7)) << 4))
                constexpr int RB = C::OUT_ROW_BYTES, HALVES = 128 / RB, CPR = RB / 16;
                const int out_row = (p.c_group_stride ? tl.g * (int)(p.c_group_stride / p.ldc) : 0) + tl.m0 +
                                    row_off + q * 32;
                const uint32_t r = (uint32_t)lane;
                const bool live = row < p.M;
#pragma unroll
                for (int hh = 0; hh < HALVES; ++hh) {
                  const uint32_t stage = smem_u32(sOut) + (uint32_t)((ew * C::NBUF + sbuf) * C::TILE_BYTES);
                  if (lane == 0) bulk_wait_read<C::NBUF - 1>();
                  __syncwarp();
#pragma unroll
                  for (int j = 0; j < CPR; ++j) {
                    const uint32_t sw = RB == 64 ? ((r >> 1) & 3u) : (r & 7u);
                    const uint32_t a = stage + r * RB + (((uint32_t)j ^ sw) << 4);
                    const float* src = v + hh * 16 + 4 * j;
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(live ? src[0] : 0.f),
                                 "f"(live ? src[1] : 0.f), "f"(live ? src[2] : 0.f), "f"(live ? src[3] : 0.f)
                                 : "memory");
                  }
                  fence_proxy_async_smem();
                  __syncwarp();
                  tma_store_commit_warp(&tmC, stage, tl.n0 + c * 32 + hh * 16, out_row);
                  sbuf = (sbuf + 1) % C::NBUF;
                }
                continue;
              }
            }
            uint32_t stage = 0;
            if (C::TMA_STORE && p.tma_out) {  // reuse a staging tile only once its last TMA store read it
              stage = smem_u32(sOut) + (uint32_t)((ew * C::NBUF + sbuf) * C::TILE_BYTES);
              if (lane == 0) bulk_wait_read<C::NBUF - 1>();
              __syncwarp();
            }
            epi_store_chunk<BN, EPI>(p, tl, row, tl.n0 + c * 32, v, mbits[i], stage);
            if (C::TMA_STORE && p.tma_out) {
              fence_proxy_async_smem();
              __syncwarp();
              // output row: group base (weight-gradient groups) + tile row + warp slab
              const int out_row = (p.c_group_stride ? tl.g * (int)(p.c_group_stride / p.ldc) : 0) + tl.m0 +
                                  row_off + q * 32;
              tma_store_commit_warp(&tmC, stage, tl.n0 + c * 32, out_row);
              sbuf = (sbuf + 1) % C::NBUF;
            }
            if (p.colsum_part) {  // column sums of the final fp32 values of this tile
              if (row >= p.M) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = 0.f;
              }
              colsum_smem[q * BN + c * 32 + lane] = warp_transpose_sum(v, lane);
            }
          }
        }
        if (p.colsum_part) {
          epi_bar();
          for (int col = ew * 32 + lane; col < BN; col += 256)
            if (tl.n0 + col < p.N)
              p.colsum_part[(int64_t)((tl.m0 + row_off) / BM) * p.N + tl.n0 + col] =
                  colsum_smem[col] + colsum_smem[BN + col] + colsum_smem[2 * BN + col] + colsum_smem[3 * BN + col];
          epi_bar();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // the leader's MMA waits for both CTAs' epilogues
        if (rank == 0)
          mbar_arrive(smem_u32(tempty + acc));
        else
          mbar_arrive_cluster(mapa_shared(smem_u32(tempty + acc), 0));
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if constexpr (C::TMA_STORE) {
      if (lane == 0) bulk_wait_all();  // outputs written before the CTA retires
    }
    if constexpr (C::GATE_STAGE) bulk_wait_all();  // every lane's row stores
  }
  tc_fence_before();
  if (CG == 2)
    cluster_sync_all();
  else
    __syncthreads();
  if (p.probe && blockIdx.x == 0 && threadIdx.x == 0) {
    p.probe[2] = clock64();
    p.probe[3] = globaltimer_ns();
  }
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
    else
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
                      uint32_t box_inner, uint32_t box_outer, int swizzle, bool f32) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  const CUresult r = encode_fn()(&m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                 2, const_cast<void*>(base), dims,
                                 strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(FMOE_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) +
                                   ") inner=" + std::to_string(inner) + " outer=" + std::to_string(outer));
  return m;
}

template <int BN, bool A_MN, bool B_MN, int CG, int EPI>
static void launch_t(Ctx* ctx, const CUtensorMap& ta, const CUtensorMap& tb, const Params& p,
                     int64_t max_tiles, const SplitMaps* split) {
  auto kern = tc_gemm_kernel<BN, A_MN, B_MN, CG, EPI>;
  using C = Cfg<BN, CG, EPI>;
  // Output tensor map for the TMA-store epilogue: 32x32 boxes matching the
  // staging tiles (bf16: [M][N], 64B swizzle; fp32: [groups*M][N], 128B swizzle).
  // fp32 group outputs use it only when no tile can cross into the next group.
  Params q = p;
  q.tma_out = 0;
  CUtensorMap tc_out = ta;
  if (C::TMA_STORE) {
    if (C::F32OUT) {
      const bool grouped = p.c_group_stride != 0;
      const bool ok = p.ldc == p.N && (p.N % 4) == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 &&
                      (!grouped || (p.M % (BM * CG) == 0 && p.c_group_stride == (int64_t)p.M * p.ldc));
      if (ok) {  // (TMA stores measured 1.3-1.5x faster than direct fp32 row stores)
        const int64_t rows = grouped ? (int64_t)p.M * p.n_groups : p.M;
        tc_out = make_tmap(p.C, p.N, rows, p.ldc * 4, C::OUT_ROW_BYTES / 4, 32, C::OUT_ROW_BYTES, true);
        q.tma_out = 1;
      }
    } else if (!p.route_out) {
      tc_out = make_tmap(p.C, p.N, p.M, p.ldc * 2, 32, 32, 64);
      q.tma_out = 1;
    }
  }
  static std::once_flag attr_once[64];  // function attributes are per device
  std::call_once(attr_once[ctx->device & 63], [&] {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  // persistent grid: one CTA (CG=1) or CTA pair (CG=2) per tile slot, <= #SMs
  int64_t grid = (p.grid_limit > 0 ? std::min<int64_t>(p.grid_limit, ctx->num_sms) : ctx->num_sms) / CG * CG;
  if (max_tiles * CG < grid) grid = max_tiles * CG;
  if (grid < CG) return;
  if (q.row_split) {
    if (CG != 1 || p.mode != RAGGED_M || p.tile_group || p.N > BN) shape_error("tc gemm: row_split needs one N tile");
    q.row_split = (int)grid;
    q.row_chunks = (int)((ceil_div((int64_t)p.M, grid) + BM - 1) / BM);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (q.phases > 1 && (!split || !C::F32OUT)) shape_error("tc gemm: split product without its planes / fp32 output");
  const SplitMaps sm = split ? *split : SplitMaps{ta, ta, tb, tb};
  CK(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc_out, sm, q));
  CK_LAUNCH(ctx);
}

// Only the (tile, operand-major, CTA-group, epilogue) combinations the MoE layer uses
// are instantiated; each kernel carries exactly one epilogue.
void launch(Ctx* ctx, int bn, bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb,
            const Params& p, int64_t max_tiles, int cg, const SplitMaps* split) {
#define FMOE_TC_CASE(BN_, AM, BM_, CG_, EPI_)                                   \
  if (bn == BN_ && a_mn == AM && b_mn == BM_ && cg == CG_ && p.epi == EPI_) {   \
    launch_t<BN_, AM, BM_, CG_, EPI_>(ctx, ta, tb, p, max_tiles, split);        \
    return;                                                                     \
  }
  // expert pool, CTA pairs (256-row aligned plans)
  FMOE_TC_CASE(256, false, true, 2, EPI_BF16)        // fc1 (+bias, relu, relu bitmap), fc2 (+bias)
  FMOE_TC_CASE(256, false, false, 2, EPI_MASK_BF16)  // dgrad fc2 (+relu mask, d_b1 column sums)
  FMOE_TC_CASE(256, false, false, 2, EPI_BF16)       // dgrad fc1
  FMOE_TC_CASE(256, true, true, 2, EPI_F32)          // weight gradients
  // expert pool, single CTAs (128-row aligned plans)
  FMOE_TC_CASE(256, false, true, 1, EPI_BF16)
  FMOE_TC_CASE(256, false, false, 1, EPI_MASK_BF16)
  FMOE_TC_CASE(256, false, false, 1, EPI_BF16)
  FMOE_TC_CASE(256, true, true, 1, EPI_F32)
  // FMOE_F32 expert GEMMs on the tensor cores (bf16x6, fp32 outputs; the
  // weight gradients and gate products reuse the EPI_F32 instances)
  FMOE_TC_CASE(256, false, true, 2, EPI_F32X)        // fc1 (+bias, relu), fc2 (+bias)
  FMOE_TC_CASE(256, false, false, 2, EPI_F32X)       // dgrad fc2 (*mask), dgrad fc1
  FMOE_TC_CASE(256, false, true, 1, EPI_F32X)
  FMOE_TC_CASE(256, false, false, 1, EPI_F32X)
  // gate
  FMOE_TC_CASE(64, false, true, 1, EPI_GATE)         // logits + softmax + top-k, E <= 64
  FMOE_TC_CASE(128, false, true, 1, EPI_GATE)        // E <= 128
  FMOE_TC_CASE(256, false, true, 1, EPI_GATE)        // E <= 256
  FMOE_TC_CASE(256, false, true, 1, EPI_F32)         // logits only, E > 256
  FMOE_TC_CASE(256, false, false, 1, EPI_GATE_DX)    // gate d_x + scatter_backward
  FMOE_TC_CASE(64, false, true, 1, EPI_F32)          // FMOE_F32 gate logits, E <= 64
  FMOE_TC_CASE(128, false, true, 1, EPI_F32)         // FMOE_F32 gate logits, E <= 128
  FMOE_TC_CASE(256, false, false, 1, EPI_F32)        // FMOE_F32 gate d_x
  FMOE_TC_CASE(64, true, true, 1, EPI_F32)           // gate d_wg split-K partials
  FMOE_TC_CASE(128, true, true, 1, EPI_F32)
#undef FMOE_TC_CASE
  shape_error("tc gemm: unsupported tile configuration");
}

}  // namespace tc
}  // namespace fmoe_b200
