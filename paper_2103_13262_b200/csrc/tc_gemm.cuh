// tc_gemm.cuh -- the grouped tcgen05/TMEM/TMA GEMM for sm_100a (bf16 in,
// fp32 accumulate), shared by every dense contraction of the MoE layer:
//
//   gate logits + softmax + top-k   x[N,d] * Wg[d,E]                 (gate.cpp:30-33)
//   expert fc1 + bias + relu        xs[rows,d] * W1_e[d,h]           (expert.cpp:30-31)
//   expert fc2 + bias               H[rows,h] * W2_e[h,d]            (expert.cpp:32)
//   dgrad fc2 * relu mask           dYs[rows,d] * W2_e^T             (expert.cpp:47-48)
//   dgrad fc1                       dPre[rows,h] * W1_e^T            (expert.cpp:55)
//   wgrad fc2 / fc1                 H_e^T dYs_e, xs_e^T dPre_e       (expert.cpp:42,50)
//   gate dx + scatter_backward      dz[N,E] * Wg^T + sum_j d_xs[pos] (gate.cpp:63, dispatch.cpp:80-95)
//   gate dWg (split-K partials)     x^T dz                           (gate.cpp:62)
//
// Design (SURVEY §7, B200 guide "Canonical Blackwell GEMM"):
//   * persistent: grid = #SMs, static round-robin over tiles; the tile list
//     is derived on device from the dispatch plan (no host sync);
//   * warp-specialised, 384 threads: warp0 = TMA producer, warp1 = MMA issuer
//     (one elected lane, tcgen05.mma.cta_group::1.kind::f16 M=128, N=BN, K=16),
//     warp2 = TMEM allocator, warps 4..11 = epilogue (one TMEM lane = one row,
//     two warps per lane quarter splitting the tile's columns);
//   * smem ring of STAGES x (A 128x64 + B BNx64) bf16, 128B-swizzled TMA
//     boxes, full/empty mbarriers; 2 TMEM accumulators (2*BN fp32 columns)
//     so the epilogue of tile i overlaps the MMAs of tile i+1;
//   * operands may be K-major or MN-major (weights are used in their stored
//     reference layout W1[d,h] / W2[h,d] for both the forward and the
//     transposed backward products -- no materialised transposes);
//   * two tile spaces: RAGGED_M (128-row tiles of the 128-aligned expanded
//     buffer, each tile owned by one expert) and RAGGED_K (per-group K row
//     ranges: the weight gradients, whose contraction runs over tokens).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace fmoe_b200 {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = one 128-byte swizzle row
constexpr int NUM_THREADS = 384;  // 4 control warps + 8 epilogue warps

enum Mode : int { RAGGED_M = 0, RAGGED_K = 1 };
enum Epi : int {
  EPI_BF16 = 0,       // C = bf16(acc [+ bias] [relu])
  EPI_MASK_BF16 = 1,  // C = bf16(acc * (mask > 0))           dgrad fc2 (relu_backward, strict >)
  EPI_F32 = 2,        // C = acc (fp32)                         weight gradients
  EPI_GATE = 3,       // softmax + top-k over the row           gate forward
  EPI_GATE_DX = 4,    // C = bf16(sum_j d_xs[pos(i,j)] + acc)   scatter_backward + gate d_x
  EPI_F32X = 5,       // C = acc [+ bias] [relu] [* (maskf > 0)] (fp32)   FMOE_F32 expert GEMMs
};

// FMOE_F32 on the tensor cores ("bf16x6"): every fp32 operand is stored as
// three bf16 planes, a0 = bf16(a), a1 = bf16(a - a0), a2 = bf16(a - a0 - a1)
// (each difference exact in fp32; a = a0 + a1 + a2 + r, |r| <= 2^-24 |a|), and
// a product runs as six bf16 passes over the whole K range into one fp32 TMEM
// accumulator -- a0*b2, a2*b0, a1*b1, a0*b1, a1*b0, then a0*b0 (small terms
// first).  The omitted a1*b2, a2*b1, a2*b2 and residual terms are <= ~2^-24 of
// each product: fp32-class accuracy at the cost of 6 bf16 GEMMs.  (Two planes
// and three passes leave ~1e-5 relative error per product -- enough to flip
// relu masks near zero and miss SURVEY 8(c)'s 1e-4 gradient bound, measured.)
// Params.phases = 6 with sel_a / sel_b (plane of each pass, one nibble per
// pass) selects it; planes 1, 2 come in through SplitMaps.
constexpr int SPLIT_PASSES = 6;
constexpr uint32_t SPLIT_SEL_A = 0x010120u;  // passes 0..5 (low nibble first): 0 2 1 0 1 0
constexpr uint32_t SPLIT_SEL_B = 0x001102u;  //                                  2 0 1 1 0 0

struct Params {
  int mode;
  int M, N, K;               // RAGGED_M: M = rows (tensor extent), K = contraction
  int n_groups;              // RAGGED_K: number of groups
  const int* tile_group;     // RAGGED_M: group of each 128-row tile (NULL: all group 0)
  const int* n_mtiles;       // RAGGED_M: device count of valid row tiles (NULL: ceil(M/128))
  const int* k_offsets;      // RAGGED_K: [G+1] K-row range of each group (multiples of 64)
  int k_split;               // RAGGED_K without k_offsets: group g = rows [g*k_split, min(K, (g+1)*k_split))
  // RAGGED_K (optional): groups in decreasing K-length; tiles are then dealt
  // to the persistent CTAs heaviest first in a snake (boustrophedon) order so
  // skewed expert sizes (Zipf routing) stay balanced across SMs
  const int* group_order;
  int b_group_rows;          // RAGGED_M: rows of the 2-D B tensor per group
  // epilogue
  int epi;
  void* C;
  int64_t ldc;
  int64_t c_group_stride;    // RAGGED_K: elements between groups' outputs
  const float* bias;         // [G][N] fp32 or NULL
  int64_t bias_group_stride;
  int relu;
  const __nv_bfloat16* mask; // EPI_MASK_BF16: [rows][ldm]
  int64_t ldm;
  // EPI_GATE
  float* scores;             // [M][N]
  int* topk_idx;             // [M][topk]
  float* topk_val;
  int topk;                  // <= 8 fused; 0 = scores only
  // EPI_GATE_DX
  const __nv_bfloat16* gather_src;  // d_xs [rows][N]
  const int* inverse_pos;           // [M][gk]
  int gk;
  // optional fused column sums of the epilogue values (RAGGED_M bf16
  // epilogues): colsum_part[m_tile][N] = sum over the tile's 128 rows, fp32
  // (bias gradients without re-reading the activation; reduced per expert
  // by reduce_tile_partials in a fixed order -> deterministic)
  float* colsum_part;
  // relu bitmaps [rows][N/32]: written by the fc1 epilogue (bit = value > 0),
  // read by the dgrad-fc2 epilogue instead of the bf16 activations (64 MiB
  // instead of 1 GiB at cfg2)
  uint32_t* relu_bits_out;
  const uint32_t* relu_bits;
  // Expert parallelism, overlapped exchange (RAGGED_M A operand arriving from
  // the peers while the GEMM runs): before loading the A rows of a tile the
  // producer waits until every source rank whose chunk (expert g, source s)
  // intersects those rows has published it -- arrive_flags[g*W + s] reaches
  // arrive_epoch (written by the sender with st.release.sys after its rows,
  // ep_push_kernel) -- so tiles start as their rows land instead of after the
  // whole exchange.  arrive_rt = [start[el*W], rows[el*W]] of every chunk.
  const uint32_t* arrive_flags;
  uint32_t arrive_epoch;
  const int32_t* arrive_rt;
  int arrive_W, arrive_C;    // world, chunks (el * W)
  // RAGGED_M (optional): order in which the (pair) row tiles are dealt --
  // expected arrival order of their rows under the overlapped exchange
  const int* mtile_order;
  // persistent grid cap (0: all SMs); SMs left free run the concurrent push
  int grid_limit;
  // A operand gathered by TMA tile::gather4 (the single-GPU bf16 layer: no
  // scatter pass): row r of the expanded layout is row
  // gather_rows[r] of the A tensor map's matrix (x, box {64, 1}); -1 = padding
  // (read as zeros).  RAGGED_M with a K-major A (fc1): each producer lane
  // gathers 4 of the tile's rows per k-block; RAGGED_K with an MN-major A (the
  // fc1 weight gradient, A = x^T): the k-block's 64 K-rows, 4 per lane.
  const int* gather_rows;
  int gather_oob;  // a row coordinate past the end of x
  // RAGGED_M without tile_group and N <= BN (the gate): nonzero asks launch()
  // for balanced contiguous row ranges, one per persistent CTA -- slot s owns
  // rows [s*M/S, (s+1)*M/S) and walks them in 128-row chunks, the last chunk
  // shifted back to end at the range end (its overlap recomputed, stored
  // once) -- instead of whole 128-row tiles dealt round-robin, whose
  // ceil(M/128/S) vs floor(...) split leaves SMs idle for a whole tile.
  // launch() replaces it with S and sets row_chunks.
  int row_split, row_chunks;
  // optional clock probe (Ctx::d_probe slot): CTA 0 writes (clock64,
  // globaltimer) at its start and end
  unsigned long long* probe;
  int tma_out;  // set by launch(): outputs leave through TMA stores
  // bf16x6 (FMOE_F32, fp32-output epilogues only): 1 = plain bf16 GEMM
  // (default, 0 reads as 1); > 1 = that many passes over the whole K range,
  // pass i contracting plane (sel_a >> 4i) & 3 of A with plane (sel_b >> 4i) & 3
  // of B
  int phases;
  uint32_t sel_a, sel_b;
  // EPI_F32X: fp32 relu-backward operand [rows][ldm] (strict > 0; bias and
  // relu as for EPI_BF16)
  const float* maskf;
  // Expert parallelism over peer memory (EPI_BF16, RAGGED_M): every output row
  // is stored straight into the rank that sent it (fused global_gather,
  // collectives.cpp:205-265).  Row q of expert block g from source s -- rows
  // [route_start[g*W+s], + route_rows[g*W+s]) -- lands at row
  // route_dst[g*W+s] + (q - route_start[g*W+s]) of route_out[s]; pad rows are
  // dropped.
  void* const* route_out;
  const int32_t* route_start;
  const int32_t* route_rows;
  const int32_t* route_dst;
  int route_world;
};

// Host: build a 2-D bf16 tensor map over a row-major [outer, inner] matrix
// with a (box_inner x box_outer) box, 128B swizzle, zero OOB fill.
CUtensorMap make_tmap(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                      uint32_t box_inner, uint32_t box_outer, int swizzle = 128, bool f32 = false);

// Host: launch.  a_mn / b_mn select MN-major operands; bn in {64,128,256};
// cg = 2 runs CTA pairs (tcgen05 cta_group::2, 256-row tiles; RAGGED_M then
// needs 256-row aligned expert blocks).  max_tiles counts (pair) tiles.
// Planes 1 and 2 of the operands of a split (bf16x6) product.
struct SplitMaps {
  CUtensorMap a1, a2, b1, b2;
};
void launch(Ctx* ctx, int bn, bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb,
            const Params& p, int64_t max_tiles, int cg = 1, const SplitMaps* split = nullptr);

}  // namespace tc
}  // namespace fmoe_b200
