// plan.cuh -- internal interfaces of the device dispatch plan and permutes.
#pragma once

#include "common.cuh"

namespace fmoe_b200 {

int64_t plan_capacity(int64_t n_b, int64_t k, int64_t n_experts, int64_t align);
int64_t plan_scratch_bytes(int64_t n_b, int64_t k, int64_t n_experts);
void plan_build(Ctx* ctx, const int32_t* topk_idx, const fmoe_plan& p);

// permutes (permute.cu); T = element type, S = score type
struct ScatterRoute;
// route (optional, expert parallelism over peer memory): write slot rows into
// the expert ranks' receive buffers instead of xs (see peer.cuh).
void scatter(Ctx* ctx, fmoe_dtype t, const void* x, int64_t d, const fmoe_plan& p, void* xs,
             const ScatterRoute* route = nullptr);
void gather_combine(Ctx* ctx, fmoe_dtype t, const void* ys, int64_t d, const fmoe_plan& p,
                    const void* w, void* y);
// scatter_backward; d_x[i] = sum_j d_xs[pos(i,j)] (+ addend[i], the gate's d_x).
void scatter_bwd(Ctx* ctx, fmoe_dtype t, const void* d_xs, int64_t d, const fmoe_plan& p, void* dx,
                 const void* addend = nullptr);
// gather_combine_backward; when dz != nullptr (bf16 layer path) the gate's
// softmax-Jacobian d_logits row is produced in the same pass (bf16, [n_b, E]).
void gather_combine_bwd(Ctx* ctx, fmoe_dtype t, const void* dy, const void* ys, int64_t d,
                        const fmoe_plan& p, const void* w, void* d_ys, void* d_w,
                        const void* scores, const int32_t* topk_idx, __nv_bfloat16* dz,
                        const ScatterRoute* route = nullptr);
// order[r] = the group of rank r by decreasing row count (ties by index).
void order_groups_desc(Ctx* ctx, const int32_t* offsets, int64_t groups, int32_t* order);
// Bias gradients: out[g][c] = sum over the rows of block g (ascending) of src[row][c].
void block_colsum(Ctx* ctx, fmoe_dtype t, const void* src, int64_t n_cols, const int32_t* offsets,
                  const int32_t* counts, int64_t n_blocks, void* out);

// bf16 bias gradients over 128-row tiles of an aligned layout:
// part[t][c] = sum of tile t's rows; out[e][c] = sum of expert e's tile partials.
void tile_colsum(Ctx* ctx, const __nv_bfloat16* src, int64_t n_cols, const int32_t* n_tiles,
                 int64_t max_tiles, float* part);
// (part2 / n_cols2 / out2: a second partial set over the same tiles, same launch)
void reduce_tile_partials(Ctx* ctx, const float* part, int64_t n_cols, const int32_t* offsets,
                          int64_t n_blocks, float* out, const float* part2 = nullptr, int64_t n_cols2 = 0,
                          float* out2 = nullptr);

// gate (gate.cu)
void gate_softmax_topk(Ctx* ctx, fmoe_dtype t, const void* logits, int64_t n, int64_t e, int64_t k,
                       void* scores, int32_t* idx, void* vals, bool scores_ready);
void gate_dlogits(Ctx* ctx, fmoe_dtype t, const void* scores, const int32_t* idx, const void* d_topk,
                  int64_t n, int64_t e, int64_t k, void* dz);
// deterministic reduction of split-K partials: out[i] = sum_s part[s][i]
void reduce_splits(Ctx* ctx, const float* part, int64_t n_splits, int64_t n, float* out);

}  // namespace fmoe_b200
