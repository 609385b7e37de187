// plan.cu -- build_plan on device (dispatch.cpp:10-47): expert histogram,
// exclusive scan (optionally 128-row aligned blocks) and the stable
// (row, slot) position of every selection, without a global sort.
//
//   K2a plan_hist  : one warp per chunk of 512 flat selections f = i*k + j;
//                    __match_any_sync-aggregated shared-memory histogram
//                    -> chunk_hist[e][c] (expert-major); out-of-range index
//                    -> error flag.
//   K2b plan_colscan: one warp per expert, all in parallel: counts[e] and,
//                    in place, rel[e][c] = sum_{c'<c} hist[e][c'].
//   K2c plan_offsets: one CTA: aligned exclusive scan of counts -> offsets;
//                    padding rows (src_row = -1); 128-row tile -> expert table.
//   K2d plan_rank  : re-walks each chunk in order; within a 32-wide step the
//                    rank of a lane among equal experts is popc(match & lt),
//                    across steps a per-warp shared counter carries it.  Hence
//                    pos(f) = offsets[e] + rel[e][c] + #{f' < f in chunk c : idx[f'] = e},
//                    exactly the reference's row-major fill order.
// Integer-exact by construction; checked bit-for-bit against the oracle.
#include <mutex>

#include "common.cuh"
#include "plan.cuh"

namespace fmoe_b200 {

constexpr int kChunk = 512;       // selections per warp chunk
constexpr int kWarpsPerCta = 4;

// chunk_hist is expert-major ([E][n_chunks]) so plan_colscan reads each
// expert's column contiguously.
__global__ void plan_hist(const int32_t* __restrict__ idx, int64_t nk, int n_experts, int n_chunks,
                          int32_t* __restrict__ chunk_hist, int* __restrict__ err) {
  pdl_wait();
  extern __shared__ int32_t sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* hist = sh + w * n_experts;
  for (int e = lane; e < n_experts; e += 32) hist[e] = 0;
  __syncwarp();
  const int64_t chunk = (int64_t)blockIdx.x * kWarpsPerCta + w;
  const int64_t f0 = chunk * kChunk;
  if (f0 < nk) {
    // all of the lane's keys in flight at once (the loop below is latency-bound otherwise)
    int keys[kChunk / 32];
#pragma unroll
    for (int t = 0; t < kChunk / 32; ++t) {
      const int64_t f = f0 + t * 32 + lane;
      keys[t] = f < nk ? __ldg(idx + f) : -1;
    }
#pragma unroll
    for (int t = 0; t < kChunk / 32; ++t) {
      const int64_t f = f0 + t * 32 + lane;
      int key = keys[t];
      if (f < nk && (key < 0 || key >= n_experts)) {
        atomicExch(err, 1);
        key = -1;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      if (key >= 0 && (__ffs(peers) - 1) == lane) hist[key] += __popc(peers);
      __syncwarp();
    }
    for (int e = lane; e < n_experts; e += 32) chunk_hist[(int64_t)e * n_chunks + chunk] = hist[e];
  }
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// K2b: one warp per expert, all experts in parallel: counts[e] and, in
// place, each chunk's exclusive prefix inside its expert column (chunk order).
__global__ void plan_colscan(int32_t* __restrict__ chunk_hist, int n_chunks, int n_experts,
                             int32_t* __restrict__ counts) {
  pdl_wait();
  const int e = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= n_experts) return;
  int32_t* col = chunk_hist + (int64_t)e * n_chunks;
  constexpr int R = 8;  // consecutive chunks per lane per pass
  int carry = 0;
  for (int c0 = 0; c0 < n_chunks; c0 += 32 * R) {
    const int base = c0 + lane * R;
    int v[R];
#pragma unroll
    for (int u = 0; u < R; ++u) v[u] = base + u < n_chunks ? col[base + u] : 0;
    int loc = 0;
#pragma unroll
    for (int u = 0; u < R; ++u) loc += v[u];
    const int incl = warp_incl_scan(loc, lane);
    int b = carry + incl - loc;
#pragma unroll
    for (int u = 0; u < R; ++u) {
      if (base + u < n_chunks) col[base + u] = b;
      b += v[u];
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) counts[e] = carry;
}

// K2c: one CTA: aligned exclusive scan of the counts -> offsets; padding rows
// (src_row = -1); 128-row tile -> expert table.
__global__ void plan_offsets(const int32_t* __restrict__ counts, int n_experts, int align,
                             int32_t* __restrict__ offsets, int32_t* __restrict__ src_row,
                             int32_t* __restrict__ tile_expert, int32_t* __restrict__ n_tiles) {
  pdl_wait();
  extern __shared__ int32_t sh[];  // [n_experts] aligned counts -> exclusive offsets
  int32_t* acnt = sh;
  __shared__ int32_t warp_tot[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  for (int e = threadIdx.x; e < n_experts; e += blockDim.x) {
    const int c = counts[e];
    acnt[e] = (c + align - 1) / align * align;
  }
  __syncthreads();
  const int per = (n_experts + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(lo + per, n_experts);
  int run = 0;
  for (int e = lo; e < hi; ++e) run += acnt[e];
  const int incl = warp_incl_scan(run, lane);
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = lane < nwarps ? warp_tot[lane] : 0;
    v = warp_incl_scan(v, lane);
    warp_tot[lane] = v;
  }
  __syncthreads();
  int base = incl - run + (warp > 0 ? warp_tot[warp - 1] : 0);
  for (int e = lo; e < hi; ++e) {
    const int a = acnt[e];
    acnt[e] = base;
    offsets[e] = base;
    base += a;
  }
  if (threadIdx.x == blockDim.x - 1) {
    offsets[n_experts] = base;
    if (n_tiles) n_tiles[0] = base / 128;
  }
  __syncthreads();
  for (int e = warp; e < n_experts; e += nwarps) {
    const int off = acnt[e], cnt = counts[e];
    const int end = off + (cnt + align - 1) / align * align;
    for (int r = off + cnt + lane; r < end; r += 32) src_row[r] = -1;
    if (tile_expert)
      for (int t = off / 128 + lane; t < end / 128; t += 32) tile_expert[t] = e;
  }
}

__global__ void plan_rank(const int32_t* __restrict__ idx, int64_t nk, int k, int n_experts, int n_chunks,
                          const int32_t* __restrict__ chunk_base, const int32_t* __restrict__ offsets,
                          int32_t* __restrict__ src_row,
                          int32_t* __restrict__ slot, int32_t* __restrict__ inverse_pos) {
  pdl_wait();
  extern __shared__ int32_t sh[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* run = sh + w * n_experts;
  for (int e = lane; e < n_experts; e += 32) run[e] = 0;
  __syncwarp();
  const int64_t chunk = (int64_t)blockIdx.x * kWarpsPerCta + w;
  const int64_t f0 = chunk * kChunk;
  if (f0 >= nk) return;
  const int32_t* base = chunk_base + chunk;  // base[key * n_chunks]
  const unsigned lt = (1u << lane) - 1u;
  int keys[kChunk / 32];
#pragma unroll
  for (int t = 0; t < kChunk / 32; ++t) {
    const int64_t f = f0 + t * 32 + lane;
    keys[t] = f < nk ? __ldg(idx + f) : -1;
  }
  int bases[kChunk / 32];  // the chunk base of every key, loads in flight together
#pragma unroll
  for (int t = 0; t < kChunk / 32; ++t) {
    if (keys[t] >= n_experts || keys[t] < 0) keys[t] = -1;
    bases[t] = keys[t] >= 0 ? __ldg(base + (int64_t)keys[t] * n_chunks) + __ldg(offsets + keys[t]) : 0;
  }
#pragma unroll
  for (int t = 0; t < kChunk / 32; ++t) {
    const int64_t f = f0 + t * 32 + lane;
    const int key = keys[t];
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    int before = 0;
    if (key >= 0) before = run[key];
    __syncwarp();
    if (key < 0 && f < nk) inverse_pos[f] = 0;  // flagged by plan_hist; keep later reads in bounds
    if (key >= 0) {
      const int pos = bases[t] + before + __popc(peers & lt);
      const int i = (int)(f / k);
      src_row[pos] = i;
      slot[pos] = (int)(f - (int64_t)i * k);
      inverse_pos[f] = pos;
      if ((__ffs(peers) - 1) == lane) run[key] = before + __popc(peers);
    }
    __syncwarp();
  }
}

int64_t plan_capacity(int64_t n_b, int64_t k, int64_t n_experts, int64_t align) {
  const int64_t nk = n_b * k;
  if (align <= 1) return nk;
  return ceil_div(nk + n_experts * (align - 1), align) * align;
}

int64_t plan_scratch_bytes(int64_t n_b, int64_t k, int64_t n_experts) {
  const int64_t chunks = ceil_div(n_b * k, kChunk) + 1;
  return chunks * n_experts * 4 + 256;
}

void plan_build(Ctx* ctx, const int32_t* topk_idx, const fmoe_plan& p) {
  const int64_t nk = p.n_b * p.k;
  const int E = (int)p.n_experts;
  if (E < 1) shape_error("build_plan: need at least one expert");
  if ((int64_t)E * kWarpsPerCta * 4 > 200 * 1024)
    shape_error("build_plan: too many experts for the device plan (max 12800)");
  if (p.align != 1 && p.align != 128 && p.align != 256)
    shape_error("build_plan: align must be 1, 128 or 256");
  if (nk > (int64_t)1 << 30) shape_error("build_plan: n_b*k too large");
  const int64_t chunks = ceil_div(nk, kChunk);
  int32_t* chunk_hist = reinterpret_cast<int32_t*>(p.scratch);
  const size_t smem = (size_t)E * kWarpsPerCta * 4;
  static std::once_flag attr_once[64];  // function attributes are per device
  std::call_once(attr_once[ctx->device & 63], [] {
    CK(cudaFuncSetAttribute(plan_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(plan_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(plan_offsets, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  const unsigned grid = (unsigned)std::max<int64_t>(1, ceil_div(chunks, kWarpsPerCta));
  if (nk > 0) {
    CK(launch_pdl(plan_hist, dim3(grid), dim3(32 * kWarpsPerCta), smem, ctx->stream, topk_idx, nk, E, (int)chunks,
                  chunk_hist, ctx->d_error));
    CK_LAUNCH(ctx);
  }
  if (nk > 0) {
    CK(launch_pdl(plan_colscan, dim3((unsigned)ceil_div((int64_t)E * 32, 256)), dim3(256), 0, ctx->stream, chunk_hist,
                  (int)chunks, E, p.counts));
    CK_LAUNCH(ctx);
  } else {
    CK(cudaMemsetAsync(p.counts, 0, (size_t)E * 4, ctx->stream));
  }
  CK(launch_pdl(plan_offsets, dim3(1), dim3(1024), (size_t)E * 4, ctx->stream, p.counts, E, (int)p.align, p.offsets,
                p.src_row, p.align % 128 == 0 ? p.tile_expert : (int32_t*)nullptr, p.n_tiles));
  CK_LAUNCH(ctx);
  if (nk > 0) {
    CK(launch_pdl(plan_rank, dim3(grid), dim3(32 * kWarpsPerCta), smem, ctx->stream, topk_idx, nk, (int)p.k, E,
                  (int)chunks, (const int32_t*)chunk_hist, (const int32_t*)p.offsets, p.src_row, p.slot,
                  p.inverse_pos));
    CK_LAUNCH(ctx);
  }
}

}  // namespace fmoe_b200
