// Probe of TMA tile::gather4 semantics on sm_100a (run once on the GPU box):
//  1. one CTA: 32 lanes each gather 4 rows (64 bf16 columns, SWIZZLE_128B) of
//     x[n][d] into a 128-row K-major tile; rows >= n must read as zero; the
//     smem layout must be the tile-load layout (16-byte chunk j of row r at
//     ((j ^ (r & 7)) << 4)).
//  2. a CTA pair (.cta_group::2): both CTAs gather their 128 rows into their own
//     shared memory and complete on the LEADER's mbarrier (peer bit cleared).
//  3. MN-major: gather 4 K-rows of 64 M-elements into an MN-major SW128 tile.
// nvcc -gencode arch=compute_100a,code=sm_100a -o gather_probe tma_gather_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
               :: "r"(dst), "l"((uint64_t)m), "r"(bar), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}
__device__ __forceinline__ void gather4_pair(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
               :: "r"(dst), "l"((uint64_t)m), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(b), "r"(c) : "memory"); }
__device__ __forceinline__ void expect_tx(uint32_t b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ bool try_wait(uint32_t b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(b), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// K-major: out[cta][128][64] = unswizzled tile; rows idx[cta*128 + i]
template <int PAIR>
__global__ void __cluster_dims__(PAIR ? 2 : 1, 1, 1) probe_kmajor(const __grid_constant__ CUtensorMap tm, const int* idx, int col0, __nv_bfloat16* out, int* status) {
  __shared__ __align__(1024) uint8_t tile[128 * 128];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x;
  const uint32_t rank = PAIR ? ctarank() : 0;
  if (lane == 0) { mbar_init(su32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (PAIR) cluster_sync(); else __syncthreads();
  if (lane == 0 && rank == 0) expect_tx(su32(&bar), (PAIR ? 2 : 1) * 128 * 128);
  if (PAIR) cluster_sync(); else __syncthreads();
  const int* r = idx + rank * 128 + 4 * lane;
  if (PAIR) gather4_pair(su32(tile) + lane * 512, &tm, su32(&bar), col0, r[0], r[1], r[2], r[3]);
  else gather4(su32(tile) + lane * 512, &tm, su32(&bar), col0, r[0], r[1], r[2], r[3]);
  if (rank == 0) {
    long n = 0;
    while (!try_wait(su32(&bar), 0)) if (++n > 200000000) { status[0] = 1; break; }
  }
  if (PAIR) cluster_sync(); else __syncthreads();
  for (int i = lane; i < 128 * 64; i += 32) {
    const int row = i / 64, c = i % 64, chunk = c / 8, w = c % 8;
    const int off = row * 128 + (((chunk ^ (row & 7)) << 4)) + w * 2;
    out[(size_t)rank * 128 * 64 + i] = *reinterpret_cast<const __nv_bfloat16*>(tile + off);
  }
}

// MN-major: gather K-rows idx[0..63] of x columns m0..m0+63 into a 64(M) x 64(K) SW128 MN-major box:
// K-row k at k*128 bytes, 16-byte chunk j (elements 8j..8j+7 of M) at ((j ^ (k & 7)) << 4)
__global__ void probe_mnmajor(const __grid_constant__ CUtensorMap tm, const int* idx, int m0, __nv_bfloat16* out, int* status) {
  __shared__ __align__(1024) uint8_t tile[64 * 128];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x;
  if (lane == 0) { mbar_init(su32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (lane == 0) expect_tx(su32(&bar), 64 * 128);
  __syncthreads();
  if (lane < 16) {
    const int* r = idx + 4 * lane;
    gather4(su32(tile) + lane * 512, &tm, su32(&bar), m0, r[0], r[1], r[2], r[3]);
  }
  long n = 0;
  while (!try_wait(su32(&bar), 0)) if (++n > 200000000) { status[1] = 1; break; }
  __syncthreads();
  for (int i = lane; i < 64 * 64; i += 32) {
    const int k = i / 64, m = i % 64, chunk = m / 8, w = m % 8;
    out[i] = *reinterpret_cast<const __nv_bfloat16*>(tile + k * 128 + ((chunk ^ (k & 7)) << 4) + w * 2);
  }
}

int main() {
  const int n = 1000, d = 256;
  std::vector<__nv_bfloat16> hx((size_t)n * d);
  for (int r = 0; r < n; ++r) for (int c = 0; c < d; ++c) hx[(size_t)r * d + c] = __float2bfloat16((float)((r * 7 + c) % 251 + 1));
  __nv_bfloat16* x; CK(cudaMalloc(&x, hx.size() * 2)); CK(cudaMemcpy(x, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
  std::vector<int> hi(256);
  for (int i = 0; i < 256; ++i) hi[i] = (i % 13 == 5) ? n + 7 : (i * 37 + 11) % n;  // some OOB rows
  int* idx; CK(cudaMalloc(&idx, 256 * 4)); CK(cudaMemcpy(idx, hi.data(), 256 * 4, cudaMemcpyHostToDevice));
  int* st; CK(cudaMalloc(&st, 16)); CK(cudaMemset(st, 0, 16));
  __nv_bfloat16* out; CK(cudaMalloc(&out, 2 * 128 * 64 * 2));
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fp; cudaDriverEntryPointQueryResult q; CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  Enc enc = (Enc)fp;
  CUtensorMap tm; cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)n}; cuuint64_t str[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, 1}; cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)cr);
  std::vector<__nv_bfloat16> ho(2 * 128 * 64);
  int ok_all = 1;
  for (int pair = 0; pair < 2; ++pair) {
    CK(cudaMemset(out, 0xff, ho.size() * 2));
    if (pair) probe_kmajor<1><<<2, 32>>>(tm, idx, 64, out, st); else probe_kmajor<0><<<1, 32>>>(tm, idx, 64, out, st);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(ho.data(), out, ho.size() * 2, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int cta = 0; cta <= pair; ++cta)
      for (int r = 0; r < 128; ++r) for (int c = 0; c < 64; ++c) {
        const int src = hi[cta * 128 + r];
        const float want = src >= n ? 0.f : __bfloat162float(hx[(size_t)src * d + 64 + c]);
        if (__bfloat162float(ho[(size_t)cta * 8192 + r * 64 + c]) != want) ++bad;
      }
    printf("kmajor pair=%d mismatches %d\n", pair, bad);
    ok_all &= bad == 0;
  }
  CK(cudaMemset(out, 0xff, ho.size() * 2));
  probe_mnmajor<<<1, 32>>>(tm, idx, 128, out, st);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(ho.data(), out, 64 * 64 * 2, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int k = 0; k < 64; ++k) for (int m = 0; m < 64; ++m) {
    const int src = hi[k];
    const float want = src >= n ? 0.f : __bfloat162float(hx[(size_t)src * d + 128 + m]);
    if (__bfloat162float(ho[k * 64 + m]) != want) ++bad;
  }
  printf("mnmajor mismatches %d\n", bad);
  ok_all &= bad == 0;
  int hs[4]; CK(cudaMemcpy(hs, st, 16, cudaMemcpyDeviceToHost));
  printf("timeouts %d %d\nPROBE %s\n", hs[0], hs[1], ok_all && !hs[0] && !hs[1] ? "OK" : "FAILED");
  return 0;
}
