// train.cu -- one SGD training step of the MoE layer on device
// (train_step, moe_layer.cpp:144-205; sync_gradients / sgd_step,
// param_sync.cpp:46-66):
//   forward -> mean-squared error against the target and d_y = 2*diff/n ->
//   backward -> (EP) expert gradients * 1/W -> gate gradient averaged over the
//   world (allreduce_sum in ascending rank order, then * 1/W) -> SGD on every
//   parameter -> (EP) world-average loss.
// FMOE_F64 follows the reference's arithmetic exactly (sequential loss sum,
// a += alpha*b as one fma); FMOE_F32 / FMOE_BF16 reduce the loss with a fixed
// two-level tree in fp64 (deterministic) and keep fp32 master copies of the
// bf16 weights, so repeated small updates are not lost to bf16 rounding.
#include <type_traits>
#include <vector>

#include "comm.cuh"
#include "layer.cuh"
#include "ops.cuh"

namespace fmoe_b200 {
namespace {

constexpr int kLossBlocks = 296;  // 2 x 148 SMs, fixed so the sum order is fixed
constexpr int kLossThreads = 256;

__device__ __forceinline__ double ld(const double* p, int64_t i) { return p[i]; }
__device__ __forceinline__ double ld(const float* p, int64_t i) { return (double)p[i]; }
__device__ __forceinline__ double ld(const __nv_bfloat16* p, int64_t i) { return (double)__bfloat162float(p[i]); }

// d_y[i] = 2 * (y[i] - t[i]) / n  (moe_layer.cpp:153-158)
template <typename T>
__global__ void mse_grad_kernel(const T* __restrict__ y, const T* __restrict__ t, int64_t n, T* __restrict__ dy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if constexpr (std::is_same<T, double>::value) {
    const double diff = y[i] - t[i];
    dy[i] = 2.0 * diff / (double)n;
  } else {
    const float diff = to_f(y[i]) - to_f(t[i]);
    dy[i] = from_f<T>(2.0f * diff / (float)n);
  }
}

// FMOE_F64: the reference's loop, loss += diff*diff/n in element order.
__global__ void mse_loss_seq_kernel(const double* __restrict__ y, const double* __restrict__ t, int64_t n,
                                    double* __restrict__ loss) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double dn = (double)n;
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double diff = y[i] - t[i];
    acc = acc + diff * diff / dn;
  }
  *loss = acc;
}

// FMOE_F32 / FMOE_BF16: fixed partition, fp64 partial sums, then an ordered sum.
template <typename T>
__global__ void mse_loss_partial_kernel(const T* __restrict__ y, const T* __restrict__ t, int64_t n,
                                        double* __restrict__ part) {
  __shared__ double sh[kLossThreads];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kLossThreads + threadIdx.x; i < n; i += (int64_t)kLossBlocks * kLossThreads) {
    const double diff = ld(y, i) - ld(t, i);
    acc += diff * diff;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kLossThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void mse_loss_final_kernel(const double* __restrict__ part, int64_t n, double* __restrict__ loss) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0;
  for (int b = 0; b < kLossBlocks; ++b) acc += part[b];
  *loss = acc / (double)n;
}

// a *= s  (scale_inplace, matrix.cpp)
template <typename G>
__global__ void scale_kernel(G* __restrict__ a, int64_t n, G s) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = a[i] * s;
}

// sgd_step (param_sync.cpp:63-66): p = fma(-lr, g, p); with a master copy the
// update happens on the fp32 master and the bf16 parameter is its rounding.
template <typename P, typename G>
__global__ void sgd_kernel(P* __restrict__ p, const G* __restrict__ g, int64_t n, G neg_lr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = fma(neg_lr, g[i], p[i]);
}
__global__ void sgd_master_kernel(__nv_bfloat16* __restrict__ p, float* __restrict__ m, const float* __restrict__ g,
                                  int64_t n, float neg_lr) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = fmaf(neg_lr, g[i], m[i]);
  m[i] = v;
  p[i] = __float2bfloat16_rn(v);
}
__global__ void widen_kernel(const __nv_bfloat16* __restrict__ p, float* __restrict__ m, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) m[i] = __bfloat162float(p[i]);
}

unsigned blocks_for(int64_t n) { return (unsigned)ceil_div(n, 256); }

void scale(Ctx* c, fmoe_dtype gt, void* a, int64_t n, double s) {
  if (n == 0) return;
  if (gt == FMOE_F64)
    scale_kernel<double><<<blocks_for(n), 256, 0, c->stream>>>((double*)a, n, s);
  else
    scale_kernel<float><<<blocks_for(n), 256, 0, c->stream>>>((float*)a, n, (float)s);
  CK_LAUNCH(c);
}

}  // namespace

void Layer::sgd(void* param, float* master, const void* grad, int64_t n, double lr, bool weight) {
  if (n == 0) return;
  if (t == FMOE_F64) {
    sgd_kernel<double, double><<<blocks_for(n), 256, 0, ctx->stream>>>((double*)param, (const double*)grad, n, -lr);
  } else if (t == FMOE_F32 || !weight) {  // fp32 parameters (incl. bf16-mode biases)
    sgd_kernel<float, float><<<blocks_for(n), 256, 0, ctx->stream>>>((float*)param, (const float*)grad, n,
                                                                     (float)-lr);
  } else {
    sgd_master_kernel<<<blocks_for(n), 256, 0, ctx->stream>>>((__nv_bfloat16*)param, master, (const float*)grad, n,
                                                             (float)-lr);
  }
  CK_LAUNCH(ctx);
}

// fp32 master copies of the bf16 weights (SGD updates them; the bf16 weights
// are their rounding).  Allocated on the first train_step or checkpoint load.
void Layer::ensure_masters() {
  if (t != FMOE_BF16 || m_wg) return;
  const int64_t d = cfg.d_m, h = cfg.d_h, el = cfg.n_e_local;
  auto grab = [&](size_t bytes) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
    owned.push_back(p);
    return (float*)p;
  };
  m_wg = grab((size_t)d * E * 4);
  m_w1 = grab((size_t)el * d * h * 4);
  m_w2 = grab((size_t)el * h * d * 4);
}

double Layer::train_step(const void* x, const void* target, double lr) {
  const int64_t n = cfg.n_b * cfg.d_m, el = cfg.n_e_local, d = cfg.d_m, h = cfg.d_h;
  const int W = (int)cfg.world_size;
  const bool ep = W > 1;
  // the gate gradient is all-reduced over the world (param_sync.cpp:46-61):
  // an expert-parallel step needs the transport for it, so refuse before any
  // forward/backward work or gradient scaling is issued
  if (ep && (!ctx->transport || ctx->transport->world != W || ctx->transport->rank != cfg.rank))
    protocol_error("train_step: expert-parallel training (world " + std::to_string(W) +
                   ") needs a transport of the same world and rank for the gate all-reduce: "
                   "fmoe_comm_init, fmoe_comm_attach or fmoe_ctx_join_world");
  if (!t_y) {  // buffers for the step, allocated on first use
    auto grab = [&](size_t bytes) {
      void* p = nullptr;
      CK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
      owned.push_back(p);
      return p;
    };
    t_y = grab((size_t)n * es);
    t_dy = grab((size_t)n * es);
    t_dx = grab((size_t)n * es);
    t_loss = (double*)grab((kLossBlocks + 2) * sizeof(double));
  }
  ensure_masters();
  if (t == FMOE_BF16 && !masters_fresh) {  // fp32 masters widened from the current bf16 weights
    widen_kernel<<<blocks_for(d * E), 256, 0, ctx->stream>>>((const __nv_bfloat16*)wg, m_wg, d * E);
    widen_kernel<<<blocks_for(el * d * h), 256, 0, ctx->stream>>>((const __nv_bfloat16*)w1, m_w1, el * d * h);
    widen_kernel<<<blocks_for(el * h * d), 256, 0, ctx->stream>>>((const __nv_bfloat16*)w2, m_w2, el * h * d);
    CK_LAUNCH(ctx);
    masters_fresh = true;
  }
  forward(x, t_y);
  // loss and d_y
  if (n > 0) {
    dispatch_dtype(t, [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      mse_grad_kernel<T><<<blocks_for(n), 256, 0, ctx->stream>>>((const T*)t_y, (const T*)target, n, (T*)t_dy);
      if constexpr (std::is_same<T, double>::value) {
        mse_loss_seq_kernel<<<1, 32, 0, ctx->stream>>>((const double*)t_y, (const double*)target, n, t_loss);
      } else {
        mse_loss_partial_kernel<T><<<kLossBlocks, kLossThreads, 0, ctx->stream>>>((const T*)t_y, (const T*)target, n,
                                                                                   t_loss + 2);
        mse_loss_final_kernel<<<1, 32, 0, ctx->stream>>>(t_loss + 2, n, t_loss);
      }
    });
    CK_LAUNCH(ctx);
  } else {
    CK(cudaMemsetAsync(t_loss, 0, 8, ctx->stream));
  }
  backward(t_dy, t_dx);
  const fmoe_dtype gt = t == FMOE_F64 ? FMOE_F64 : FMOE_F32;  // gradient dtype
  if (ep) {
    // experts saw the whole world's rows, each rank normalised by its own batch
    const double inv = 1.0 / (double)W;
    scale(ctx, gt, dw1, el * d * h, inv);
    scale(ctx, gt, db1, el * h, inv);
    scale(ctx, gt, dw2, el * h * d, inv);
    scale(ctx, gt, db2, el * d, inv);
    // gate (ParamTag::World): average over every rank
    std::vector<int> world(W);
    for (int r = 0; r < W; ++r) world[r] = r;
    allreduce_sum(ctx, gt, dwg, d * E, world.data(), W);
    scale(ctx, gt, dwg, d * E, 1.0 / (double)W);
  }
  sgd(wg, m_wg, dwg, d * E, lr, true);
  sgd(w1, m_w1, dw1, el * d * h, lr, true);
  sgd(b1, nullptr, db1, el * h, lr, false);
  sgd(w2, m_w2, dw2, el * h * d, lr, true);
  sgd(b2, nullptr, db2, el * d, lr, false);
  if (ep) {
    std::vector<int> world(W);
    for (int r = 0; r < W; ++r) world[r] = r;
    allreduce_sum(ctx, FMOE_F64, t_loss, 1, world.data(), W);
  }
  double loss = 0.0;
  CK(cudaMemcpyAsync(&loss, t_loss, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ep ? loss / (double)W : loss;
}

}  // namespace fmoe_b200
