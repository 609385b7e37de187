// layer.cuh -- MoE layer state (moe_layer.hpp:17-66) on device.
#pragma once

#include <vector>

#include "common.cuh"

namespace fmoe_b200 {

struct Layer {
  Ctx* ctx;
  fmoe_layer_config cfg;
  int64_t E = 0;  // total experts
  fmoe_dtype t;
  size_t es = 0, ss = 0, gs = 0;
  std::vector<void*> owned;
  // parameters (gate replicated, local experts in slot order)
  void *wg = nullptr, *w1 = nullptr, *b1 = nullptr, *w2 = nullptr, *b2 = nullptr;
  // gradients
  void *dwg = nullptr, *dw1 = nullptr, *db1 = nullptr, *dw2 = nullptr, *db2 = nullptr;
  // forward cache (MoEForwardCache, moe_layer.hpp:42-50)
  const void* x_saved = nullptr;  // caller keeps x alive until backward
  void *scores = nullptr, *vals = nullptr, *logits = nullptr;
  int32_t* idx = nullptr;
  fmoe_plan plan{};
  void *xs = nullptr, *hidden = nullptr, *ys = nullptr;
  // bf16, one GPU, FMOE_TC_GATHER=1: fc1 and its weight gradient gather their
  // input rows from x (TMA gather4, ops.cuh RowGather); xs is then filled only
  // on request (activations(): the operator-level cache view)
  bool gather_xs = false, xs_fresh = false;
  void ensure_xs();
  void* preact = nullptr;  // x*w1 + b1, when kept (fmoe_layer_keep_preact; SIMT / F32 dtypes)
  bool preact_kept = false;
  bool fwd_done = false;
  bool routed = false;
  int prof_slot = -1;   // profiling slot of the current forward (Prof)  // forward_routed: routing injected, no gate on this step
  // backward scratch
  void *d_ys = nullptr, *d_pre = nullptr, *d_xs = nullptr, *d_w = nullptr, *dz = nullptr, *gdx = nullptr;
  __nv_bfloat16* dz_bf16 = nullptr;
  float* part = nullptr;   // gate d_wg split-K partials
  float* tpart = nullptr;  // expert bias-gradient tile partials
  uint32_t* relu_bits = nullptr;  // bf16: hidden > 0 bitmap (fc1 -> dgrad fc2)
  // FMOE_F32 on the tensor cores (f32x.cu): bf16x6 operand planes of x, Wg,
  // dz, xs, hidden, d_ys, d_pre, W1, W2 (three each); null on the SIMT route
  __nv_bfloat16* f32_planes = nullptr;
  struct F32Planes planes_view() const;
  // host-buffer steps: two device buffer sets (x, y, dy, dx each) and their events
  void* io = nullptr;
  struct HostIO {
    cudaEvent_t x_done[2] = {}, dy_done[2] = {}, y_ready[2] = {}, dx_ready[2] = {}, compute_done[2] = {},
                out_done[2] = {};
    int64_t seq = 0;
  } hio;
  void* h_stage = nullptr;
  // training step (train.cu): output, d_y, d_x, loss scratch; fp32 masters of
  // the bf16 weights (widened on the first step after init / an explicit resync)
  void *t_y = nullptr, *t_dy = nullptr, *t_dx = nullptr;
  double* t_loss = nullptr;
  float *m_wg = nullptr, *m_w1 = nullptr, *m_w2 = nullptr;
  bool masters_fresh = false;
  void ensure_masters();
  // expert parallelism (ep.cu)
  struct Ep;
  Ep* ep = nullptr;

  Layer(Ctx* c, const fmoe_layer_config& cf);
  ~Layer();
  fmoe_expert_params params() const;
  fmoe_expert_grads grads() const;
  void init_weights();
  void set_keep_preact(bool keep);
  void forward(const void* x, void* y);
  void forward_routed(const void* x, const int32_t* topk_idx, const void* topk_scores, void* y);
  void dispatch_and_experts(const void* x, void* y);
  void backward(const void* dy, void* dx, cudaEvent_t dx_ready = nullptr);
  double train_step(const void* x, const void* target, double lr);
  void sgd(void* param, float* master, const void* grad, int64_t n, double lr, bool weight);
  void step_host(const void* x_host, const void* dy_host, void* y_host, void* dx_host);
  void step_host_submit(const void* x_host, const void* dy_host, void* y_host, void* dx_host);
  void step_host_wait();
  void host_io_setup();
  void load_checkpoint(const char* path);  // checkpoint.cu
  void save_checkpoint(const char* path);
  void ep_alloc();
  void ep_check() const;  // ProtocolError unless a matching transport is attached
  void ep_forward(const void* x, void* y);
  void ep_backward(const void* dy, void* dx);
  static void ep_free(Ep* e);
};

}  // namespace fmoe_b200
