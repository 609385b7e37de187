// layer_capi.cu -- extern "C" entry points of the MoE layer (fmoe_layer_*).
#include "layer.cuh"

using namespace fmoe_b200;

#define FMOE_GUARD(...)               \
  try {                               \
    __VA_ARGS__;                      \
    return FMOE_OK;                   \
  } catch (const std::exception& e) { \
    return guard_status(e);           \
  } catch (...) {                     \
    g_last_error = "unknown error";   \
    return FMOE_ERR_CUDA;             \
  }

namespace {
Layer* L(fmoe_layer* l) {
  if (!l) shape_error("null layer");
  return reinterpret_cast<Layer*>(l);
}
}  // namespace

extern "C" {

int fmoe_layer_create(fmoe_ctx* ctx, const fmoe_layer_config* cfg, fmoe_layer** out) {
  FMOE_GUARD({
    if (!ctx || !cfg || !out) shape_error("fmoe_layer_create: null argument");
    *out = reinterpret_cast<fmoe_layer*>(new Layer(reinterpret_cast<Ctx*>(ctx), *cfg));
  })
}

int fmoe_layer_destroy(fmoe_layer* layer) { FMOE_GUARD(delete L(layer)) }

int fmoe_layer_init_weights(fmoe_layer* layer) { FMOE_GUARD(L(layer)->init_weights()) }

int fmoe_layer_params(fmoe_layer* layer, void** w_g, fmoe_expert_params* experts) {
  FMOE_GUARD({
    Layer* l = L(layer);
    if (w_g) *w_g = l->wg;
    if (experts) *experts = l->params();
  })
}

int fmoe_layer_keep_preact(fmoe_layer* layer, int keep) { FMOE_GUARD(L(layer)->set_keep_preact(keep != 0)) }

int fmoe_layer_activations(fmoe_layer* layer, const void** xs, const void** hidden, const void** preact,
                           const void** ys) {
  FMOE_GUARD({
    Layer* l = L(layer);
    if (xs) {
      l->ensure_xs();
      *xs = l->xs;
    }
    if (hidden) *hidden = l->hidden;
    if (preact) *preact = l->preact;
    if (ys) *ys = l->ys;
  })
}

int fmoe_layer_grads(fmoe_layer* layer, void** d_wg, fmoe_expert_grads* experts) {
  FMOE_GUARD({
    Layer* l = L(layer);
    if (d_wg) *d_wg = l->dwg;
    if (experts) *experts = l->grads();
  })
}

int fmoe_layer_routing(fmoe_layer* layer, const int32_t** topk_idx, const void** topk_scores,
                       const void** scores, fmoe_plan* plan) {
  FMOE_GUARD({
    Layer* l = L(layer);
    if (topk_idx) *topk_idx = l->idx;
    if (topk_scores) *topk_scores = l->vals;
    if (scores) *scores = l->scores;
    if (plan) *plan = l->plan;
  })
}

int fmoe_layer_fwd(fmoe_layer* layer, const void* x, void* y) {
  FMOE_GUARD({
    if ((!x || !y) && L(layer)->cfg.n_b > 0) shape_error("forward: null x or y");  // empty batches may be NULL
    L(layer)->forward(x, y);
  })
}

int fmoe_layer_fwd_routed(fmoe_layer* layer, const void* x, const int32_t* topk_idx, const void* topk_scores,
                          void* y) {
  FMOE_GUARD({
    if ((!x || !y || !topk_idx || !topk_scores) && L(layer)->cfg.n_b > 0) shape_error("forward_routed: null argument");
    L(layer)->forward_routed(x, topk_idx, topk_scores, y);
  })
}

int fmoe_layer_routing_grad(fmoe_layer* layer, const void** d_topk_scores) {
  FMOE_GUARD({
    if (d_topk_scores) *d_topk_scores = L(layer)->d_w;
  })
}

int fmoe_layer_bwd(fmoe_layer* layer, const void* dy, void* dx) {
  FMOE_GUARD({
    if ((!dy || !dx) && L(layer)->cfg.n_b > 0) shape_error("backward: null dy or dx");
    L(layer)->backward(dy, dx);
  })
}

// The names SURVEY §8b lists for the C-ABI's layer entry points.
int fmoe_moe_fwd(fmoe_layer* layer, const void* x, void* y) { return fmoe_layer_fwd(layer, x, y); }
int fmoe_moe_bwd(fmoe_layer* layer, const void* dy, void* dx) { return fmoe_layer_bwd(layer, dy, dx); }

int fmoe_layer_train_step(fmoe_layer* layer, const void* x, const void* target, double lr, double* loss) {
  FMOE_GUARD({
    if (!x || !target) shape_error("train_step: null x or target");
    const double v = L(layer)->train_step(x, target, lr);
    if (loss) *loss = v;
  })
}

int fmoe_layer_sync_masters(fmoe_layer* layer) { FMOE_GUARD(L(layer)->masters_fresh = false) }

int fmoe_layer_step_host(fmoe_layer* layer, const void* x_host, const void* dy_host, void* y_host,
                         void* dx_host) {
  FMOE_GUARD({
    if (!x_host || !y_host) shape_error("step_host: null x or y");
    L(layer)->step_host(x_host, dy_host, y_host, dx_host);
  })
}

int fmoe_layer_step_host_async(fmoe_layer* layer, const void* x_host, const void* dy_host, void* y_host,
                               void* dx_host) {
  FMOE_GUARD({
    if ((!x_host || !y_host) && L(layer)->cfg.n_b > 0) shape_error("step_host_async: null x or y");
    L(layer)->step_host_submit(x_host, dy_host, y_host, dx_host);
  })
}

int fmoe_layer_step_host_wait(fmoe_layer* layer) { FMOE_GUARD(L(layer)->step_host_wait()) }

}  // extern "C"
