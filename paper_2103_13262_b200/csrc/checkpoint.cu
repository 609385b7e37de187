// checkpoint.cu -- load / save a layer's weights in the reference's
// checkpoint format (checkpoint.cpp:63-122, codec in ckpt.h) straight from /
// into device memory, one expert at a time.
//
//   load: gate + this rank's expert slice g in [rank*n_e_local, ...) (the
//         other experts are skipped on disk), rounded once to the layer dtype
//         (bf16 weights / fp32 biases on the product path, as init_weights);
//   save: every expert must be local (world_size 1 -- save_checkpoint needs
//         the expert list to cover every global index, checkpoint.cpp:66-67);
//         values are widened exactly to f64.
#include <vector>

#include "ckpt.h"
#include "layer.cuh"

namespace fmoe_b200 {

namespace {

[[noreturn]] void rethrow(const ckpt::CkptError& e) {
  throw Error(e.code == ckpt::SHAPE ? FMOE_ERR_SHAPE : FMOE_ERR_PROTOCOL, e.msg);
}

void upload(const std::vector<double>& src, void* dst, fmoe_dtype as, cudaStream_t s) {
  if (as == FMOE_F64) {
    CK(cudaMemcpyAsync(dst, src.data(), src.size() * 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  } else if (as == FMOE_F32) {
    std::vector<float> f(src.begin(), src.end());
    CK(cudaMemcpyAsync(dst, f.data(), f.size() * 4, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  } else {
    std::vector<__nv_bfloat16> b(src.size());
    for (size_t i = 0; i < src.size(); ++i) b[i] = __float2bfloat16_rn((float)src[i]);
    CK(cudaMemcpyAsync(dst, b.data(), b.size() * 2, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
}

std::vector<double> download(const void* src, size_t n, fmoe_dtype as, cudaStream_t s) {
  std::vector<double> out(n);
  if (as == FMOE_F64) {
    CK(cudaMemcpyAsync(out.data(), src, n * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  } else if (as == FMOE_F32) {
    std::vector<float> f(n);
    CK(cudaMemcpyAsync(f.data(), src, n * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (size_t i = 0; i < n; ++i) out[i] = f[i];
  } else {
    std::vector<__nv_bfloat16> b(n);
    CK(cudaMemcpyAsync(b.data(), src, n * 2, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (size_t i = 0; i < n; ++i) out[i] = (double)__bfloat162float(b[i]);
  }
  return out;
}

}  // namespace

void Layer::load_checkpoint(const char* path) {
  const int64_t d = cfg.d_m, h = cfg.d_h, el = cfg.n_e_local;
  const fmoe_dtype bias_t = t == FMOE_BF16 ? FMOE_F32 : t;
  const size_t bs = t == FMOE_BF16 ? 4 : es;
  try {
    ckpt::Reader in(path);
    const ckpt::Header hd = in.header();
    if ((int64_t)hd.d_m != d || (int64_t)hd.d_h != h || (int64_t)hd.experts != E)
      shape_error("load_checkpoint: file has d_m=" + std::to_string(hd.d_m) + " d_h=" + std::to_string(hd.d_h) +
                  " experts=" + std::to_string(hd.experts) + ", the layer d_m=" + std::to_string(d) +
                  " d_h=" + std::to_string(h) + " experts=" + std::to_string(E));
    // bf16: the weights are the rounding of fp32 masters, which the file's f64
    // values also fill (checkpoint -> resume continues at master precision)
    const bool masters = t == FMOE_BF16;
    if (masters) ensure_masters();
    std::vector<double> buf((size_t)d * E);
    in.matrix(d, E, buf.data(), "gate w_g");
    upload(buf, wg, t, ctx->stream);
    if (masters) upload(buf, m_wg, FMOE_F32, ctx->stream);
    const int64_t first = cfg.rank * el;
    for (int64_t g = 0; g < E; ++g) {
      const bool mine = g >= first && g < first + el;
      const int64_t slot = g - first;
      auto part = [&](uint64_t rows, uint64_t cols, void* dst, fmoe_dtype as, size_t esz, const char* what,
                      float* master) {
        if (!mine) {
          in.matrix(rows, cols, nullptr, what);
          return;
        }
        buf.resize(rows * cols);
        in.matrix(rows, cols, buf.data(), what);
        upload(buf, static_cast<uint8_t*>(dst) + (size_t)slot * rows * cols * esz, as, ctx->stream);
        if (master) upload(buf, master + (size_t)slot * rows * cols, FMOE_F32, ctx->stream);
      };
      part(d, h, w1, t, es, "expert w1", masters ? m_w1 : nullptr);
      part(1, h, b1, bias_t, bs, "expert b1", nullptr);
      part(h, d, w2, t, es, "expert w2", masters ? m_w2 : nullptr);
      part(1, d, b2, bias_t, bs, "expert b2", nullptr);
    }
  } catch (const ckpt::CkptError& e) {
    rethrow(e);
  }
  masters_fresh = t == FMOE_BF16;  // the masters hold the file's values (rounded once to fp32)
}

void Layer::save_checkpoint(const char* path) {
  if (cfg.world_size != 1)
    shape_error("save_checkpoint: expert list must cover every global index (an expert-parallel rank holds only "
                "its slice; save from a world_size 1 layer)");
  const int64_t d = cfg.d_m, h = cfg.d_h;
  const fmoe_dtype bias_t = t == FMOE_BF16 ? FMOE_F32 : t;
  const size_t bs = t == FMOE_BF16 ? 4 : es;
  CK(cudaStreamSynchronize(ctx->stream));
  try {
    ckpt::Writer out(path);
    ckpt::Header hd;
    hd.n_b = cfg.n_b;
    hd.d_m = d;
    hd.d_h = h;
    hd.k = cfg.k;
    hd.n_e_local = cfg.n_e_local;
    hd.world_size = cfg.world_size;
    hd.experts = E;
    hd.seed = cfg.seed;
    out.header(hd);
    // a bf16 layer that trains keeps fp32 masters (SGD's state): save those, so
    // a resumed run continues exactly where the uninterrupted one would
    const bool masters = t == FMOE_BF16 && masters_fresh && m_wg;
    const fmoe_dtype wt = masters ? FMOE_F32 : t;
    const size_t ws = masters ? 4 : es;
    const void *swg = masters ? (const void*)m_wg : wg, *sw1 = masters ? (const void*)m_w1 : w1,
               *sw2 = masters ? (const void*)m_w2 : w2;
    out.matrix(d, E, download(swg, (size_t)d * E, wt, ctx->stream).data());
    for (int64_t g = 0; g < E; ++g) {
      auto at = [&](const void* base, size_t n, size_t esz) { return static_cast<const uint8_t*>(base) + g * n * esz; };
      out.matrix(d, h, download(at(sw1, d * h, ws), d * h, wt, ctx->stream).data());
      out.matrix(1, h, download(at(b1, h, bs), h, bias_t, ctx->stream).data());
      out.matrix(h, d, download(at(sw2, h * d, ws), h * d, wt, ctx->stream).data());
      out.matrix(1, d, download(at(b2, d, bs), d, bias_t, ctx->stream).data());
    }
    out.close();
  } catch (const ckpt::CkptError& e) {
    rethrow(e);
  }
}

}  // namespace fmoe_b200

using namespace fmoe_b200;

extern "C" {

int fmoe_checkpoint_info(const char* path, fmoe_ckpt_info* out) {
  try {
    if (!path || !out) shape_error("checkpoint_info: null argument");
    try {
      ckpt::Reader in(path);
      const ckpt::Header h = in.header();
      *out = fmoe_ckpt_info{(int64_t)h.n_b, (int64_t)h.d_m, (int64_t)h.d_h, (int64_t)h.k, (int64_t)h.n_e_local,
                            (int64_t)h.world_size, (int64_t)h.experts, h.seed};
    } catch (const ckpt::CkptError& e) {
      rethrow(e);
    }
    return FMOE_OK;
  } catch (const std::exception& e) {
    return guard_status(e);
  }
}

int fmoe_layer_load_checkpoint(fmoe_layer* layer, const char* path) {
  try {
    if (!layer || !path) shape_error("load_checkpoint: null argument");
    reinterpret_cast<Layer*>(layer)->load_checkpoint(path);
    return FMOE_OK;
  } catch (const std::exception& e) {
    return guard_status(e);
  }
}

int fmoe_layer_save_checkpoint(fmoe_layer* layer, const char* path) {
  try {
    if (!layer || !path) shape_error("save_checkpoint: null argument");
    reinterpret_cast<Layer*>(layer)->save_checkpoint(path);
    return FMOE_OK;
  } catch (const std::exception& e) {
    return guard_status(e);
  }
}

}  // extern "C"
