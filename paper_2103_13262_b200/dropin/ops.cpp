// ops.cpp -- device plumbing and the stateless operators of the drop-in:
// matrix primitives, generators, gate, dispatch and the expert pool
// (reference API: proj/include/fmoe/{matrix,rng,gate,dispatch,expert}.hpp).
#include <atomic>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <utility>

#include "dropin.hpp"
#include "fmoe/dispatch.hpp"
#include "fmoe/errors.hpp"
#include "fmoe/expert.hpp"
#include "fmoe/gate.hpp"
#include "fmoe/param_tag.hpp"
#include "fmoe/rng.hpp"

namespace fmoe {
namespace dropin {

void check(int status) {
  if (status == FMOE_OK) return;
  const std::string msg = fmoe_last_error();
  switch (status) {
    case FMOE_ERR_SHAPE: throw ShapeError(msg);
    case FMOE_ERR_PROTOCOL: throw ProtocolError(msg);
    case FMOE_ERR_TRANSPORT: throw TransportError(msg);
    default: throw std::runtime_error("fmoe_b200: " + msg);
  }
}

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("fmoe drop-in: ") + what + ": " + cudaGetErrorString(e));
}

int default_device() {
  const char* s = std::getenv("FMOE_DEVICE");
  return s ? std::atoi(s) : 0;
}

Device::Device() : device(default_device()) {
  cuda(cudaSetDevice(device), "cudaSetDevice");
  cuda(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  check(fmoe_ctx_create(device, stream, &ctx));
}

Device::~Device() {
  if (ctx) fmoe_ctx_destroy(ctx);
  if (stream) cudaStreamDestroy(stream);
}

Device& local() {
  thread_local Device d;
  return d;
}

Buf::Buf(std::size_t bytes, cudaStream_t s) : s_(s) {
  cuda(cudaMallocAsync(&p_, bytes < 16 ? 16 : bytes, s), "cudaMallocAsync");
}
Buf::~Buf() {
  if (p_ && owned_) cudaFreeAsync(p_, s_);
}
Buf::Buf(Buf&& o) noexcept : p_(o.p_), s_(o.s_), owned_(o.owned_) { o.p_ = nullptr; }
Buf& Buf::operator=(Buf&& o) noexcept {
  if (this != &o) {
    if (p_ && owned_) cudaFreeAsync(p_, s_);
    p_ = o.p_;
    s_ = o.s_;
    owned_ = o.owned_;
    o.p_ = nullptr;
  }
  return *this;
}

Buf upload(const Matrix& m, cudaStream_t s) {
  if (const auto& st = m.device_store()) return Buf::view(st->f64(m.device_offset()));
  return upload(m.data(), m.size() * sizeof(double), s);
}

Buf upload_copy(const Matrix& m, cudaStream_t s) {
  if (const auto& st = m.device_store()) {
    Buf b(m.size() * sizeof(double), s);
    if (m.size())
      cuda(cudaMemcpyAsync(b.get(), st->f64(m.device_offset()), m.size() * sizeof(double), cudaMemcpyDeviceToDevice,
                           s),
           "D2D");
    return b;
  }
  return upload(m.data(), m.size() * sizeof(double), s);
}

namespace {
// One stream per device for the stores' pool allocations and frees; the
// device's default memory pool keeps freed blocks for reuse.
cudaStream_t pool_stream(int device) {
  static std::once_flag once[64];
  static cudaStream_t streams[64];
  std::call_once(once[device & 63], [device] {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaStreamCreateWithFlags(&streams[device & 63], cudaStreamNonBlocking);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      std::uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaSetDevice(cur);
  });
  return streams[device & 63];
}
}  // namespace

std::shared_ptr<detail::DeviceStore> device_store(std::size_t bytes, const Device& d) {
  auto st = std::make_shared<detail::DeviceStore>();
  st->device = d.device;
  st->bytes = bytes;
  cudaStream_t ps = pool_stream(d.device);
  cuda(cudaMallocAsync(&st->ptr, bytes < 16 ? 16 : bytes, ps), "cudaMallocAsync (device store)");
  cudaEvent_t ev;
  cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
  cuda(cudaEventRecord(ev, ps), "cudaEventRecord");
  cuda(cudaStreamWaitEvent(d.stream, ev, 0), "cudaStreamWaitEvent");
  cudaEventDestroy(ev);
  return st;
}

Buf upload(const void* host, std::size_t bytes, cudaStream_t s) {
  Buf b(bytes, s);
  if (bytes) cuda(cudaMemcpyAsync(b.get(), host, bytes, cudaMemcpyHostToDevice, s), "H2D");
  // host buffers may be temporaries: the copy must finish before we return
  cuda(cudaStreamSynchronize(s), "H2D sync");
  return b;
}

Buf upload_i32(const std::int64_t* v, std::size_t n, cudaStream_t s, const char* what) {
  std::vector<std::int32_t> t(n);
  for (std::size_t i = 0; i < n; ++i) {
    if (v[i] < std::numeric_limits<std::int32_t>::min() || v[i] > std::numeric_limits<std::int32_t>::max())
      throw ShapeError(std::string(what) + ": index " + std::to_string(v[i]) + " does not fit the device plan");
    t[i] = static_cast<std::int32_t>(v[i]);
  }
  return upload(t.data(), n * 4, s);
}

void download(void* host, const void* dev, std::size_t bytes, const Device& d) {
  if (bytes) cuda(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, d.stream), "D2H");
  check(fmoe_ctx_check(d.ctx));
}

std::vector<std::int64_t> download_i32(const Buf& b, std::size_t n, const Device& d) {
  std::vector<std::int32_t> t(n);
  download(t.data(), b.get(), n * 4, d);
  return std::vector<std::int64_t>(t.begin(), t.end());
}

}  // namespace dropin

std::uint64_t Matrix::next_id() noexcept {
  static std::atomic<std::uint64_t> next{1};
  return next.fetch_add(1, std::memory_order_relaxed);
}

detail::DeviceStore::~DeviceStore() {
  if (ptr) cudaFreeAsync(ptr, dropin::pool_stream(device));
}

// First host access of a device-backed Matrix: copy its values down (the
// stores are complete: every drop-in call synchronised before returning).
void Matrix::fetch() const noexcept {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (host_ok_.load(std::memory_order_acquire)) return;
  data_.resize(rows_ * cols_);
  if (!data_.empty()) {
    const cudaError_t e = cudaMemcpy(data_.data(), dev_->f64(dev_off_), data_.size() * sizeof(double),
                                     cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      std::fprintf(stderr, "fmoe drop-in: device -> host copy of a result failed: %s\n", cudaGetErrorString(e));
      std::abort();
    }
  }
  host_ok_.store(true, std::memory_order_release);
}

using dropin::Buf;
using dropin::check;
using dropin::download;
using dropin::local;
using dropin::upload;

// ------------------------------------------------------------ value types
namespace {
template <typename M, typename V>
M rows_to_matrix(std::initializer_list<std::initializer_list<V>> rows) {
  const std::size_t r = rows.size(), c = r ? rows.begin()->size() : 0;
  M m(r, c);
  std::size_t i = 0;
  for (const auto& row : rows) {
    if (row.size() != c) throw ShapeError("from_rows: ragged row lengths");
    std::size_t j = 0;
    for (V v : row) m(i, j++) = v;
    ++i;
  }
  return m;
}
}  // namespace

Matrix Matrix::from_rows(std::initializer_list<std::initializer_list<double>> rows) {
  return rows_to_matrix<Matrix, double>(rows);
}
IndexMatrix IndexMatrix::from_rows(std::initializer_list<std::initializer_list<std::int64_t>> rows) {
  return rows_to_matrix<IndexMatrix, std::int64_t>(rows);
}
Matrix Matrix::identity(std::size_t n) {
  Matrix m(n, n);
  for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}

const char* to_string(ParamTag tag) {
  switch (tag) {
    case ParamTag::World: return "world";
    case ParamTag::DataParallel: return "data_parallel";
    case ParamTag::NoSync: return "none";
  }
  return "?";
}

// ------------------------------------------------------ dense primitives
Matrix matmul(const Matrix& a, const Matrix& b) {
  if (a.cols() != b.rows())
    throw ShapeError("matmul: inner dimensions " + std::to_string(a.cols()) + " and " + std::to_string(b.rows()) +
                     " differ");
  Matrix c(a.rows(), b.cols());
  if (c.size() == 0) return c;
  auto& d = local();
  Buf da = upload(a, d.stream), db = upload(b, d.stream), dc(c.size() * 8, d.stream);
  check(fmoe_matmul(d.ctx, FMOE_F64, da.get(), db.get(), (int64_t)a.rows(), (int64_t)a.cols(), (int64_t)b.cols(),
                    dc.get()));
  download(c, dc, d);
  return c;
}

Matrix softmax_rows(const Matrix& a) {
  Matrix out(a.rows(), a.cols());
  if (out.size() == 0) return out;
  auto& d = local();
  Buf da = upload(a, d.stream), dout(out.size() * 8, d.stream);
  check(fmoe_softmax_rows(d.ctx, FMOE_F64, da.get(), (int64_t)a.rows(), (int64_t)a.cols(), dout.get()));
  download(out, dout, d);
  return out;
}

TopK topk_rows(const Matrix& a, std::size_t k) {
  if (k < 1 || k > a.cols())
    throw ShapeError("topk_rows: k out of range [1, " + std::to_string(a.cols()) + "]");
  TopK r{IndexMatrix(a.rows(), k), Matrix(a.rows(), k)};
  if (a.rows() == 0) return r;
  auto& d = local();
  Buf da = upload(a, d.stream), di(a.rows() * k * 4, d.stream), dv(a.rows() * k * 8, d.stream);
  check(fmoe_topk_rows(d.ctx, FMOE_F64, da.get(), (int64_t)a.rows(), (int64_t)a.cols(), (int64_t)k,
                       di.as<int32_t>(), dv.get()));
  const auto idx = dropin::download_i32(di, a.rows() * k, d);
  std::memcpy(r.indices.data(), idx.data(), idx.size() * 8);
  download(r.values, dv, d);
  return r;
}

Matrix transpose(const Matrix& a) {
  Matrix t(a.cols(), a.rows());
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t j = 0; j < a.cols(); ++j) t(j, i) = a(i, j);
  return t;
}

Matrix add_bias_rows(const Matrix& a, const Matrix& bias) {
  if (bias.rows() != 1 || bias.cols() != a.cols()) throw ShapeError("add_bias_rows: bias must be 1 x cols(a)");
  Matrix out = a;
  for (std::size_t i = 0; i < out.rows(); ++i)
    for (std::size_t j = 0; j < out.cols(); ++j) out(i, j) = out(i, j) + bias(0, j);
  return out;
}

Matrix relu(const Matrix& a) {
  Matrix out = a;
  for (std::size_t i = 0; i < out.size(); ++i) out.data()[i] = out.data()[i] < 0.0 ? 0.0 : out.data()[i];
  return out;
}

Matrix relu_backward(const Matrix& d_y, const Matrix& x) {
  if (!d_y.same_shape(x)) throw ShapeError("relu_backward: shape mismatch");
  Matrix out(d_y.rows(), d_y.cols());
  for (std::size_t i = 0; i < out.size(); ++i) out.data()[i] = x.data()[i] > 0.0 ? d_y.data()[i] : 0.0;
  return out;
}

void add_inplace(Matrix& a, const Matrix& b) {
  if (!a.same_shape(b)) throw ShapeError("add_inplace: shape mismatch");
  for (std::size_t i = 0; i < a.size(); ++i) a.data()[i] = a.data()[i] + b.data()[i];
}

void axpy_inplace(Matrix& a, double alpha, const Matrix& b) {
  if (!a.same_shape(b)) throw ShapeError("axpy_inplace: shape mismatch");
  // the reference build contracts a += alpha*b into one fma
  for (std::size_t i = 0; i < a.size(); ++i) a.data()[i] = std::fma(alpha, b.data()[i], a.data()[i]);
}

void scale_inplace(Matrix& a, double s) {
  for (std::size_t i = 0; i < a.size(); ++i) a.data()[i] = a.data()[i] * s;
}

// ------------------------------------------------------------- generators
std::uint64_t stream_seed(std::uint64_t base_seed, std::uint64_t stream_id) {
  // splitmix64 finaliser over base + golden-ratio step * (id + 1)
  std::uint64_t z = base_seed + 0x9E3779B97F4A7C15ULL * (stream_id + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

GateParams init_gate(std::size_t d_m, std::size_t total_experts, std::uint64_t seed) {
  GateParams g{Matrix(d_m, total_experts), ParamTag::World};
  UniformRng(stream_seed(seed, 0x67617465ULL)).fill(g.w_g, -0.1, 0.1);
  return g;
}

ExpertParams init_expert(std::size_t d_m, std::size_t d_h, std::uint64_t seed) {
  ExpertParams p{Matrix(d_m, d_h), Matrix(1, d_h), Matrix(d_h, d_m), Matrix(1, d_m), ParamTag::NoSync};
  UniformRng rng(seed);
  for (Matrix* m : {&p.w1, &p.b1, &p.w2, &p.b2}) rng.fill(*m, -0.1, 0.1);
  return p;
}

// ------------------------------------------------------------------- gate
GateOutput gate_forward(const Matrix& x, const GateParams& params, std::size_t k) {
  const std::size_t n = x.rows(), E = params.w_g.cols();
  if (x.cols() != params.w_g.rows())
    throw ShapeError("gate_forward: x cols " + std::to_string(x.cols()) + " != gate rows " +
                     std::to_string(params.w_g.rows()));
  if (k < 1 || k > E) throw ShapeError("gate_forward: k out of range");
  GateOutput out{Matrix(n, E), IndexMatrix(n, k), Matrix(n, k)};
  if (n == 0) return out;
  auto& d = local();
  Buf dx = upload(x, d.stream), dw = upload(params.w_g, d.stream);
  Buf ds(n * E * 8, d.stream), di(n * k * 4, d.stream), dv(n * k * 8, d.stream);
  check(fmoe_gate_fwd(d.ctx, FMOE_F64, dx.get(), dw.get(), (int64_t)n, (int64_t)x.cols(), (int64_t)E, (int64_t)k,
                      ds.get(), di.as<int32_t>(), dv.get()));
  download(out.scores, ds, d);
  const auto idx = dropin::download_i32(di, n * k, d);
  std::memcpy(out.topk_indices.data(), idx.data(), idx.size() * 8);
  download(out.topk_scores, dv, d);
  return out;
}

GateGrads gate_backward(const Matrix& x, const GateParams& params, const GateOutput& out,
                        const Matrix& d_topk_scores) {
  const std::size_t n = x.rows(), dm = x.cols(), E = params.w_g.cols(), k = out.topk_indices.cols();
  if (params.w_g.rows() != dm) throw ShapeError("gate_backward: x cols != gate rows");
  if (out.scores.rows() != n || out.scores.cols() != E) throw ShapeError("gate_backward: scores shape mismatch");
  if (d_topk_scores.rows() != n || d_topk_scores.cols() != k || out.topk_indices.rows() != n)
    throw ShapeError("gate_backward: upstream gradient shape mismatch");
  for (std::size_t i = 0; i < out.topk_indices.size(); ++i)
    if (out.topk_indices.data()[i] < 0 || out.topk_indices.data()[i] >= (std::int64_t)E)
      throw ShapeError("gate_backward: top-k index out of range");
  GateGrads g{Matrix(dm, E), Matrix(n, dm)};
  if (n == 0 || k == 0) return g;
  auto& d = local();
  Buf dx = upload(x, d.stream), dw = upload(params.w_g, d.stream), ds = upload(out.scores, d.stream);
  Buf di = dropin::upload_i32(out.topk_indices.data(), n * k, d.stream, "gate_backward");
  Buf dt = upload(d_topk_scores, d.stream);
  Buf dwg(dm * E * 8, d.stream), ddx(n * dm * 8, d.stream);
  check(fmoe_gate_bwd(d.ctx, FMOE_F64, dx.get(), dw.get(), ds.get(), di.as<int32_t>(), dt.get(), (int64_t)n,
                      (int64_t)dm, (int64_t)E, (int64_t)k, dwg.get(), ddx.get()));
  download(g.d_wg, dwg, d);
  download(g.d_x, ddx, d);
  return g;
}

// --------------------------------------------------------------- dispatch
namespace {
// A host DispatchPlan on the device (align 1: the reference layout).
struct DevPlan {
  Buf counts, offsets, src, slot, inv;
  fmoe_plan p{};
};

DevPlan device_plan(const DispatchPlan& plan, const char* who) {
  const std::size_t E = plan.num_experts, nk = plan.n_b * plan.k;
  if (plan.counts.size() != E || plan.offsets.size() != E || plan.expanded_src_row.size() != nk ||
      plan.expanded_slot.size() != nk || plan.inverse_pos.rows() != plan.n_b || plan.inverse_pos.cols() != plan.k)
    throw ShapeError(std::string(who) + ": plan arrays do not match its n_b, k and num_experts");
  // the device permutes follow inverse_pos; make sure it is the inverse of
  // (expanded_src_row, expanded_slot), as build_plan guarantees
  for (std::size_t i = 0; i < plan.n_b; ++i)
    for (std::size_t j = 0; j < plan.k; ++j) {
      const std::int64_t p = plan.inverse_pos(i, j);
      if (p < 0 || p >= (std::int64_t)nk || plan.expanded_src_row[p] != (std::int64_t)i ||
          plan.expanded_slot[p] != (std::int64_t)j)
        throw ShapeError(std::string(who) + ": inverse_pos is not the inverse of the expanded rows");
    }
  auto& d = local();
  std::vector<std::int64_t> off(plan.offsets);
  off.push_back((std::int64_t)nk);
  DevPlan r;
  r.counts = dropin::upload_i32(plan.counts.data(), E, d.stream, who);
  r.offsets = dropin::upload_i32(off.data(), E + 1, d.stream, who);
  r.src = dropin::upload_i32(plan.expanded_src_row.data(), nk, d.stream, who);
  r.slot = dropin::upload_i32(plan.expanded_slot.data(), nk, d.stream, who);
  r.inv = dropin::upload_i32(plan.inverse_pos.data(), nk, d.stream, who);
  r.p.n_b = (int64_t)plan.n_b;
  r.p.k = (int64_t)plan.k;
  r.p.n_experts = (int64_t)E;
  r.p.align = 1;
  r.p.capacity = (int64_t)nk;
  r.p.counts = r.counts.as<int32_t>();
  r.p.offsets = r.offsets.as<int32_t>();
  r.p.src_row = r.src.as<int32_t>();
  r.p.slot = r.slot.as<int32_t>();
  r.p.inverse_pos = r.inv.as<int32_t>();
  return r;
}
}  // namespace

DispatchPlan build_plan(const IndexMatrix& topk_indices, std::size_t num_experts) {
  DispatchPlan plan;
  plan.num_experts = num_experts;
  plan.n_b = topk_indices.rows();
  plan.k = topk_indices.cols();
  const std::size_t nk = plan.n_b * plan.k;
  for (std::size_t f = 0; f < nk; ++f) {
    const std::int64_t e = topk_indices.data()[f];
    if (e < 0 || e >= (std::int64_t)num_experts)
      throw ShapeError("build_plan: expert index " + std::to_string(e) + " out of range [0, " +
                       std::to_string(num_experts) + ")");
  }
  plan.counts.assign(num_experts, 0);
  plan.offsets.assign(num_experts, 0);
  plan.expanded_src_row.assign(nk, 0);
  plan.expanded_slot.assign(nk, 0);
  plan.inverse_pos = IndexMatrix(plan.n_b, plan.k);
  if (num_experts == 0) return plan;
  if (plan.k == 0) return plan;
  auto& d = local();
  int64_t cap = 0, scratch = 0;
  check(fmoe_plan_sizes((int64_t)plan.n_b, (int64_t)plan.k, (int64_t)num_experts, 1, &cap, &scratch));
  Buf di = dropin::upload_i32(topk_indices.data(), nk, d.stream, "build_plan");
  Buf counts(num_experts * 4, d.stream), offsets((num_experts + 1) * 4, d.stream), src(cap * 4, d.stream),
      slot(cap * 4, d.stream), inv(nk * 4, d.stream), scr(scratch, d.stream);
  fmoe_plan p{};
  p.n_b = (int64_t)plan.n_b;
  p.k = (int64_t)plan.k;
  p.n_experts = (int64_t)num_experts;
  p.align = 1;
  p.capacity = cap;
  p.counts = counts.as<int32_t>();
  p.offsets = offsets.as<int32_t>();
  p.src_row = src.as<int32_t>();
  p.slot = slot.as<int32_t>();
  p.inverse_pos = inv.as<int32_t>();
  p.scratch = scr.get();
  check(fmoe_plan_build(d.ctx, di.as<int32_t>(), &p, 1));
  plan.counts = dropin::download_i32(counts, num_experts, d);
  plan.offsets = dropin::download_i32(offsets, num_experts, d);
  plan.expanded_src_row = dropin::download_i32(src, nk, d);
  plan.expanded_slot = dropin::download_i32(slot, nk, d);
  const auto ip = dropin::download_i32(inv, nk, d);
  std::memcpy(plan.inverse_pos.data(), ip.data(), nk * 8);
  return plan;
}

Matrix scatter(const Matrix& x, const DispatchPlan& plan) {
  if (x.rows() != plan.n_b) throw ShapeError("scatter: input rows != plan batch size");
  Matrix xs(plan.n_b * plan.k, x.cols());
  if (xs.size() == 0) return xs;
  DevPlan dp = device_plan(plan, "scatter");
  auto& d = local();
  Buf dx = upload(x, d.stream), dxs(xs.size() * 8, d.stream);
  check(fmoe_scatter(d.ctx, FMOE_F64, dx.get(), (int64_t)x.cols(), &dp.p, dxs.get()));
  download(xs, dxs, d);
  return xs;
}

Matrix gather_combine(const Matrix& ys, const DispatchPlan& plan, const Matrix& topk_scores) {
  if (ys.rows() != plan.n_b * plan.k) throw ShapeError("gather_combine: ys rows != n_b * k");
  if (topk_scores.rows() != plan.n_b || topk_scores.cols() != plan.k)
    throw ShapeError("gather_combine: topk_scores shape mismatch");
  Matrix y(plan.n_b, ys.cols());
  if (y.size() == 0) return y;
  if (plan.k == 0) return y;
  DevPlan dp = device_plan(plan, "gather_combine");
  auto& d = local();
  Buf dys = upload(ys, d.stream), dw = upload(topk_scores, d.stream), dy(y.size() * 8, d.stream);
  check(fmoe_gather_combine(d.ctx, FMOE_F64, dys.get(), (int64_t)ys.cols(), &dp.p, dw.get(), dy.get()));
  download(y, dy, d);
  return y;
}

Matrix scatter_backward(const Matrix& d_xs, const DispatchPlan& plan) {
  if (d_xs.rows() != plan.n_b * plan.k) throw ShapeError("scatter_backward: rows != n_b * k");
  Matrix dx(plan.n_b, d_xs.cols());
  if (dx.size() == 0 || plan.k == 0) return dx;
  DevPlan dp = device_plan(plan, "scatter_backward");
  auto& d = local();
  Buf dxs = upload(d_xs, d.stream), ddx(dx.size() * 8, d.stream);
  check(fmoe_scatter_bwd(d.ctx, FMOE_F64, dxs.get(), (int64_t)d_xs.cols(), &dp.p, ddx.get()));
  download(dx, ddx, d);
  return dx;
}

GatherCombineGrads gather_combine_backward(const Matrix& d_y, const Matrix& ys, const DispatchPlan& plan,
                                           const Matrix& topk_scores) {
  if (d_y.rows() != plan.n_b) throw ShapeError("gather_combine_backward: d_y rows != n_b");
  if (ys.rows() != plan.n_b * plan.k || ys.cols() != d_y.cols())
    throw ShapeError("gather_combine_backward: ys shape mismatch");
  if (topk_scores.rows() != plan.n_b || topk_scores.cols() != plan.k)
    throw ShapeError("gather_combine_backward: topk_scores shape mismatch");
  GatherCombineGrads g{Matrix(plan.n_b * plan.k, d_y.cols()), Matrix(plan.n_b, plan.k)};
  if (plan.n_b == 0 || plan.k == 0) return g;
  DevPlan dp = device_plan(plan, "gather_combine_backward");
  auto& d = local();
  Buf ddy = upload(d_y, d.stream), dys = upload(ys, d.stream), dw = upload(topk_scores, d.stream);
  Buf ddys(g.d_ys.size() * 8, d.stream), ddw(g.d_topk_scores.size() * 8, d.stream);
  check(fmoe_gather_combine_bwd(d.ctx, FMOE_F64, ddy.get(), dys.get(), (int64_t)d_y.cols(), &dp.p, dw.get(),
                                ddys.get(), ddw.get()));
  download(g.d_ys, ddys, d);
  download(g.d_topk_scores, ddw, d);
  return g;
}

// ------------------------------------------------------------ expert pool
namespace {
struct Shapes {
  std::size_t dm = 0, dh = 0;
};

Shapes pool_shapes(std::span<const ExpertParams> experts, std::size_t dm_default, const char* who) {
  Shapes s{dm_default, 0};
  if (experts.empty()) return s;
  s.dm = experts[0].w1.rows();
  s.dh = experts[0].w1.cols();
  for (const auto& e : experts)
    if (e.w1.rows() != s.dm || e.w1.cols() != s.dh || e.b1.rows() != 1 || e.b1.cols() != s.dh ||
        e.w2.rows() != s.dh || e.w2.cols() != s.dm || e.b2.rows() != 1 || e.b2.cols() != s.dm)
      throw ShapeError(std::string(who) + ": expert parameter shapes disagree");
  return s;
}

std::vector<std::int64_t> block_offsets(std::span<const std::int64_t> counts, std::size_t rows, const char* who) {
  std::vector<std::int64_t> off(counts.size() + 1, 0);
  for (std::size_t e = 0; e < counts.size(); ++e) {
    if (counts[e] < 0) throw ShapeError(std::string(who) + ": negative block count");
    off[e + 1] = off[e] + counts[e];
  }
  if (off.back() != (std::int64_t)rows)
    throw ShapeError(std::string(who) + ": blocks cover " + std::to_string(off.back()) + " rows, input has " +
                     std::to_string(rows));
  return off;
}

// Stacked expert weights on the device ([E, d_m, d_h] etc., fmoe_expert_params).
struct DevPool {
  Buf w1, b1, w2, b2;
  fmoe_expert_params p{};
};
DevPool device_pool(std::span<const ExpertParams> experts, const Shapes& s, cudaStream_t st) {
  const std::size_t E = experts.size();
  DevPool P;
  P.w1 = Buf(E * s.dm * s.dh * 8, st);
  P.b1 = Buf(E * s.dh * 8, st);
  P.w2 = Buf(E * s.dh * s.dm * 8, st);
  P.b2 = Buf(E * s.dm * 8, st);
  // stacked [E, ...] copies: device-to-device for device-backed parameters
  // (after train_step), from the host values otherwise
  auto put = [&](const Matrix& m, Buf& b, std::size_t e, std::size_t n) {
    double* dst = b.as<double>() + e * n;
    if (const auto& ds = m.device_store())
      dropin::cuda(cudaMemcpyAsync(dst, ds->f64(m.device_offset()), n * 8, cudaMemcpyDeviceToDevice, st), "D2D");
    else if (n)
      dropin::cuda(cudaMemcpyAsync(dst, m.data(), n * 8, cudaMemcpyHostToDevice, st), "H2D");
  };
  for (std::size_t e = 0; e < E; ++e) {
    put(experts[e].w1, P.w1, e, s.dm * s.dh);
    put(experts[e].b1, P.b1, e, s.dh);
    put(experts[e].w2, P.w2, e, s.dh * s.dm);
    put(experts[e].b2, P.b2, e, s.dm);
  }
  dropin::cuda(cudaStreamSynchronize(st), "H2D sync");
  P.p = {P.w1.get(), P.b1.get(), P.w2.get(), P.b2.get()};
  return P;
}

// Device residency of the expert pool: the stacked weights of the last two
// pools a thread used stay on the device, keyed by every parameter Matrix's
// content identity (id, version) -- a forward and its backward, and steps of
// an unchanged state, upload the weights once instead of on every call
// (sgd_step / train_step write the weights and so bump their versions).
struct PoolKey {
  std::vector<std::uint64_t> v;
  bool operator==(const PoolKey&) const = default;
};
PoolKey pool_key(std::span<const ExpertParams> experts, const Shapes& s) {
  PoolKey k;
  k.v.reserve(experts.size() * 8 + 2);
  k.v.push_back(s.dm);
  k.v.push_back(s.dh);
  for (const auto& e : experts)
    for (const Matrix* m : {&e.w1, &e.b1, &e.w2, &e.b2}) {
      k.v.push_back(m->content_id());
      k.v.push_back(m->content_version());
    }
  return k;
}
const DevPool& device_pool_cached(std::span<const ExpertParams> experts, const Shapes& s, dropin::Device& d) {
  struct Entry {
    PoolKey key;
    DevPool pool;
    std::uint64_t used = 0;
  };
  thread_local Entry slots[2];  // after local(): destroyed before the thread's stream
  thread_local std::uint64_t clock = 0;
  PoolKey key = pool_key(experts, s);
  for (Entry& e : slots)
    if (e.used && e.key == key) {
      e.used = ++clock;
      return e.pool;
    }
  Entry& victim = slots[0].used <= slots[1].used ? slots[0] : slots[1];
  victim.pool = DevPool{};  // free before allocating the replacement
  victim.pool = device_pool(experts, s, d.stream);
  victim.key = std::move(key);
  victim.used = ++clock;
  return victim.pool;
}

// Block plan of a pool call: counts/offsets only (align 1).
struct DevBlocks {
  Buf counts, offsets;
  fmoe_plan p{};
};
DevBlocks device_blocks(std::span<const std::int64_t> counts, const std::vector<std::int64_t>& off,
                        cudaStream_t st) {
  DevBlocks b;
  const std::size_t E = counts.size();
  b.counts = dropin::upload_i32(counts.data(), E, st, "experts");
  b.offsets = dropin::upload_i32(off.data(), E + 1, st, "experts");
  b.p.n_b = off.back();
  b.p.k = 1;
  b.p.n_experts = (int64_t)E;
  b.p.align = 1;
  b.p.capacity = off.back();
  b.p.counts = b.counts.as<int32_t>();
  b.p.offsets = b.offsets.as<int32_t>();
  b.p.inverse_pos = b.offsets.as<int32_t>();  // unused by the expert kernels
  return b;
}

Matrix rows_of(const Matrix& m, std::size_t r0, std::size_t n) {
  Matrix out(n, m.cols());
  if (n) std::memcpy(out.data(), m.row_data(r0), n * m.cols() * 8);
  return out;
}
}  // namespace

MultiExpertResult multi_expert_forward(const Matrix& xs, std::span<const std::int64_t> counts,
                                       std::span<const ExpertParams> experts) {
  static const char* who = "multi_expert_forward";
  if (counts.size() != experts.size()) throw ShapeError("multi_expert_forward: counts and experts disagree");
  const auto off = block_offsets(counts, xs.rows(), who);
  const Shapes s = pool_shapes(experts, xs.cols(), who);
  if (!experts.empty() && xs.cols() != s.dm) throw ShapeError("expert_forward: input cols != d_m");
  MultiExpertResult r{Matrix(xs.rows(), s.dm), std::vector<ForwardCache>(experts.size())};
  const std::size_t n = xs.rows();
  Matrix pre(n, s.dh), hid(n, s.dh);
  if (n > 0) {
    auto& d = local();
    const DevPool& P = device_pool_cached(experts, s, d);
    DevBlocks B = device_blocks(counts, off, d.stream);
    Buf dx = upload(xs, d.stream), dpre(n * s.dh * 8, d.stream), dhid(n * s.dh * 8, d.stream),
        dys(n * s.dm * 8, d.stream);
    check(fmoe_experts_fwd_cached(d.ctx, FMOE_F64, &B.p, (int64_t)s.dm, (int64_t)s.dh, P.p, dx.get(), dpre.get(),
                                  dhid.get(), dys.get()));
    download(r.ys, dys, d);
    download(pre, dpre, d);
    download(hid, dhid, d);
  }
  for (std::size_t e = 0; e < experts.size(); ++e) {
    const std::size_t r0 = (std::size_t)off[e], c = (std::size_t)counts[e];
    r.caches[e] = ForwardCache{rows_of(xs, r0, c), rows_of(pre, r0, c), rows_of(hid, r0, c)};
  }
  return r;
}

MultiExpertGrads multi_expert_backward(const Matrix& d_ys, const std::vector<ForwardCache>& caches,
                                       std::span<const ExpertParams> experts) {
  static const char* who = "multi_expert_backward";
  if (caches.size() != experts.size()) throw ShapeError("multi_expert_backward: caches and experts disagree");
  std::vector<std::int64_t> counts(experts.size());
  for (std::size_t e = 0; e < experts.size(); ++e) counts[e] = (std::int64_t)caches[e].input.rows();
  const auto off = block_offsets(counts, d_ys.rows(), who);
  const Shapes s = pool_shapes(experts, d_ys.cols(), who);
  if (!experts.empty() && d_ys.cols() != s.dm) throw ShapeError("expert_backward: upstream gradient shape mismatch");
  const std::size_t n = d_ys.rows(), E = experts.size();
  Matrix xs(n, s.dm), pre(n, s.dh), hid(n, s.dh);
  for (std::size_t e = 0; e < E; ++e) {
    const ForwardCache& c = caches[e];
    const std::size_t rows = c.input.rows();
    if (c.input.cols() != s.dm || c.preact.rows() != rows || c.preact.cols() != s.dh || c.hidden.rows() != rows ||
        c.hidden.cols() != s.dh)
      throw ShapeError("expert_backward: cache shape mismatch");
    if (rows == 0) continue;
    std::memcpy(xs.row_data(off[e]), c.input.data(), rows * s.dm * 8);
    std::memcpy(pre.row_data(off[e]), c.preact.data(), rows * s.dh * 8);
    std::memcpy(hid.row_data(off[e]), c.hidden.data(), rows * s.dh * 8);
  }
  MultiExpertGrads g{Matrix(n, s.dm), std::vector<ExpertGrads>(E)};
  for (auto& eg : g.experts) eg = ExpertGrads{Matrix(s.dm, s.dh), Matrix(1, s.dh), Matrix(s.dh, s.dm), Matrix(1, s.dm)};
  if (E == 0) return g;
  auto& d = local();
  const DevPool& P = device_pool_cached(experts, s, d);
  DevBlocks B = device_blocks(counts, off, d.stream);
  Buf dx = upload(xs, d.stream), dpre = upload(pre, d.stream), dhid = upload(hid, d.stream),
      ddy = upload(d_ys, d.stream), ddx(n * s.dm * 8, d.stream);
  Buf gw1(E * s.dm * s.dh * 8, d.stream), gb1(E * s.dh * 8, d.stream), gw2(E * s.dh * s.dm * 8, d.stream),
      gb2(E * s.dm * 8, d.stream);
  fmoe_expert_grads G{gw1.get(), gb1.get(), gw2.get(), gb2.get()};
  check(fmoe_experts_bwd_cached(d.ctx, FMOE_F64, &B.p, (int64_t)s.dm, (int64_t)s.dh, P.p, dx.get(), dpre.get(),
                                dhid.get(), ddy.get(), ddx.get(), G));
  download(g.d_xs, ddx, d);
  for (std::size_t e = 0; e < E; ++e) {
    auto& eg = g.experts[e];
    download(eg.d_w1.data(), gw1.as<double>() + e * s.dm * s.dh, s.dm * s.dh * 8, d);
    download(eg.d_b1.data(), gb1.as<double>() + e * s.dh, s.dh * 8, d);
    download(eg.d_w2.data(), gw2.as<double>() + e * s.dh * s.dm, s.dh * s.dm * 8, d);
    download(eg.d_b2.data(), gb2.as<double>() + e * s.dm, s.dm * 8, d);
  }
  return g;
}

std::pair<Matrix, ForwardCache> expert_forward(const Matrix& x_block, const ExpertParams& params) {
  if (x_block.cols() != params.w1.rows()) throw ShapeError("expert_forward: input cols != d_m");
  const std::int64_t count = (std::int64_t)x_block.rows();
  MultiExpertResult r = multi_expert_forward(x_block, std::span<const std::int64_t>(&count, 1),
                                             std::span<const ExpertParams>(&params, 1));
  return {std::move(r.ys), std::move(r.caches[0])};
}

std::pair<Matrix, ExpertGrads> expert_backward(const Matrix& d_y, const ForwardCache& cache,
                                               const ExpertParams& params) {
  if (d_y.rows() != cache.input.rows() || d_y.cols() != params.w2.cols())
    throw ShapeError("expert_backward: upstream gradient shape mismatch");
  std::vector<ForwardCache> caches{cache};
  MultiExpertGrads g = multi_expert_backward(d_y, caches, std::span<const ExpertParams>(&params, 1));
  return {std::move(g.d_xs), std::move(g.experts[0])};
}

}  // namespace fmoe
