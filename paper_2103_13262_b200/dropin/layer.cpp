// layer.cpp -- transports, collectives, gradient sync and the MoE layer of the
// drop-in (reference API: proj/include/fmoe/{transport,collectives,param_sync,
// moe_layer,checkpoint}.hpp).  The layer composes the drop-in operators in the
// reference's order (moe_layer.cpp:67-142), so each stage runs on the GPU
// through the C-ABI and the cache holds the reference's intermediates.
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>

#include "dropin.hpp"
#include "fmoe/checkpoint.hpp"
#include "ckpt.h"
#include "fmoe/collectives.hpp"
#include "fmoe/errors.hpp"
#include "fmoe/moe_layer.hpp"
#include "fmoe/param_sync.hpp"
#include "fmoe/rng.hpp"
#include "fmoe/transport.hpp"

namespace fmoe {

using dropin::Buf;
using dropin::check;

// ------------------------------------------------------------- transports
namespace {
// A rank's device context bound to a communicator (in-process or NCCL).
class DeviceTransport final : public Transport {
 public:
  DeviceTransport(int rank, int world, int device, std::shared_ptr<void> keep) : rank_(rank), world_(world),
                                                                                keep_(std::move(keep)) {
    dev_.device = device;
    dropin::cuda(cudaSetDevice(device), "cudaSetDevice");
    dropin::cuda(cudaStreamCreateWithFlags(&dev_.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    check(fmoe_ctx_create(device, dev_.stream, &dev_.ctx));
  }
  ~DeviceTransport() override {
    if (dev_.ctx) fmoe_ctx_destroy(dev_.ctx);
    if (dev_.stream) cudaStreamDestroy(dev_.stream);
  }
  int rank() const override { return rank_; }
  int world_size() const override { return world_; }
  fmoe_ctx* device_context() const override { return dev_.ctx; }
  cudaStream_t stream() const { return dev_.stream; }
  void barrier() override {
    // an empty-payload allreduce over the world is a rendezvous of every rank
    std::vector<int> all(world_);
    for (int r = 0; r < world_; ++r) all[r] = r;
    Buf one(8, dev_.stream);
    dropin::cuda(cudaMemsetAsync(one.get(), 0, 8, dev_.stream), "memset");
    check(fmoe_allreduce_sum(dev_.ctx, FMOE_F64, one.get(), 1, all.data(), world_));
    check(fmoe_ctx_check(dev_.ctx));
  }

 private:
  struct Raw {
    int device = 0;
    cudaStream_t stream = nullptr;
    fmoe_ctx* ctx = nullptr;
  } dev_;
  int rank_, world_;
  std::shared_ptr<void> keep_;
};

DeviceTransport& device_of(Transport& t) {
  auto* d = dynamic_cast<DeviceTransport*>(&t);
  if (!d) throw ProtocolError("fmoe drop-in: transport was not created by InProcWorld or nccl_connect");
  return *d;
}
}  // namespace

struct InProcWorld::Shared {
  fmoe_world* world = nullptr;
  int size = 0;
  ~Shared() {
    if (world) fmoe_world_destroy(world);
  }
};

InProcWorld::InProcWorld(int world_size) : shared_(std::make_shared<Shared>()) {
  if (world_size < 1) throw ShapeError("InProcWorld: world size must be at least 1");
  shared_->size = world_size;
  check(fmoe_world_create(world_size, &shared_->world));
}
InProcWorld::~InProcWorld() = default;
int InProcWorld::world_size() const { return shared_->size; }

std::unique_ptr<Transport> InProcWorld::transport(int rank) {
  if (rank < 0 || rank >= shared_->size) throw ShapeError("InProcWorld: rank out of range");
  auto t = std::make_unique<DeviceTransport>(rank, shared_->size, dropin::default_device(), shared_);
  check(fmoe_ctx_join_world(t->device_context(), shared_->world, rank));
  return t;
}

std::vector<std::uint8_t> nccl_unique_id() {
  std::vector<std::uint8_t> id(128);
  check(fmoe_comm_unique_id(id.data(), (int64_t)id.size()));
  return id;
}

std::unique_ptr<Transport> nccl_connect(int rank, int world_size, const std::vector<std::uint8_t>& id, int device) {
  if (device < 0) device = dropin::default_device();
  auto t = std::make_unique<DeviceTransport>(rank, world_size, device, nullptr);
  check(fmoe_comm_init(t->device_context(), id.data(), (int64_t)id.size(), world_size, rank));
  return t;
}

std::vector<HostPort> localhost_endpoints(int world_size, std::uint16_t base_port) {
  std::vector<HostPort> v;
  for (int r = 0; r < world_size; ++r) v.push_back({"127.0.0.1", static_cast<std::uint16_t>(base_port + r)});
  return v;
}

std::unique_ptr<Transport> tcp_connect(int, const std::vector<HostPort>&, std::chrono::milliseconds) {
  throw TransportError("tcp_connect: the B200 drop-in exchanges rows over NCCL; use nccl_connect");
}

// ------------------------------------------------------------ collectives
std::vector<std::int64_t> ExchangePlan::local_expert_rows() const {
  std::vector<std::int64_t> rows(local_experts, 0);
  for (int s = 0; s < world; ++s)
    for (std::size_t e = 0; e < local_experts; ++e) rows[e] += recv_count(s, e);
  return rows;
}

ExchangePlan exchange_counts(std::span<const std::int64_t> local_counts, Transport& transport) {
  DeviceTransport& t = device_of(transport);
  transport.next_tag();
  const std::size_t n = local_counts.size();
  const int W = t.world_size();
  if (n % (std::size_t)W != 0)
    throw ShapeError("exchange_counts: " + std::to_string(n) + " experts not divisible by world size " +
                     std::to_string(W));
  ExchangePlan plan;
  plan.rank = t.rank();
  plan.world = W;
  plan.local_experts = n / (std::size_t)W;
  plan.send_counts.assign(n, 0);
  plan.recv_counts.assign(n, 0);
  if (n == 0) return plan;
  fmoe_exchange_plan c{};
  c.send_counts = plan.send_counts.data();
  c.recv_counts = plan.recv_counts.data();
  check(fmoe_exchange_counts(t.device_context(), local_counts.data(), (int64_t)n, &c));
  plan.send_total = c.send_total;
  plan.recv_total = c.recv_total;
  return plan;
}

namespace {
Matrix a2a(const Matrix& in, const ExchangePlan& plan, Transport& transport, bool forward) {
  DeviceTransport& t = device_of(transport);
  transport.next_tag();
  const std::int64_t expect = forward ? plan.send_total : plan.recv_total;
  const std::int64_t out_rows = forward ? plan.recv_total : plan.send_total;
  const char* who = forward ? "all_to_all_rows" : "all_to_all_rows_reverse";
  if ((std::int64_t)in.rows() != expect)
    throw ProtocolError(std::string(who) + ": input rows " + std::to_string(in.rows()) + " != plan total " +
                        std::to_string(expect));
  if (plan.world != t.world_size() || plan.rank != t.rank())
    throw ProtocolError(std::string(who) + ": plan belongs to another rank or world");
  Matrix out((std::size_t)out_rows, in.cols());
  std::vector<std::int64_t> send(plan.send_counts), recv(plan.recv_counts);
  fmoe_exchange_plan c{plan.world, plan.rank, (int64_t)plan.local_experts, send.data(), recv.data(),
                       plan.send_total, plan.recv_total};
  cudaStream_t s = t.stream();
  Buf din = dropin::upload(in, s), dout(out.size() * 8, s);
  check(forward ? fmoe_a2a_rows(t.device_context(), FMOE_F64, din.get(), (int64_t)in.cols(), &c, dout.get())
                : fmoe_a2a_rows_reverse(t.device_context(), FMOE_F64, din.get(), (int64_t)in.cols(), &c, dout.get()));
  if (out.size()) dropin::cuda(cudaMemcpyAsync(out.data(), dout.get(), out.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
  check(fmoe_ctx_check(t.device_context()));
  return out;
}
}  // namespace

Matrix all_to_all_rows(const Matrix& xs, const ExchangePlan& plan, Transport& transport) {
  return a2a(xs, plan, transport, true);
}
Matrix all_to_all_rows_reverse(const Matrix& ys, const ExchangePlan& plan, Transport& transport) {
  return a2a(ys, plan, transport, false);
}

Matrix allreduce_sum(const Matrix& m, std::span<const int> group, Transport& transport) {
  DeviceTransport& t = device_of(transport);
  transport.next_tag();
  if (group.empty()) throw ProtocolError("allreduce_sum: empty group");
  Matrix out = m;
  cudaStream_t s = t.stream();
  Buf b = dropin::upload_copy(m, s);  // reduced in place: a private copy
  check(fmoe_allreduce_sum(t.device_context(), FMOE_F64, b.get(), (int64_t)m.size(), group.data(),
                           (int64_t)group.size()));
  if (out.size()) dropin::cuda(cudaMemcpyAsync(out.data(), b.get(), out.size() * 8, cudaMemcpyDeviceToHost, s), "D2H");
  check(fmoe_ctx_check(t.device_context()));
  return out;
}

// ------------------------------------------------------------ param sync
std::optional<std::vector<int>> resolve_group(ParamTag tag, const ProcessTopology& topology, int rank) {
  const int W = topology.world_size, mp = topology.model_parallel_size;
  if (W < 1 || mp < 1 || W % mp != 0)
    throw ShapeError("resolve_group: model parallel size " + std::to_string(mp) + " does not divide world " +
                     std::to_string(W));
  if (rank < 0 || rank >= W) throw ShapeError("resolve_group: rank out of range");
  std::vector<int> g;
  if (tag == ParamTag::NoSync) return std::nullopt;
  // World: every rank; DataParallel: the ranks with the same model-parallel slot
  const int first = tag == ParamTag::World ? 0 : rank % mp, step = tag == ParamTag::World ? 1 : mp;
  for (int r = first; r < W; r += step) g.push_back(r);
  return g;
}

void sync_gradients(std::vector<TaggedGrad>& grads, const ProcessTopology& topology, Transport* transport) {
  if (transport && transport->world_size() != topology.world_size)
    throw ProtocolError("sync_gradients: topology world " + std::to_string(topology.world_size) +
                        " != transport world " + std::to_string(transport->world_size()));
  const int rank = transport ? transport->rank() : 0;
  for (auto& g : grads) {
    if (!g.grad) throw ShapeError("sync_gradients: null gradient " + g.name);
    const auto group = resolve_group(g.tag, topology, rank);
    if (!transport || !group || group->size() < 2) continue;
    Matrix sum = allreduce_sum(*g.grad, *group, *transport);
    scale_inplace(sum, 1.0 / static_cast<double>(group->size()));
    *g.grad = std::move(sum);
  }
}

void sgd_step(Matrix& param, const Matrix& grad, double lr) {
  if (!param.same_shape(grad)) throw ShapeError("sgd_step: parameter/gradient shape mismatch");
  axpy_inplace(param, -lr, grad);
}

// ---------------------------------------------------------------- layer
namespace {
void validate(const MoEConfig& c) {
  if (c.n_b < 1 || c.d_m < 1 || c.d_h < 1 || c.n_e_local < 1 || c.world_size < 1)
    throw ShapeError("MoEConfig: all dimensions must be at least 1");
  if (c.k < 1 || c.k > c.total_experts()) throw ShapeError("MoEConfig: k must lie in [1, total experts]");
}
}  // namespace

MoELayerState init_state(const MoEConfig& config, int rank) {
  validate(config);
  if (rank < 0 || (std::size_t)rank >= config.world_size) throw ShapeError("init_state: rank out of range");
  MoELayerState s;
  s.config = config;
  s.topology = {(int)config.world_size, 1};
  s.rank = rank;
  s.gate = init_gate(config.d_m, config.total_experts(), config.seed);
  for (std::size_t slot = 0; slot < config.n_e_local; ++slot)
    s.experts.push_back(init_expert(config.d_m, config.d_h,
                                    stream_seed(config.seed, (std::uint64_t)rank * config.n_e_local + slot)));
  return s;
}

Matrix naive_forward(const Matrix& x, const MoELayerState& state) {
  const MoEConfig& c = state.config;
  if (c.world_size != 1 || state.experts.size() != c.total_experts())
    throw ShapeError("naive_forward: needs a single-worker state holding every expert");
  if (x.cols() != c.d_m) throw ShapeError("naive_forward: input cols != d_m");
  Matrix y(x.rows(), c.d_m);
  for (std::size_t i = 0; i < x.rows(); ++i) {
    Matrix xi(1, c.d_m);
    std::memcpy(xi.data(), x.row_data(i), c.d_m * 8);
    const GateOutput g = gate_forward(xi, state.gate, c.k);
    for (std::size_t j = 0; j < c.k; ++j) {
      const auto [yi, cache] = expert_forward(xi, state.experts[(std::size_t)g.topk_indices(0, j)]);
      const double w = g.topk_scores(0, j);
      for (std::size_t col = 0; col < c.d_m; ++col) y(i, col) = std::fma(w, yi(0, col), y(i, col));
    }
  }
  return y;
}

Matrix forward(const Matrix& x, const MoELayerState& state, Transport* transport, MoEForwardCache* cache) {
  const MoEConfig& c = state.config;
  if (x.cols() != c.d_m) throw ShapeError("forward: input cols != d_m");
  const bool ep = transport && c.world_size > 1;
  if (ep && transport->world_size() != (int)c.world_size)
    throw ProtocolError("forward: transport world != config world");
  if (!ep && state.experts.size() != c.total_experts())
    throw ShapeError("forward: single-worker call needs all experts local");
  if (!ep)
    if (auto y = dropin::fast_forward(x, state, cache)) return std::move(*y);  // device-resident route (fast.cpp)

  GateOutput gate_out = gate_forward(x, state.gate, c.k);
  DispatchPlan plan = build_plan(gate_out.topk_indices, c.total_experts());
  const Matrix xs = scatter(x, plan);
  std::optional<ExchangePlan> exchange;
  std::vector<std::int64_t> blocks;
  MultiExpertResult run;
  Matrix ys;
  if (ep) {
    exchange = exchange_counts(plan.counts, *transport);
    blocks = exchange->local_expert_rows();
    run = multi_expert_forward(all_to_all_rows(xs, *exchange, *transport), blocks, state.experts);
    ys = all_to_all_rows_reverse(run.ys, *exchange, *transport);
  } else {
    blocks = plan.counts;
    run = multi_expert_forward(xs, blocks, state.experts);
    ys = std::move(run.ys);
  }
  Matrix y = gather_combine(ys, plan, gate_out.topk_scores);
  if (cache) {
    cache->input = x;
    cache->gate_out = std::move(gate_out);
    cache->plan = std::move(plan);
    cache->exchange = std::move(exchange);
    cache->local_block_counts = std::move(blocks);
    cache->expert_outputs = std::move(ys);
    cache->expert_caches = std::move(run.caches);
  }
  return y;
}

std::pair<Matrix, MoEGrads> backward(const Matrix& d_y, const MoEForwardCache& cache, const MoELayerState& state,
                                     Transport* transport) {
  const bool ep = cache.exchange.has_value();
  if (ep && !transport) throw ProtocolError("backward: cache came from a distributed forward, transport required");
  if (!ep)
    if (auto r = dropin::fast_backward(d_y, cache, state)) return std::move(*r);  // device-resident route
  GatherCombineGrads comb = gather_combine_backward(d_y, cache.expert_outputs, cache.plan, cache.gate_out.topk_scores);
  MoEGrads grads;
  Matrix d_xs;
  if (ep) {
    MultiExpertGrads run = multi_expert_backward(all_to_all_rows(comb.d_ys, *cache.exchange, *transport),
                                                 cache.expert_caches, state.experts);
    grads.experts = std::move(run.experts);
    d_xs = all_to_all_rows_reverse(run.d_xs, *cache.exchange, *transport);
  } else {
    MultiExpertGrads run = multi_expert_backward(comb.d_ys, cache.expert_caches, state.experts);
    grads.experts = std::move(run.experts);
    d_xs = std::move(run.d_xs);
  }
  Matrix d_x = scatter_backward(d_xs, cache.plan);
  GateGrads g = gate_backward(cache.input, state.gate, cache.gate_out, comb.d_topk_scores);
  grads.d_wg = std::move(g.d_wg);
  add_inplace(d_x, g.d_x);
  return {std::move(d_x), std::move(grads)};
}

double train_step(const Matrix& x, const Matrix& target, MoELayerState& state, double lr, Transport* transport) {
  if (!(transport && state.config.world_size > 1) && state.experts.size() == state.config.total_experts())
    if (auto loss = dropin::fast_train_step(x, target, state, lr)) return *loss;  // one device step (fast.cpp)
  MoEForwardCache cache;
  const Matrix y = forward(x, state, transport, &cache);
  if (!target.same_shape(y)) throw ShapeError("train_step: target shape != output shape");
  // local mean-squared error (the reported loss is the world average)
  const double n = static_cast<double>(y.size());
  double loss = 0.0;
  Matrix d_y(y.rows(), y.cols());
  for (std::size_t i = 0; i < y.size(); ++i) {
    const double diff = y.data()[i] - target.data()[i];
    loss += diff * diff / n;
    d_y.data()[i] = 2.0 * diff / n;
  }
  auto [d_x, grads] = backward(d_y, cache, state, transport);
  (void)d_x;
  const bool ep = transport && state.config.world_size > 1;
  if (ep) {
    // experts saw the whole world's rows while each rank normalised by its own batch
    const double inv = 1.0 / static_cast<double>(state.config.world_size);
    for (auto& e : grads.experts)
      for (Matrix* m : {&e.d_w1, &e.d_b1, &e.d_w2, &e.d_b2}) scale_inplace(*m, inv);
  }
  std::vector<TaggedGrad> tagged{{"gate.w_g", &grads.d_wg, state.gate.tag}};
  for (std::size_t s = 0; s < state.experts.size(); ++s) {
    const std::string p = "expert." + std::to_string(s) + ".";
    const ParamTag tag = state.experts[s].tag;
    auto& e = grads.experts[s];
    tagged.push_back({p + "w1", &e.d_w1, tag});
    tagged.push_back({p + "b1", &e.d_b1, tag});
    tagged.push_back({p + "w2", &e.d_w2, tag});
    tagged.push_back({p + "b2", &e.d_b2, tag});
  }
  sync_gradients(tagged, state.topology, ep ? transport : nullptr);
  sgd_step(state.gate.w_g, grads.d_wg, lr);
  for (std::size_t s = 0; s < state.experts.size(); ++s) {
    auto& p = state.experts[s];
    auto& e = grads.experts[s];
    sgd_step(p.w1, e.d_w1, lr);
    sgd_step(p.b1, e.d_b1, lr);
    sgd_step(p.w2, e.d_w2, lr);
    sgd_step(p.b2, e.d_b2, lr);
  }
  if (ep) {
    Matrix l(1, 1);
    l(0, 0) = loss;
    const auto group = resolve_group(ParamTag::World, state.topology, state.rank);
    loss = allreduce_sum(l, *group, *transport)(0, 0) / static_cast<double>(state.config.world_size);
  }
  return loss;
}

ToyTask make_toy_task(const MoEConfig& config) {
  validate(config);
  const std::size_t rows = config.n_b * config.world_size;
  ToyTask t{Matrix(rows, config.d_m), Matrix(rows, config.d_m)};
  UniformRng(stream_seed(config.seed, 0x746F7969ULL)).fill(t.inputs, -1.0, 1.0);  // "toyi"
  Matrix teacher(config.d_m, config.d_m);
  UniformRng(stream_seed(config.seed, 0x746F7974ULL)).fill(teacher, -0.5, 0.5);  // "toyt"
  t.targets = matmul(t.inputs, teacher);
  // mild nonlinearity; the reference build contracts t += (0.1*x)*x into one fma
  for (std::size_t i = 0; i < t.targets.size(); ++i) {
    const double xv = t.inputs.data()[i];
    t.targets.data()[i] = std::fma(0.1 * xv, xv, t.targets.data()[i]);
  }
  return t;
}

// ------------------------------------------------------------ checkpoint
// The reference's file format through the shared codec (csrc/ckpt.h); the
// Matrix values are written / read bit for bit (f64).
namespace {
[[noreturn]] void ckpt_rethrow(const fmoe_b200::ckpt::CkptError& e) {
  if (e.code == fmoe_b200::ckpt::SHAPE) throw ShapeError(e.msg);
  throw ProtocolError(e.msg);
}
void ckpt_write(fmoe_b200::ckpt::Writer& out, const Matrix& m) { out.matrix(m.rows(), m.cols(), m.data()); }
Matrix ckpt_read(fmoe_b200::ckpt::Reader& in, const char* what) {
  uint64_t r = 0, c = 0;
  std::vector<double> v = in.matrix_any(&r, &c, what);
  Matrix m(r, c);
  std::copy(v.begin(), v.end(), m.data());
  return m;
}
}  // namespace

void save_checkpoint(const std::string& path, const MoEConfig& config, const GateParams& gate,
                     std::span<const ExpertParams> experts) {
  if (experts.size() != config.total_experts())
    throw ShapeError("save_checkpoint: expert list must cover every global index");
  try {
    fmoe_b200::ckpt::Writer out(path);
    fmoe_b200::ckpt::Header h;
    h.n_b = config.n_b;
    h.d_m = config.d_m;
    h.d_h = config.d_h;
    h.k = config.k;
    h.n_e_local = config.n_e_local;
    h.world_size = config.world_size;
    h.experts = config.total_experts();
    h.seed = config.seed;
    out.header(h);
    ckpt_write(out, gate.w_g);
    for (const ExpertParams& e : experts) {
      ckpt_write(out, e.w1);
      ckpt_write(out, e.b1);
      ckpt_write(out, e.w2);
      ckpt_write(out, e.b2);
    }
    out.close();
  } catch (const fmoe_b200::ckpt::CkptError& e) {
    ckpt_rethrow(e);
  }
}

Checkpoint load_checkpoint(const std::string& path) {
  Checkpoint c;
  try {
    fmoe_b200::ckpt::Reader in(path);
    const fmoe_b200::ckpt::Header h = in.header();
    c.config.n_b = h.n_b;
    c.config.d_m = h.d_m;
    c.config.d_h = h.d_h;
    c.config.k = h.k;
    c.config.n_e_local = h.n_e_local;
    c.config.world_size = h.world_size;
    c.config.seed = h.seed;
    c.gate.w_g = ckpt_read(in, "gate w_g");
    c.gate.tag = ParamTag::World;
    c.experts.resize(h.experts);
    for (auto& e : c.experts) {
      e.w1 = ckpt_read(in, "expert w1");
      e.b1 = ckpt_read(in, "expert b1");
      e.w2 = ckpt_read(in, "expert w2");
      e.b2 = ckpt_read(in, "expert b2");
      e.tag = ParamTag::NoSync;
    }
  } catch (const fmoe_b200::ckpt::CkptError& e) {
    ckpt_rethrow(e);
  }
  return c;
}

}  // namespace fmoe
