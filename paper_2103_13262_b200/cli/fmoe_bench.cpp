// fmoe_bench.cpp -- the reference's benchmark CLI (tools/fmoe_bench.cpp) for
// the B200 layer: same subcommands, flags, inputs and CSV schema
//   scenario,n_b,d_m,d_h,n_e,k,world,reps,mean_ms,stddev_ms,gflops
// (fmoe_bench.cpp:36-37, 94-107), so CPU and GPU rows land in one table.
// Host data come from the reference's generators (the drop-in's
// UniformRng / stream_seed / init_state / make_toy_task); every step runs on
// device through the C-ABI (include/fmoe_b200.h).  Timing: CUDA events on the
// layer stream around each repetition after the warm-up rounds, mean and
// sample stddev as measure() (fmoe_bench.cpp:44-63).
//
//   fmoe_bench bench-local [--n-b N --d-m D --d-h H --k K --n-e E[,E...]
//                           --seed S --reps R --warmup W --out F --dtype bf16|f32|f64]
//   fmoe_bench bench-dist  --world W [...]     one thread + GPU per rank, NCCL,
//                                              expert parallelism (fused peer exchange)
//   fmoe_bench train-toy   --steps T --lr LR [--world W ...]   step,loss rows
// Exit codes as the reference: 0 ok, 2 usage / shape error, 3 transport error, 1 other.
#include <cuda_runtime.h>

#include <cmath>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fmoe/moe_layer.hpp"
#include "fmoe/rng.hpp"
#include "fmoe_b200.h"

namespace {

constexpr const char* kCsvHeader = "scenario,n_b,d_m,d_h,n_e,k,world,reps,mean_ms,stddev_ms,gflops";

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(int rc) {
  if (rc != FMOE_OK) throw Fail(rc == FMOE_ERR_SHAPE ? 2 : rc == FMOE_ERR_TRANSPORT ? 3 : 1, fmoe_last_error());
}
void cu(cudaError_t e) {
  if (e != cudaSuccess) throw Fail(1, cudaGetErrorString(e));
}

struct Opts {
  size_t n_b = 1024, d_m = 256, d_h = 1024, k = 2, n_e = 4;
  std::vector<size_t> n_e_list;
  uint64_t seed = 42;
  int reps = 16, warmup = 2, world = 1, steps = 20;
  double lr = 0.05;
  std::string out, dtype = "bf16";
  std::string api = "device";  // bench-local: device (C-ABI layer) | reference (fmoe::forward/backward)
};

fmoe_dtype dtype_of(const std::string& s) {
  if (s == "bf16") return FMOE_BF16;
  if (s == "f32") return FMOE_F32;
  if (s == "f64") return FMOE_F64;
  throw Fail(2, "--dtype must be bf16, f32 or f64");
}
size_t esize(fmoe_dtype t) { return t == FMOE_F64 ? 8 : t == FMOE_F32 ? 4 : 2; }

uint64_t default_seed() {
  if (const char* env = std::getenv("FMOE_SEED")) {
    char* end = nullptr;
    const unsigned long long v = std::strtoull(env, &end, 10);
    if (end != env) return v;
  }
  return 42;
}

Opts parse(int argc, char** argv, int first) {
  Opts o;
  o.seed = default_seed();
  for (int i = first; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw Fail(2, a + " needs a value");
      return argv[++i];
    };
    auto num = [&]() { return (size_t)std::stoull(val()); };
    if (a == "--n-b") o.n_b = num();
    else if (a == "--d-m") o.d_m = num();
    else if (a == "--d-h") o.d_h = num();
    else if (a == "--k") o.k = num();
    else if (a == "--n-e") {
      std::stringstream ss(val());
      std::string item;
      o.n_e_list.clear();
      while (std::getline(ss, item, ',')) o.n_e_list.push_back(std::stoull(item));
      if (!o.n_e_list.empty()) o.n_e = o.n_e_list[0];
    } else if (a == "--seed") o.seed = std::stoull(val());
    else if (a == "--reps") o.reps = std::stoi(val());
    else if (a == "--warmup") o.warmup = std::stoi(val());
    else if (a == "--out") o.out = val();
    else if (a == "--world") o.world = std::stoi(val());
    else if (a == "--steps") o.steps = std::stoi(val());
    else if (a == "--lr") o.lr = std::stod(val());
    else if (a == "--dtype") o.dtype = val();
    else if (a == "--api") o.api = val();
    else throw Fail(2, "unknown flag " + a);
  }
  if (o.reps < 1 || o.warmup < 0 || o.world < 1) throw Fail(2, "--reps >= 1, --warmup >= 0, --world >= 1");
  if (o.n_e_list.empty()) o.n_e_list.push_back(o.n_e);
  return o;
}

// ------------------------------------------------------------ CSV output
std::string hardware_line() {
  int dev = 0;
  cudaDeviceProp p{};
  cu(cudaGetDevice(&dev));
  cu(cudaGetDeviceProperties(&p, dev));
  int n = 0;
  cu(cudaGetDeviceCount(&n));
  return std::string("# hardware: ") + p.name + ", " + std::to_string(p.multiProcessorCount) + " SMs, " +
         std::to_string(n) + " GPU(s) visible";
}

struct Csv {
  std::ofstream file;
  std::ostream* os = &std::cout;
  explicit Csv(const std::string& path) {
    if (!path.empty()) {
      file.open(path);
      if (!file) throw Fail(1, "cannot open output file " + path);
      os = &file;
    }
  }
  std::ostream& out() { return *os; }
};

struct Timing {
  double mean_ms = 0, stddev_ms = 0;
};

void row(std::ostream& out, const char* scenario, const Opts& o, size_t n_e, int world, const Timing& t,
         double flops) {
  out << scenario << ',' << o.n_b << ',' << o.d_m << ',' << o.d_h << ',' << n_e << ',' << o.k << ',' << world << ','
      << o.reps << ',' << t.mean_ms << ',' << t.stddev_ms << ',' << flops / (t.mean_ms * 1e-3) / 1e9 << "\n";
}

// fmoe_bench.cpp:110-126
double flops_fwd(const Opts& o, size_t total) {
  return 2.0 * o.n_b * o.d_m * total + 4.0 * o.n_b * o.k * o.d_m * o.d_h;
}
double flops_bwd(const Opts& o, size_t total) {
  return 4.0 * o.n_b * o.d_m * total + 8.0 * o.n_b * o.k * o.d_m * o.d_h;
}

// ------------------------------------------------------------ device layer
// Rank r's layer on device `dev` with the reference inputs of stream
// (x_stream, dy_stream) converted to the layer dtype.
struct Rank {
  int dev = 0;
  cudaStream_t stream = nullptr;
  fmoe_ctx* ctx = nullptr;
  fmoe_layer* layer = nullptr;
  void *x = nullptr, *dy = nullptr, *y = nullptr, *dx = nullptr, *target = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;

  void create(int device, const fmoe_layer_config& cfg) {
    dev = device;
    cu(cudaSetDevice(dev));
    cu(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    cu(cudaEventCreate(&e0));
    cu(cudaEventCreate(&e1));
    ck(fmoe_ctx_create(dev, stream, &ctx));
    ck(fmoe_layer_create(ctx, &cfg, &layer));
    ck(fmoe_layer_init_weights(layer));  // init_state(config, rank)
    const size_t bytes = cfg.n_b * cfg.d_m * esize(cfg.dtype);
    for (void** p : {&x, &dy, &y, &dx, &target}) cu(cudaMalloc(p, bytes));
  }
  void upload(void* dst, const fmoe::Matrix& m, fmoe_dtype t) {
    std::vector<uint8_t> buf(m.size() * esize(t));
    for (size_t i = 0; i < m.size(); ++i) {
      const double v = m.data()[i];
      if (t == FMOE_F64) std::memcpy(&buf[8 * i], &v, 8);
      else if (t == FMOE_F32) { const float f = (float)v; std::memcpy(&buf[4 * i], &f, 4); }
      else {  // round to nearest even bf16 of the fp32 value
        const float f = (float)v;
        uint32_t u;
        std::memcpy(&u, &f, 4);
        const uint16_t b = (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
        std::memcpy(&buf[2 * i], &b, 2);
      }
    }
    cu(cudaMemcpy(dst, buf.data(), buf.size(), cudaMemcpyHostToDevice));
  }
  void destroy() {
    if (layer) fmoe_layer_destroy(layer);
    if (ctx) fmoe_ctx_destroy(ctx);
    for (void* p : {x, dy, y, dx, target})
      if (p) cudaFree(p);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (stream) cudaStreamDestroy(stream);
  }
};

fmoe::Matrix seeded(uint64_t seed, uint64_t stream, size_t rows, size_t cols) {
  fmoe::UniformRng rng(fmoe::stream_seed(seed, stream));
  fmoe::Matrix m(rows, cols);
  rng.fill(m, -1.0, 1.0);
  return m;
}

template <typename F>
Timing measure(Rank& r, int warmup, int reps, F&& fn) {
  for (int i = 0; i < warmup; ++i) fn();
  std::vector<double> s;
  for (int i = 0; i < reps; ++i) {
    cu(cudaEventRecord(r.e0, r.stream));
    fn();
    cu(cudaEventRecord(r.e1, r.stream));
    cu(cudaEventSynchronize(r.e1));
    float ms = 0;
    cu(cudaEventElapsedTime(&ms, r.e0, r.e1));
    s.push_back(ms);
  }
  Timing t;
  for (double v : s) t.mean_ms += v;
  t.mean_ms /= reps;
  double var = 0;
  for (double v : s) var += (v - t.mean_ms) * (v - t.mean_ms);
  t.stddev_ms = reps > 1 ? std::sqrt(var / (reps - 1)) : 0.0;
  return t;
}

// ------------------------------------------------------------ subcommands
// bench-local --api reference: the reference's own moe_batched_forward /
// moe_batched_fwdbwd loops (fmoe_bench.cpp:210-253, host steady_clock timing)
// over its C++ API -- init_state, forward, backward of include/fmoe/
// moe_layer.hpp with host Matrix values -- served by libfmoe_dropin.so on the
// GPU in FMOE_F64 (bit-identical to the reference library), weights resident
// on the device between calls.
template <typename F>
Timing measure_host(int warmup, int reps, F&& fn) {
  for (int i = 0; i < warmup; ++i) fn();
  std::vector<double> s;
  for (int i = 0; i < reps; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    fn();
    s.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  Timing t;
  for (double v : s) t.mean_ms += v;
  t.mean_ms /= reps;
  double var = 0;
  for (double v : s) var += (v - t.mean_ms) * (v - t.mean_ms);
  t.stddev_ms = reps > 1 ? std::sqrt(var / (reps - 1)) : 0.0;
  return t;
}

int bench_local_reference_api(const Opts& o) {
  Csv csv(o.out);
  csv.out() << hardware_line()
            << "\n# api: reference C++ API (fmoe::init_state / forward / backward, include/fmoe/moe_layer.hpp) "
               "through libfmoe_dropin.so, FMOE_F64, host timing\n"
            << kCsvHeader << "\n";
  for (size_t n_e : o.n_e_list) {
    if (n_e == 0 || o.k > n_e) throw Fail(2, "bench-local: need 1 <= k <= n_e");
    const fmoe::MoEConfig config{o.n_b, o.d_m, o.d_h, o.k, n_e, 1, o.seed};
    const fmoe::MoELayerState state = fmoe::init_state(config);
    const fmoe::Matrix x = seeded(o.seed, 102, o.n_b, o.d_m);
    const fmoe::Matrix d_y = seeded(o.seed, 103, o.n_b, o.d_m);
    fmoe::Matrix sink;
    const Timing fwd = measure_host(o.warmup, o.reps, [&] { sink = fmoe::forward(x, state); });
    row(csv.out(), "moe_batched_forward", o, n_e, 1, fwd, flops_fwd(o, n_e));
    const Timing both = measure_host(o.warmup, o.reps, [&] {
      fmoe::MoEForwardCache cache;
      sink = fmoe::forward(x, state, nullptr, &cache);
      fmoe::backward(d_y, cache, state);
    });
    row(csv.out(), "moe_batched_fwdbwd", o, n_e, 1, both, flops_fwd(o, n_e) + flops_bwd(o, n_e));
    // the same step with y and d_x read on the host (device-backed results
    // are copied down on first access): what a caller that consumes them pays
    double sum = 0.0;
    const Timing host = measure_host(o.warmup, o.reps, [&] {
      fmoe::MoEForwardCache cache;
      const fmoe::Matrix y = fmoe::forward(x, state, nullptr, &cache);
      const fmoe::Matrix dx = fmoe::backward(d_y, cache, state).first;
      sum += y.data()[0] + dx.data()[0];
    });
    row(csv.out(), "moe_batched_fwdbwd_host_results", o, n_e, 1, host, flops_fwd(o, n_e) + flops_bwd(o, n_e));
    if (sum != sum) std::cerr << "nan\n";
  }
  return 0;
}

int bench_local(const Opts& o) {
  if (o.api == "reference") return bench_local_reference_api(o);
  if (o.api != "device") throw Fail(2, "--api must be device or reference");
  const fmoe_dtype t = dtype_of(o.dtype);
  Csv csv(o.out);
  csv.out() << hardware_line() << "\n# dtype: " << o.dtype << ", device timing (CUDA events)\n" << kCsvHeader << "\n";
  for (size_t n_e : o.n_e_list) {
    if (n_e == 0 || o.k > n_e) throw Fail(2, "bench-local: need 1 <= k <= n_e");
    fmoe_layer_config cfg{(int64_t)o.n_b, (int64_t)o.d_m, (int64_t)o.d_h, (int64_t)o.k, (int64_t)n_e, 1, 0,
                          o.seed, t};
    Rank r;
    r.create(0, cfg);
    r.upload(r.x, seeded(o.seed, 102, o.n_b, o.d_m), t);  // fmoe_bench.cpp:226-227
    r.upload(r.dy, seeded(o.seed, 103, o.n_b, o.d_m), t);
    const Timing fwd = measure(r, o.warmup, o.reps, [&] { ck(fmoe_layer_fwd(r.layer, r.x, r.y)); });
    row(csv.out(), "moe_batched_forward", o, n_e, 1, fwd, flops_fwd(o, n_e));
    const Timing both = measure(r, o.warmup, o.reps, [&] {
      ck(fmoe_layer_fwd(r.layer, r.x, r.y));
      ck(fmoe_layer_bwd(r.layer, r.dy, r.dx));
    });
    row(csv.out(), "moe_batched_fwdbwd", o, n_e, 1, both, flops_fwd(o, n_e) + flops_bwd(o, n_e));
    r.destroy();
  }
  return 0;
}

// Ranks as threads, one GPU each (device = rank % visible devices), one NCCL
// communicator; every rank runs the reference's bench-dist iteration.
int bench_dist(const Opts& o) {
  const fmoe_dtype t = dtype_of(o.dtype);
  const int W = o.world;
  int ndev = 0;
  cu(cudaGetDeviceCount(&ndev));
  if (W > 1 && ndev < W) throw Fail(2, "bench-dist: needs one GPU per rank (" + std::to_string(ndev) + " visible)");
  std::vector<uint8_t> id(128);
  if (W > 1) ck(fmoe_comm_unique_id(id.data(), 128));
  std::vector<Timing> res(W);
  std::vector<std::string> errs(W);
  std::vector<int> codes(W, 0);
  auto body = [&](int rank) {
    Rank r;
    try {
      fmoe_layer_config cfg{(int64_t)o.n_b, (int64_t)o.d_m, (int64_t)o.d_h, (int64_t)o.k, (int64_t)o.n_e, W, rank,
                            o.seed, t};
      r.create(rank % std::max(ndev, 1), cfg);
      if (W > 1) ck(fmoe_comm_init(r.ctx, id.data(), 128, W, rank));
      r.upload(r.x, seeded(o.seed, 200 + rank, o.n_b, o.d_m), t);  // fmoe_bench.cpp:259-262
      r.upload(r.dy, seeded(o.seed, 300 + rank, o.n_b, o.d_m), t);
      res[rank] = measure(r, o.warmup, o.reps, [&] {
        ck(fmoe_layer_fwd(r.layer, r.x, r.y));
        ck(fmoe_layer_bwd(r.layer, r.dy, r.dx));
      });
      cu(cudaStreamSynchronize(r.stream));
    } catch (const Fail& e) {
      errs[rank] = e.what();
      codes[rank] = e.code;
    } catch (const std::exception& e) {
      errs[rank] = e.what();
      codes[rank] = 1;
    }
    r.destroy();
  };
  std::vector<std::thread> th;
  for (int rank = 0; rank < W; ++rank) th.emplace_back(body, rank);
  for (auto& x : th) x.join();
  for (int rank = 0; rank < W; ++rank)
    if (codes[rank]) throw Fail(codes[rank], "rank " + std::to_string(rank) + ": " + errs[rank]);
  Timing agg;  // world average of mean and stddev, as the reference's allreduce
  for (const auto& v : res) {
    agg.mean_ms += v.mean_ms / W;
    agg.stddev_ms += v.stddev_ms / W;
  }
  Csv csv(o.out);
  csv.out() << hardware_line() << "\n# dtype: " << o.dtype << ", device timing (CUDA events)\n" << kCsvHeader << "\n";
  const size_t total = o.n_e * W;
  row(csv.out(), "moe_dist_fwdbwd", o, o.n_e, W, agg, (flops_fwd(o, total) + flops_bwd(o, total)) * W);
  return 0;
}

// train-toy (fmoe_bench.cpp:303-336): --n-b is the global batch; every step is
// fmoe_layer_train_step (forward, MSE, backward, gradient sync, SGD).
int train_toy(const Opts& o) {
  const fmoe_dtype t = dtype_of(o.dtype);
  const int W = o.world;
  if (o.n_b % W) throw Fail(2, "train-toy: --n-b is the global batch and must divide by --world");
  int ndev = 0;
  cu(cudaGetDeviceCount(&ndev));
  if (W > 1 && ndev < W) throw Fail(2, "train-toy: needs one GPU per rank");
  fmoe::MoEConfig mc{o.n_b / W, o.d_m, o.d_h, o.k, o.n_e, (size_t)W, o.seed};
  const fmoe::ToyTask task = fmoe::make_toy_task(mc);
  std::vector<uint8_t> id(128);
  if (W > 1) ck(fmoe_comm_unique_id(id.data(), 128));
  std::vector<std::vector<double>> losses(W);
  std::vector<std::string> errs(W);
  std::vector<int> codes(W, 0);
  auto body = [&](int rank) {
    Rank r;
    try {
      fmoe_layer_config cfg{(int64_t)mc.n_b, (int64_t)o.d_m, (int64_t)o.d_h, (int64_t)o.k, (int64_t)o.n_e, W,
                            rank, o.seed, t};
      r.create(rank % std::max(ndev, 1), cfg);
      if (W > 1) ck(fmoe_comm_init(r.ctx, id.data(), 128, W, rank));
      fmoe::Matrix x(mc.n_b, o.d_m), y(mc.n_b, o.d_m);
      const size_t row0 = mc.n_b * rank;
      for (size_t i = 0; i < mc.n_b; ++i)
        for (size_t c = 0; c < o.d_m; ++c) {
          x(i, c) = task.inputs(row0 + i, c);
          y(i, c) = task.targets(row0 + i, c);
        }
      r.upload(r.x, x, t);
      r.upload(r.target, y, t);
      for (int s = 0; s < o.steps; ++s) {
        double loss = 0;
        ck(fmoe_layer_train_step(r.layer, r.x, r.target, o.lr, &loss));
        losses[rank].push_back(loss);
      }
    } catch (const Fail& e) {
      errs[rank] = e.what();
      codes[rank] = e.code;
    } catch (const std::exception& e) {
      errs[rank] = e.what();
      codes[rank] = 1;
    }
    r.destroy();
  };
  std::vector<std::thread> th;
  for (int rank = 0; rank < W; ++rank) th.emplace_back(body, rank);
  for (auto& x : th) x.join();
  for (int rank = 0; rank < W; ++rank)
    if (codes[rank]) throw Fail(codes[rank], "rank " + std::to_string(rank) + ": " + errs[rank]);
  Csv csv(o.out);
  csv.out() << "step,loss\n";
  csv.out().precision(17);
  for (int s = 0; s < o.steps; ++s) csv.out() << s << ',' << losses[0][s] << "\n";
  return 0;
}

int usage() {
  std::cerr << "usage: fmoe_bench {bench-local|bench-dist|train-toy} [--n-b N --d-m D --d-h H --k K --n-e E[,E..]\n"
               "                  --seed S --reps R --warmup W --out FILE --world W --steps T --lr LR\n"
               "                  --dtype bf16|f32|f64] [bench-local: --api device|reference]\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string cmd = argv[1];
  try {
    const Opts o = parse(argc, argv, 2);
    if (cmd == "bench-local") return bench_local(o);
    if (cmd == "bench-dist") return bench_dist(o);
    if (cmd == "train-toy") return train_toy(o);
    return usage();
  } catch (const Fail& e) {
    std::cerr << "fmoe_bench: " << e.what() << "\n";
    return e.code;
  } catch (const std::exception& e) {
    std::cerr << "fmoe_bench: " << e.what() << "\n";
    return 2;
  }
}
