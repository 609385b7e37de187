// dropin.hpp -- internals of libfmoe_dropin.so, the C++ drop-in for the
// reference's include/fmoe/*.hpp API over the C-ABI of libfmoe_b200.so.
//
// Every operator uploads its host Matrix arguments, runs the C-ABI entry point
// in the FMOE_F64 parity mode on the calling thread's context and downloads
// the result (value semantics, like the reference).  Status codes become the
// reference's exception types.  No operator computes on the host.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <utility>
#include <vector>

#include "fmoe/matrix.hpp"
#include "fmoe/moe_layer.hpp"
#include "fmoe_b200.h"

namespace fmoe::detail {
// Device values behind a device-backed Matrix (fmoe/matrix.hpp): a
// stream-ordered allocation from the device's memory pool, freed when the last
// Matrix referring to it goes away.  Every drop-in call synchronises its
// stream before returning, so no queued work can still touch a store whose
// last reference is dropped outside a call.
struct DeviceStore {
  void* ptr = nullptr;
  std::size_t bytes = 0;
  int device = 0;
  DeviceStore() = default;
  DeviceStore(const DeviceStore&) = delete;
  DeviceStore& operator=(const DeviceStore&) = delete;
  ~DeviceStore();
  double* f64(std::size_t offset = 0) const { return static_cast<double*>(ptr) + offset; }
};
}  // namespace fmoe::detail

namespace fmoe::dropin {

// Throws ShapeError / ProtocolError / TransportError / std::runtime_error for
// a non-zero C-ABI status, with fmoe_last_error() as the message.
void check(int status);
void cuda(cudaError_t e, const char* what);

// One C-ABI context + stream per host thread, on FMOE_DEVICE (default 0).
struct Device {
  int device = 0;
  cudaStream_t stream = nullptr;
  fmoe_ctx* ctx = nullptr;
  Device();
  ~Device();
};
Device& local();
int default_device();

// Stream-ordered device allocation (cudaMallocAsync on the owner's stream), or
// a non-owning view of device memory kept alive elsewhere (Buf::view).
class Buf {
 public:
  Buf() = default;
  Buf(std::size_t bytes, cudaStream_t s);
  static Buf view(const void* p) {
    Buf b;
    b.p_ = const_cast<void*>(p);
    b.owned_ = false;
    return b;
  }
  ~Buf();
  Buf(Buf&& o) noexcept;
  Buf& operator=(Buf&& o) noexcept;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  void* get() const { return p_; }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p_);
  }

 private:
  void* p_ = nullptr;
  cudaStream_t s_ = nullptr;
  bool owned_ = true;
};

Buf upload(const void* host, std::size_t bytes, cudaStream_t s);
// Read-only device copy of m: a view of its device values when it has them
// (no transfer), else an upload of the host values.  Never write through it.
Buf upload(const Matrix& m, cudaStream_t s);
// A private, writable device copy of m (device-to-device when m has one).
Buf upload_copy(const Matrix& m, cudaStream_t s);
// A device store of `bytes` for results produced on d.stream.
std::shared_ptr<detail::DeviceStore> device_store(std::size_t bytes, const struct Device& d);
// rows x cols f64 result backed by `store` at element offset `off`.
inline Matrix device_matrix(std::size_t rows, std::size_t cols, std::shared_ptr<const detail::DeviceStore> store,
                            std::size_t off = 0) {
  return Matrix::on_device(rows, cols, std::move(store), off);
}
Buf upload_i32(const std::int64_t* v, std::size_t n, cudaStream_t s, const char* what);
// Synchronous download (waits for the stream, then surfaces deferred errors).
void download(void* host, const void* dev, std::size_t bytes, const Device& d);
inline void download(Matrix& m, const Buf& b, const Device& d) {
  download(m.data(), b.get(), m.size() * sizeof(double), d);
}
std::vector<std::int64_t> download_i32(const Buf& b, std::size_t n, const Device& d);

// Device-resident route of the MoE layer (fast.cpp): nullopt when it does not
// apply (expert parallelism, FMOE_DROPIN_PATH=ops, a cache it did not make).
std::optional<Matrix> fast_forward(const Matrix& x, const MoELayerState& state, MoEForwardCache* cache);
std::optional<std::pair<Matrix, MoEGrads>> fast_backward(const Matrix& d_y, const MoEForwardCache& cache,
                                                         const MoELayerState& state);
std::optional<double> fast_train_step(const Matrix& x, const Matrix& target, MoELayerState& state, double lr);

}  // namespace fmoe::dropin
