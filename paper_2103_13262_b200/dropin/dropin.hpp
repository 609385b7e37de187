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
#include <vector>

#include "fmoe/matrix.hpp"
#include "fmoe_b200.h"

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

// Stream-ordered device allocation (cudaMallocAsync on the owner's stream).
class Buf {
 public:
  Buf() = default;
  Buf(std::size_t bytes, cudaStream_t s);
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
};

Buf upload(const void* host, std::size_t bytes, cudaStream_t s);
inline Buf upload(const Matrix& m, cudaStream_t s) { return upload(m.data(), m.size() * sizeof(double), s); }
Buf upload_i32(const std::int64_t* v, std::size_t n, cudaStream_t s, const char* what);
// Synchronous download (waits for the stream, then surfaces deferred errors).
void download(void* host, const void* dev, std::size_t bytes, const Device& d);
inline void download(Matrix& m, const Buf& b, const Device& d) {
  download(m.data(), b.get(), m.size() * sizeof(double), d);
}
std::vector<std::int64_t> download_i32(const Buf& b, std::size_t n, const Device& d);

}  // namespace fmoe::dropin
