// ckpt.h -- the reference's weight-checkpoint file format ("FMOE-CKPT" v1,
// checkpoint.hpp:10-16 / checkpoint.cpp:63-122), host-side codec shared by
// the layer's device load/save (checkpoint.cpp) and the C++ drop-in.
//
//   "FMOE-CKPT\0" (10 bytes) | version u32 | n_b d_m d_h k n_e_local
//   world_size E_total seed (u64 each) | gate matrix | per global expert:
//   w1 b1 w2 b2 -- each matrix: rows u64, cols u64, rows*cols f64
// Little-endian throughout (the values are written byte by byte, so the file
// is identical on any host).  Errors are reported as (code, message) through
// CkptError; callers map them to their own exception types.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace fmoe_b200 {
namespace ckpt {

constexpr char kMagic[10] = {'F', 'M', 'O', 'E', '-', 'C', 'K', 'P', 'T', '\0'};
constexpr uint32_t kVersion = 1;

enum Code { SHAPE = 1, PROTOCOL = 2 };
struct CkptError {
  int code;
  std::string msg;
};

struct Header {
  uint64_t n_b = 0, d_m = 0, d_h = 0, k = 0, n_e_local = 0, world_size = 0, experts = 0, seed = 0;
};

class Writer {
 public:
  explicit Writer(const std::string& path) : path_(path), f_(std::fopen(path.c_str(), "wb")) {
    if (!f_) throw CkptError{PROTOCOL, "checkpoint: cannot open " + path + " for writing"};
  }
  ~Writer() {
    if (f_) std::fclose(f_);
  }
  void header(const Header& h) {
    raw(kMagic, sizeof(kMagic));
    u32(kVersion);
    for (uint64_t v : {h.n_b, h.d_m, h.d_h, h.k, h.n_e_local, h.world_size, h.experts, h.seed}) u64(v);
  }
  void matrix(uint64_t rows, uint64_t cols, const double* data) {
    u64(rows);
    u64(cols);
    const uint64_t n = rows * cols;
    buf_.resize(8 * std::min<uint64_t>(n, kChunk));
    for (uint64_t at = 0; at < n; at += kChunk) {
      const uint64_t m = std::min<uint64_t>(kChunk, n - at);
      for (uint64_t i = 0; i < m; ++i) le64(&buf_[8 * i], bits(data[at + i]));
      raw(buf_.data(), 8 * m);
    }
  }
  void close() {
    if (f_ && std::fclose(f_) != 0) {
      f_ = nullptr;
      throw CkptError{PROTOCOL, "checkpoint: write to " + path_ + " failed"};
    }
    f_ = nullptr;
  }

 private:
  static constexpr uint64_t kChunk = 1 << 16;
  static uint64_t bits(double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    return u;
  }
  static void le64(unsigned char* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (unsigned char)(v >> (8 * i));
  }
  void raw(const void* p, size_t n) {
    if (std::fwrite(p, 1, n, f_) != n) throw CkptError{PROTOCOL, "checkpoint: write to " + path_ + " failed"};
  }
  void u32(uint32_t v) {
    unsigned char b[4];
    for (int i = 0; i < 4; ++i) b[i] = (unsigned char)(v >> (8 * i));
    raw(b, 4);
  }
  void u64(uint64_t v) {
    unsigned char b[8];
    le64(b, v);
    raw(b, 8);
  }
  std::string path_;
  FILE* f_;
  std::vector<unsigned char> buf_;
};

class Reader {
 public:
  explicit Reader(const std::string& path) : path_(path), f_(std::fopen(path.c_str(), "rb")) {
    if (!f_) throw CkptError{PROTOCOL, "checkpoint: cannot open " + path};
    // the file length bounds every skip (fseek past EOF succeeds silently)
    if (std::fseek(f_, 0, SEEK_END) == 0) size_ = std::ftell(f_);
    std::fseek(f_, 0, SEEK_SET);
  }
  ~Reader() {
    if (f_) std::fclose(f_);
  }
  Header header() {
    char magic[10];
    if (std::fread(magic, 1, 10, f_) != 10 || std::memcmp(magic, kMagic, 10) != 0)
      throw CkptError{PROTOCOL, "checkpoint: bad header in " + path_};
    const uint32_t version = (uint32_t)uint_le(4, "header");
    if (version != kVersion) throw CkptError{PROTOCOL, "checkpoint: unsupported version " + std::to_string(version)};
    Header h;
    uint64_t* f[] = {&h.n_b, &h.d_m, &h.d_h, &h.k, &h.n_e_local, &h.world_size, &h.experts, &h.seed};
    for (uint64_t* p : f) *p = uint_le(8, "header");
    if (h.experts != h.n_e_local * h.world_size)
      throw CkptError{PROTOCOL, "checkpoint: inconsistent expert count in " + path_};
    return h;
  }
  // Reads the next matrix, which must be rows x cols, into out (may be NULL
  // to skip it).
  void matrix(uint64_t rows, uint64_t cols, double* out, const char* what) {
    const uint64_t r = uint_le(8, what), c = uint_le(8, what);
    if (r != rows || c != cols)
      throw CkptError{SHAPE, std::string("checkpoint: ") + what + " is " + std::to_string(r) + "x" +
                                 std::to_string(c) + ", expected " + std::to_string(rows) + "x" +
                                 std::to_string(cols)};
    const uint64_t n = rows * cols;
    if (!out) {
      const long at = std::ftell(f_);
      if (at < 0 || size_ < 0 || (uint64_t)(size_ - at) < 8 * n || std::fseek(f_, (long)(8 * n), SEEK_CUR) != 0)
        truncated(what);
      return;
    }
    buf_.resize(8 * std::min<uint64_t>(n, kChunk));
    for (uint64_t at = 0; at < n; at += kChunk) {
      const uint64_t m = std::min<uint64_t>(kChunk, n - at);
      if (std::fread(buf_.data(), 1, 8 * m, f_) != 8 * m) truncated(what);
      for (uint64_t i = 0; i < m; ++i) {
        uint64_t u = 0;
        for (int b = 0; b < 8; ++b) u |= (uint64_t)buf_[8 * i + b] << (8 * b);
        std::memcpy(out + at + i, &u, 8);
      }
    }
  }
  // Reads the next matrix of any shape.
  std::vector<double> matrix_any(uint64_t* rows, uint64_t* cols, const char* what) {
    const long pos = std::ftell(f_);
    *rows = uint_le(8, what);
    *cols = uint_le(8, what);
    std::fseek(f_, pos, SEEK_SET);
    std::vector<double> v(*rows * *cols);
    matrix(*rows, *cols, v.data(), what);
    return v;
  }

 private:
  static constexpr uint64_t kChunk = 1 << 16;
  [[noreturn]] void truncated(const char* what) {
    throw CkptError{PROTOCOL, std::string("checkpoint: truncated ") + what + " in " + path_};
  }
  uint64_t uint_le(int n, const char* what) {
    unsigned char b[8];
    if (std::fread(b, 1, (size_t)n, f_) != (size_t)n) truncated(what);
    uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= (uint64_t)b[i] << (8 * i);
    return v;
  }
  std::string path_;
  FILE* f_;
  long size_ = -1;
  std::vector<unsigned char> buf_;
};

}  // namespace ckpt
}  // namespace fmoe_b200
