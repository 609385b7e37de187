// common.cuh -- shared internals of libfmoe_b200.so (not part of the C-ABI).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <utility>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "fmoe_b200.h"

namespace fmoe_b200 {

// ----------------------------------------------------------------- errors
// Internal exceptions carry the C-ABI status; every extern "C" entry point
// converts them (capi.cu), so nothing escapes the boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void shape_error(const std::string& m) { throw Error(FMOE_ERR_SHAPE, m); }
[[noreturn]] inline void protocol_error(const std::string& m) { throw Error(FMOE_ERR_PROTOCOL, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw Error(FMOE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " at " + file +
                                   ":" + std::to_string(line));
}
#define CK(x) ::fmoe_b200::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH(ctx) \
  do {                 \
    (ctx)->launches++; \
    CK(cudaGetLastError()); \
  } while (0)

// ---------------------------------------------------------------- context
// Stage marks of one MoE-layer step (CUDA events on the layer's stream,
// recorded only while profiling is armed; read back after the timed region).
enum Mark : int {
  MARK_FWD_BEGIN = 0, MARK_GATE, MARK_PLAN, MARK_SCATTER, MARK_FC1, MARK_FC2, MARK_GATHER,
  MARK_BWD_BEGIN, MARK_GCB, MARK_DGRAD2, MARK_WGRAD2, MARK_DB2, MARK_DGRAD1, MARK_WGRAD1, MARK_DB1,
  MARK_GATE_DWG, MARK_GATE_DX, N_MARKS
};
// A stage's time runs from the mark recorded just before it in the same step
// (the issue order differs between paths), so prev[] keeps that mark's id.
// Each layer forward takes the next slot and its backward records into the
// same slot, so stacks of layers sharing one context profile per layer-step.
struct Prof {
  std::vector<cudaEvent_t> ev;  // [slots][N_MARKS]
  std::vector<int8_t> prev;     // [slots][N_MARKS]: preceding mark, -1 = not recorded
  std::vector<int8_t> last;     // [slots]: last mark recorded in the slot
  int steps = 0, used = 0;      // slots allocated / taken
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t launches = 0;
  int* d_error = nullptr;  // deferred device-side error flag (plan validation)
  struct Transport* transport = nullptr;  // EP exchange (comm.cuh); owned
  bool owns_transport = true;
  void* ws = nullptr;      // grow-only scratch for operator-level calls
  size_t ws_size = 0;
  void* pws = nullptr;     // grow-only bf16x3 operand planes of operator-level FMOE_F32 calls (f32x.cu)
  size_t pws_size = 0;
  int world = 1, rank = 0;
  Prof* prof = nullptr;
  int prof_slot = -1;      // slot of the layer step being issued (-1: none)
  // host-buffer steps (Layer::step_host): input / output copy engines run on
  // their own streams so PCIe transfers overlap the layer's kernels
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  cudaEvent_t ev_io[4] = {nullptr, nullptr, nullptr, nullptr};
  // SM clock probe of the expert GEMMs (fmoe_ctx_clock_probe): per launch,
  // CTA 0 records (clock64, globaltimer) at its start and end
  unsigned long long* d_probe = nullptr;
  int probe_cap = 0, probe_next = 0;
};

// Next clock-probe slot (4 u64) of the context, or NULL when not armed / full.
inline unsigned long long* ctx_probe_slot(Ctx* c) {
  if (!c->d_probe || c->probe_next >= c->probe_cap) return nullptr;
  return c->d_probe + 4 * (c->probe_next++);
}

inline void ctx_mark(Ctx* c, int id) {
  Prof* p = c->prof;
  if (!p || c->prof_slot < 0 || c->prof_slot >= p->used) return;
  const size_t base = (size_t)c->prof_slot * N_MARKS;
  // under stream capture the mark becomes an event-record node of the graph
  // (External), so replayed steps are timed like eager ones
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cs);
  cudaEventRecordWithFlags(p->ev[base + id], c->stream,
                           cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault);
  p->prev[base + id] = p->last[c->prof_slot];
  p->last[c->prof_slot] = (int8_t)id;
}
// A layer forward takes a new profiling slot (-1 when none is left).
inline int ctx_take_slot(Ctx* c) {
  Prof* p = c->prof;
  c->prof_slot = (p && p->used < p->steps) ? p->used++ : -1;
  return c->prof_slot;
}

// ------------------------------------------- programmatic dependent launch
// The single-GPU layer's kernels (plan, permutes, reduces, the tcgen05 GEMMs)
// are launched with programmatic stream serialization: the next grid is
// scheduled while the previous one drains and executes pdl_wait()
// (griddepcontrol.wait) before touching memory, so only launch latency and
// block setup (for the GEMMs: barriers, TMEM, tensor maps) overlap -- never
// data.  A profiling mark (event record) between two kernels disables the
// overlap there.  FMOE_PDL=0 launches plainly.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("FMOE_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ------------------------------------------------------------- type traits
template <typename T>
struct ScoreOf {
  using type = float;
};
template <>
struct ScoreOf<double> {
  using type = double;
};

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ double to_f(double v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <typename T>
__device__ __forceinline__ T from_d(double v);
template <>
__device__ __forceinline__ double from_d<double>(double v) { return v; }

inline size_t dtype_size(fmoe_dtype t) { return t == FMOE_F64 ? 8 : t == FMOE_F32 ? 4 : 2; }
inline size_t score_size(fmoe_dtype t) { return t == FMOE_F64 ? 8 : 4; }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int guard_status(const std::exception& e);
extern thread_local std::string g_last_error;

// Dispatch a templated functor on the runtime dtype.
template <typename F>
void dispatch_dtype(fmoe_dtype t, F&& f) {
  switch (t) {
    case FMOE_F64: f((double*)nullptr); break;
    case FMOE_F32: f((float*)nullptr); break;
    case FMOE_BF16: f((__nv_bfloat16*)nullptr); break;
    default: shape_error("unknown dtype");
  }
}

}  // namespace fmoe_b200
