// peer.cu -- see peer.cuh.
#include <cuda.h>
#include <unistd.h>

#include <cstring>
#include <mutex>
#include <string>

#include "peer.cuh"

namespace fmoe_b200 {

namespace {

constexpr uint64_t kMagic = 0x464d4f4550454552ull;  // "FMOEPEER"

struct Blob {
  uint64_t magic;
  int64_t host;
  int32_t pid, device;
  uint64_t ptr[PB_N];
  cudaIpcMemHandle_t h[PB_N];
};

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitFn wait_fn() {
  static WaitFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitFn>(p);
  });
  if (!fn) throw Error(FMOE_ERR_CUDA, "cuStreamWaitValue32 unavailable");
  return fn;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One block: flag slot (phase, r) := epoch on every rank.  The previous
// kernel on this stream (the producer) has completed, so its stores -- local
// and remote -- are performed before this kernel runs.
__global__ void signal_kernel(void* const* flags, int W, int r, int phase, uint32_t epoch) {
  __threadfence_system();
  for (int p = threadIdx.x; p < W; p += blockDim.x) {  // any world size
    uint32_t* f = reinterpret_cast<uint32_t*>(flags[p]) + phase * W + r;
    st_release_sys(f, epoch);
  }
}

// counts all-gather + PH_COUNTS flags in one kernel.
__global__ void put_counts_kernel(const int32_t* __restrict__ counts, int64_t E, void* const* mats,
                                  void* const* flags, int W, int r, uint32_t epoch) {
  for (int p = 0; p < W; ++p) {
    int32_t* dst = reinterpret_cast<int32_t*>(mats[p]) + (int64_t)r * E;
    for (int64_t g = threadIdx.x; g < E; g += blockDim.x) dst[g] = counts[g];
  }
  __syncthreads();
  if (threadIdx.x < W) {
    __threadfence_system();
    uint32_t* f = reinterpret_cast<uint32_t*>(flags[threadIdx.x]) + PH_COUNTS * W + r;
    st_release_sys(f, epoch);
  }
}

}  // namespace

size_t PeerSet::scratch_bytes(int W) { return sizeof(Blob) * (size_t)W + 64 + 4 * (size_t)W; }

size_t PeerSet::blob_bytes() { return sizeof(Blob); }

void PeerSet::make_blob(Ctx* ctx, void* const local[PB_N], void* out) {
  Blob mine{};
  mine.magic = kMagic;
  mine.host = (int64_t)gethostid();
  mine.pid = (int32_t)getpid();
  mine.device = ctx->device;
  for (int b = 0; b < PB_N; ++b) {
    mine.ptr[b] = reinterpret_cast<uint64_t>(local[b]);
    if (cudaIpcGetMemHandle(&mine.h[b], local[b]) != cudaSuccess) {
      cudaGetLastError();
      std::memset(&mine.h[b], 0, sizeof(mine.h[b]));  // peers of this process can still use the raw pointer
    }
  }
  std::memcpy(out, &mine, sizeof(Blob));
}

bool PeerSet::open(Ctx* ctx, int world, int rank, const void* blobs, void** ptr_table) {
  close();
  W = world;
  r = rank;
  const Blob* all = static_cast<const Blob*>(blobs);
  const Blob& mine = all[r];
  bool good = mine.magic == kMagic;
  cross_process = true;
  for (int p = 0; p < W; ++p)
    if (p != r && all[p].pid == mine.pid) cross_process = false;
  for (int b = 0; b < PB_N; ++b) ptr[b].assign(W, nullptr);
  for (int p = 0; p < W && good; ++p) {
    const Blob& o = all[p];
    if (o.magic != kMagic || o.host != mine.host) {
      good = false;
      break;
    }
    const bool same_proc = o.pid == mine.pid;
    if (o.device != ctx->device) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, ctx->device, o.device);
      if (!can) {
        good = false;
        break;
      }
      if (same_proc) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(o.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) good = false;
        cudaGetLastError();
      }
    }
    for (int b = 0; b < PB_N && good; ++b) {
      if (same_proc) {
        ptr[b][p] = reinterpret_cast<void*>(o.ptr[b]);
      } else {
        void* q = nullptr;
        if (cudaIpcOpenMemHandle(&q, o.h[b], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          good = false;
        } else {
          ptr[b][p] = q;
          opened.push_back(q);
        }
      }
    }
  }
  if (!good) {
    close();
    return false;
  }
  std::vector<void*> flat((size_t)PB_N * W);
  for (int b = 0; b < PB_N; ++b)
    for (int p = 0; p < W; ++p) flat[(size_t)b * W + p] = ptr[b][p];
  CK(cudaMemcpyAsync(ptr_table, flat.data(), flat.size() * sizeof(void*), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int b = 0; b < PB_N; ++b) d_ptr[b] = ptr_table + (size_t)b * W;
  ok = true;
  return true;
}

void PeerSet::connect(Ctx* ctx, Transport* tr, void* const local[PB_N], void* scratch, void** ptr_table) {
  close();
  const int world = tr->world, rank = tr->rank;
  // blob exchange over the transport (device buffers: NCCL moves device memory)
  const size_t B = sizeof(Blob);
  std::vector<uint8_t> host(B * world);
  make_blob(ctx, local, host.data() + B * rank);
  uint8_t* dev = static_cast<uint8_t*>(scratch);
  CK(cudaMemcpyAsync(dev + B * rank, host.data() + B * rank, B, cudaMemcpyHostToDevice, ctx->stream));
  std::vector<Xfer> sends, recvs;
  for (int p = 0; p < world; ++p)
    if (p != rank) {
      sends.push_back({p, dev + B * rank, B});
      recvs.push_back({p, dev + B * p, B});
    }
  tr->group(ctx, sends, recvs);
  CK(cudaMemcpyAsync(host.data(), dev, B * world, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const bool good = open(ctx, world, rank, host.data(), ptr_table);
  // agree: the fused path runs only if every rank mapped every peer (nothing
  // device-synchronising may follow this last rendezvous, see peer.cuh)
  int32_t* okv = reinterpret_cast<int32_t*>(dev + B * world + 64);
  const int32_t me_ok = good ? 1 : 0;
  CK(cudaMemcpyAsync(okv + rank, &me_ok, 4, cudaMemcpyHostToDevice, ctx->stream));
  sends.clear();
  recvs.clear();
  for (int p = 0; p < world; ++p)
    if (p != rank) {
      sends.push_back({p, okv + rank, 4});
      recvs.push_back({p, okv + p, 4});
    }
  tr->group(ctx, sends, recvs);
  std::vector<int32_t> oks(world);
  CK(cudaMemcpyAsync(oks.data(), okv, 4 * world, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  bool all_ok = true;
  for (int p = 0; p < world; ++p) all_ok = all_ok && oks[p] == 1;
  if (!all_ok) {
    close();
    return;
  }
  lw = tr->local_world();
  if (lw) {  // publish this rank's phase events, then rendezvous
    auto& ev = lw->slots[rank].phase;
    if (ev.empty()) {
      ev.resize(PH_N);
      for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    lw->barrier();
  }
}

void PeerSet::close() {
  for (void* q : opened) cudaIpcCloseMemHandle(q);
  opened.clear();
  lw = nullptr;
  cross_process = false;
  for (int b = 0; b < PB_N; ++b) {
    d_ptr[b] = nullptr;
    ptr[b].clear();
  }
  ok = false;
}

void PeerSet::signal(Ctx* ctx, int phase) {
  if (lw) {  // same process: record, then rendezvous so every wait sees the record
    CK(cudaEventRecord(lw->slots[r].phase[phase], ctx->stream));
    lw->barrier();
    return;
  }
  signal_kernel<<<1, 32, 0, ctx->stream>>>(d_ptr[PB_FLAGS], W, r, phase, epoch);
  CK_LAUNCH(ctx);
}

void PeerSet::wait(Ctx* ctx, int phase) {
  if (lw) {
    for (int p = 0; p < W; ++p)
      if (p != r) CK(cudaStreamWaitEvent(ctx->stream, lw->slots[p].phase[phase], 0));
    return;
  }
  auto fn = wait_fn();
  uint32_t* flags = reinterpret_cast<uint32_t*>(ptr[PB_FLAGS][r]);
  for (int p = 0; p < W; ++p) {
    if (p == r) continue;
    const CUresult e = fn(reinterpret_cast<CUstream>(ctx->stream),
                          reinterpret_cast<CUdeviceptr>(flags + phase * W + p), epoch, CU_STREAM_WAIT_VALUE_GEQ);
    if (e != CUDA_SUCCESS) throw Error(FMOE_ERR_CUDA, "cuStreamWaitValue32 failed (" + std::to_string((int)e) + ")");
  }
}

void PeerSet::put_counts(Ctx* ctx, const int32_t* counts, int64_t E) {
  put_counts_kernel<<<1, 256, 0, ctx->stream>>>(counts, E, d_ptr[PB_COUNTS], d_ptr[PB_FLAGS], W, r, epoch);
  CK_LAUNCH(ctx);
  if (lw) {
    CK(cudaEventRecord(lw->slots[r].phase[PH_COUNTS], ctx->stream));
    lw->barrier();
  }
}

}  // namespace fmoe_b200
