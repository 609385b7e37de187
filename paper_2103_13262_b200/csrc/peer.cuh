// peer.cuh -- NVLink peer memory for the expert-parallel layer.
//
// The reference's all_to_all_rows / all_to_all_rows_reverse
// (collectives.cpp:146-265) move rows between ranks as framed messages.  On
// one B200 node every rank can map its peers' buffers (CUDA IPC over
// NVLink/NVSwitch), so the exchanges are fused into the kernels that produce
// the rows: the scatter writes each token row straight into its expert's
// rank (global_scatter), the fc2 / dgrad-fc1 epilogues store every output row
// straight into the rank that sent it (global_gather), and the gather-combine
// backward writes d_ys into the expert ranks.  No staging copy and no
// collective kernel remain on the data path; the only synchronisation is a
// per-phase epoch flag each rank writes into its peers' memory after its
// producing kernel and waits on with a stream memory operation (no SM spins).
//
// Inside one process (the in-process world: all ranks may share one GPU and
// its hardware queues) a stream parked on a flag could sit in front of the
// very kernel that releases it, so there the phases are ordered with CUDA
// events recorded before a host rendezvous instead of flag waits; the data
// path (direct stores into peer buffers) is the same.
//
// Setup (PeerSet::connect) exchanges a small blob per rank -- raw pointers for
// ranks of the same process, CUDA IPC handles otherwise -- over the layer's
// Transport, so the same code serves the in-process world (the single-GPU
// tests) and one process per GPU (NCCL transport for the blob exchange only).
#pragma once

#include <vector>

#include "comm.cuh"
#include "common.cuh"

namespace fmoe_b200 {

enum PeerBuf : int { PB_XS = 0, PB_DYS, PB_YS, PB_DXS, PB_COUNTS, PB_FLAGS, PB_N };
// synchronisation phases of one step (a flag slot per phase and source rank)
enum PeerPhase : int { PH_COUNTS = 0, PH_SCATTER, PH_GATHER, PH_SCATTER_BWD, PH_GATHER_BWD, PH_N };

struct PeerSet {
  int W = 1, r = 0;
  bool ok = false;
  std::vector<void*> ptr[PB_N];    // [buf][rank] device pointers usable from this rank
  std::vector<void*> opened;       // IPC mappings to close
  void** d_ptr[PB_N] = {};         // device copies of ptr[buf] (W entries, in ptr_table)
  uint32_t epoch = 0;
  LocalWorld* lw = nullptr;        // same-process world: event-ordered phases
  // every peer lives in another process (one process per GPU, or processes
  // time-sharing one GPU): kernels may spin on peer-written flags without
  // starving the kernel that releases them (which the in-process world can)
  bool cross_process = false;

  // Exchange blobs over `tr`; every rank must call it with its local buffers.
  // On any failure every rank falls back together (ok = false everywhere).
  // `scratch` (>= scratch_bytes(W)) and `ptr_table` (PB_N * W pointers) are
  // device memory allocated up front: connect makes no device-synchronising
  // call (cudaMalloc / cudaFree), because a peer that already left connect may
  // have a stream parked on a flag wait that only this rank can release.
  void connect(Ctx* ctx, Transport* tr, void* const local[PB_N], void* scratch, void** ptr_table);
  static size_t scratch_bytes(int W);
  // The same in two halves for hosts that exchange the blobs themselves
  // (fmoe_layer_peer_blob / fmoe_layer_peer_connect): this rank's blob, and
  // opening every rank's blob (rank order).  open() returns false (and leaves
  // ok = false) if any peer cannot be mapped.
  static size_t blob_bytes();
  static void make_blob(Ctx* ctx, void* const local[PB_N], void* out);
  bool open(Ctx* ctx, int world, int rank, const void* blobs, void** ptr_table);
  void close();
  // Kernel-side flag write: epoch into slot (phase, r) of every peer's flags.
  void signal(Ctx* ctx, int phase);
  // Stream wait (cuStreamWaitValue32, no SM) until every peer signalled phase.
  void wait(Ctx* ctx, int phase);
  // counts all-gather: my E counts into row r of every rank's [W][E] matrix,
  // then signal PH_COUNTS (one kernel).
  void put_counts(Ctx* ctx, const int32_t* counts, int64_t E);
};

// Where the rows of one direction go (the fused global_scatter): slot (i, j)
// of token i with expert g lands in rank g_rank[g]'s buffer at row
// inverse_pos(i, j) + g_delta[g].
struct ScatterRoute {
  const int32_t* idx = nullptr;     // topk_idx [n_b, k]
  const int32_t* g_rank = nullptr;  // [E]
  const int64_t* g_delta = nullptr; // [E]
  void* const* dst = nullptr;       // [W] destination buffers
};

}  // namespace fmoe_b200
