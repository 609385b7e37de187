// comm.cuh -- point-to-point transport for expert parallelism.
//
// The reference builds its collectives on a Transport of framed messages
// (transport.hpp:18-38) with two worlds: in-process mailboxes and TCP.  The
// B200 analogue keeps the SPMD contract (every rank issues the same grouped
// exchange in the same order) with two transports:
//   * NcclTransport  -- ncclGroupStart / ncclSend / ncclRecv / ncclGroupEnd on
//                       the layer's stream, over NVLink/NVSwitch; one process
//                       per GPU (production path).
//   * LocalTransport -- W ranks as host threads of one process (the
//                       reference's run_world_inproc test pattern), possibly
//                       on one device; rows move with cudaMemcpyAsync after a
//                       host rendezvous.  Used to test the EP data path on a
//                       single GPU.
// Self-transfers never reach the transport; the layer copies them locally
// (collectives.cpp:160-171).
#pragma once

#include <condition_variable>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace fmoe_b200 {

struct Xfer {
  int peer;
  void* ptr;
  size_t bytes;
};

struct Transport {
  int rank = 0, world = 1;
  virtual ~Transport() = default;
  // One grouped exchange.  For every ordered pair (a, b) the i-th send of a
  // to b is matched with the i-th recv of b from a; sizes must agree
  // (ProtocolError otherwise).  Zero-byte entries are skipped on both sides.
  virtual void group(Ctx* ctx, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs) = 0;
  // The in-process world behind this transport (nullptr for NCCL).
  virtual struct LocalWorld* local_world() { return nullptr; }
};

struct LocalWorld {
  explicit LocalWorld(int w);
  ~LocalWorld();
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  struct Slot {
    std::vector<Xfer> sends;
    cudaEvent_t ready = nullptr, done = nullptr;
    std::vector<cudaEvent_t> phase;  // peer-memory phase events of the rank (peer.cuh)
  };
  std::vector<Slot> slots;
  void barrier();
};

Transport* make_local_transport(LocalWorld* w, int rank);
Transport* make_nccl_transport(const void* id, int world, int rank);
// Borrow an existing ncclComm_t (world / rank read from it; not destroyed).
Transport* attach_nccl_transport(void* comm);
int nccl_unique_id(void* out, size_t bytes);

}  // namespace fmoe_b200
