// comm.cu -- transports for expert parallelism (see comm.cuh).
#include <nccl.h>

#include <chrono>
#include <cstring>

#include <string>

#include "comm.cuh"

namespace fmoe_b200 {

// ------------------------------------------------------------- local world
LocalWorld::LocalWorld(int w) : world(w), slots(w) {
  for (auto& s : slots) {
    CK(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
  }
}

LocalWorld::~LocalWorld() {
  for (auto& s : slots) {
    cudaEventDestroy(s.ready);
    cudaEventDestroy(s.done);
    for (auto e : s.phase) cudaEventDestroy(e);
  }
}

void LocalWorld::barrier() {
  std::unique_lock<std::mutex> lk(m);
  const uint64_t gen = generation;
  if (++arrived == world) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != gen; })) {
    // a peer never arrived (it failed or issued a different collective):
    // TransportError like the reference's rendezvous timeout (transport_tcp.cpp:242-244)
    throw Error(FMOE_ERR_TRANSPORT, "in-process world: barrier timed out waiting for peers");
  }
}

namespace {

struct LocalTransport : Transport {
  LocalWorld* w;
  LocalTransport(LocalWorld* lw, int r) : w(lw) {
    rank = r;
    world = lw->world;
  }
  LocalWorld* local_world() override { return w; }
  void group(Ctx* ctx, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs) override {
    auto& me = w->slots[rank];
    me.sends.clear();
    for (const auto& s : sends)
      if (s.bytes) me.sends.push_back(s);
    CK(cudaEventRecord(me.ready, ctx->stream));
    w->barrier();  // every rank has published its sends
    std::vector<size_t> cursor(world, 0);
    std::vector<char> waited(world, 0);
    for (const auto& r : recvs) {
      if (!r.bytes) continue;
      auto& peer = w->slots[r.peer];
      // next send of `peer` addressed to me
      size_t& c = cursor[r.peer];
      while (c < peer.sends.size() && peer.sends[c].peer != rank) ++c;
      if (c >= peer.sends.size()) protocol_error("local transport: rank " + std::to_string(r.peer) +
                                                 " sent fewer chunks than rank " + std::to_string(rank) + " expects");
      const Xfer& s = peer.sends[c++];
      if (s.bytes != r.bytes)
        protocol_error("local transport: rank " + std::to_string(r.peer) + " sent " + std::to_string(s.bytes) +
                       " bytes, plan expects " + std::to_string(r.bytes));
      if (!waited[r.peer]) {
        CK(cudaStreamWaitEvent(ctx->stream, peer.ready, 0));
        waited[r.peer] = 1;
      }
      CK(cudaMemcpyAsync(r.ptr, s.ptr, r.bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CK(cudaEventRecord(me.done, ctx->stream));
    w->barrier();  // all copies enqueued
    // senders may reuse their buffers only after every receiver has copied
    for (int p = 0; p < world; ++p)
      if (p != rank) CK(cudaStreamWaitEvent(ctx->stream, w->slots[p].done, 0));
    w->barrier();  // nobody republishes before all have waited
  }
};

#define NCK(x)                                                                                     \
  do {                                                                                             \
    ncclResult_t r_ = (x);                                                                         \
    if (r_ != ncclSuccess)                                                                         \
      throw Error(FMOE_ERR_TRANSPORT, std::string("NCCL: ") + ncclGetErrorString(r_) + " in " #x); \
  } while (0)

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  NcclTransport(const void* id, int w, int r) {
    world = w;
    rank = r;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    NCK(ncclCommInitRank(&comm, w, uid, r));
  }
  bool owned = true;
  // a communicator the caller created (e.g. the host framework's): borrowed
  explicit NcclTransport(ncclComm_t c) : comm(c), owned(false) {
    NCK(ncclCommCount(comm, &world));
    NCK(ncclCommUserRank(comm, &rank));
  }
  ~NcclTransport() override {
    if (comm && owned) ncclCommDestroy(comm);
  }
  void group(Ctx* ctx, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs) override {
    NCK(ncclGroupStart());
    for (const auto& s : sends)
      if (s.bytes) NCK(ncclSend(s.ptr, s.bytes, ncclUint8, s.peer, comm, ctx->stream));
    for (const auto& r : recvs)
      if (r.bytes) NCK(ncclRecv(r.ptr, r.bytes, ncclUint8, r.peer, comm, ctx->stream));
    NCK(ncclGroupEnd());
  }
};

}  // namespace

Transport* make_local_transport(LocalWorld* w, int rank) { return new LocalTransport(w, rank); }

Transport* make_nccl_transport(const void* id, int world, int rank) { return new NcclTransport(id, world, rank); }

Transport* attach_nccl_transport(void* comm) { return new NcclTransport(reinterpret_cast<ncclComm_t>(comm)); }

int nccl_unique_id(void* out, size_t bytes) {
  if (bytes < sizeof(ncclUniqueId)) shape_error("unique id buffer too small (need 128 bytes)");
  ncclUniqueId uid;
  NCK(ncclGetUniqueId(&uid));
  std::memcpy(out, &uid, sizeof(uid));
  return (int)sizeof(uid);
}

}  // namespace fmoe_b200
