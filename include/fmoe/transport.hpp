// fmoe/transport.hpp -- the communicator handed to the distributed operators
// (reference: proj/include/fmoe/transport.hpp:14-68).
//
// The reference moves framed byte messages over in-process mailboxes or TCP.
// The B200 drop-in moves device rows instead: a Transport wraps a C-ABI
// context (include/fmoe_b200.h) joined either to an NCCL communicator over
// NVLink/NVSwitch (one process per GPU, nccl_connect) or to an in-process
// world of host threads (InProcWorld, the reference's test pattern).  The SPMD
// contract is unchanged: every rank issues the same collectives in the same
// order.  TCP rendezvous is not provided (tcp_connect throws TransportError).
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "fmoe/wire.hpp"

struct fmoe_ctx;  // include/fmoe_b200.h

namespace fmoe {

class Transport {
 public:
  virtual ~Transport() = default;
  virtual int rank() const = 0;
  virtual int world_size() const = 0;
  virtual void barrier() = 0;
  // Framed byte messages (transport.hpp:25-30 of the reference) are not how
  // the drop-in moves data: both throw TransportError (see fmoe/wire.hpp).
  virtual void send_frame(int peer, MsgType type, std::uint32_t tag, std::span<const std::byte> payload);
  virtual std::vector<std::byte> recv_frame(int peer, MsgType expected_type, std::uint32_t expected_tag);
  // C-ABI context (device, stream, communicator) the collectives run on.
  virtual fmoe_ctx* device_context() const = 0;
  // Per-transport collective counter (transport.hpp:34 of the reference).
  std::uint32_t next_tag() { return next_tag_++; }

 private:
  std::uint32_t next_tag_ = 1;
};

// world_size ranks as threads of this process, all on one GPU
// (FMOE_DEVICE, default 0).  transport(r) is called once per rank, typically
// from that rank's thread.
class InProcWorld {
 public:
  explicit InProcWorld(int world_size);
  ~InProcWorld();
  int world_size() const;
  std::unique_ptr<Transport> transport(int rank);

  struct Shared;

 private:
  std::shared_ptr<Shared> shared_;
};

// NCCL world, one process per GPU: rank 0 calls nccl_unique_id() and ships the
// bytes to the other ranks out of band; every rank then calls nccl_connect.
std::vector<std::uint8_t> nccl_unique_id();
std::unique_ptr<Transport> nccl_connect(int rank, int world_size, const std::vector<std::uint8_t>& id,
                                        int device = -1);

struct HostPort {
  std::string host;
  std::uint16_t port = 0;
};
std::vector<HostPort> localhost_endpoints(int world_size, std::uint16_t base_port);
// TCP rendezvous configuration: not provided by the B200 drop-in (throws TransportError).
std::vector<HostPort> parse_hostfile(const std::string& path);
// Not provided by the B200 drop-in: throws TransportError (use nccl_connect).
std::unique_ptr<Transport> tcp_connect(int rank, const std::vector<HostPort>& endpoints,
                                       std::chrono::milliseconds timeout = std::chrono::seconds(30));

}  // namespace fmoe
