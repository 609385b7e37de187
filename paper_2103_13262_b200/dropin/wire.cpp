// wire.cpp -- the reference's framed-byte API (wire.hpp, Transport::send_frame /
// recv_frame, parse_hostfile) as explicit "not provided" stubs.  The B200
// drop-in's transports move device rows over NCCL or in-process device copies;
// the wire codec and the TCP transport are out of scope.  The
// stubs exist so code written against the reference headers links, and fails
// loudly (TransportError) if it ever relies on frames.
#include <string>

#include "fmoe/errors.hpp"
#include "fmoe/transport.hpp"
#include "fmoe/wire.hpp"

namespace fmoe {

namespace {
[[noreturn]] void no_wire(const char* what) {
  throw TransportError(std::string(what) +
                       ": the B200 drop-in has no wire codec (rows move over NCCL / device copies)");
}
}  // namespace

std::vector<std::byte> encode_frame(const Frame&) { no_wire("encode_frame"); }
void encode_header(const FrameHeader&, std::span<std::byte, kFrameHeaderSize>) { no_wire("encode_header"); }
FrameHeader decode_header(std::span<const std::byte, kFrameHeaderSize>) { no_wire("decode_header"); }
Frame decode_frame(std::span<const std::byte>) { no_wire("decode_frame"); }
std::vector<std::byte> pack_counts(std::span<const std::int64_t>) { no_wire("pack_counts"); }
std::vector<std::int64_t> unpack_counts(std::span<const std::byte>) { no_wire("unpack_counts"); }
std::vector<std::byte> pack_rows(const Matrix&, std::size_t, std::size_t) { no_wire("pack_rows"); }
void unpack_rows(std::span<const std::byte>, Matrix&, std::size_t, std::size_t) { no_wire("unpack_rows"); }

void Transport::send_frame(int, MsgType, std::uint32_t, std::span<const std::byte>) {
  no_wire("Transport::send_frame");
}
std::vector<std::byte> Transport::recv_frame(int, MsgType, std::uint32_t) { no_wire("Transport::recv_frame"); }

std::vector<HostPort> parse_hostfile(const std::string&) { no_wire("parse_hostfile (TCP rendezvous)"); }

}  // namespace fmoe
