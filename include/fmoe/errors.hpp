// fmoe/errors.hpp -- exception types of the FastMoE C++ API (reference:
// proj/include/fmoe/errors.hpp:8-23).  The drop-in library (libfmoe_dropin.so)
// maps the C-ABI status codes of include/fmoe_b200.h onto them:
//   FMOE_ERR_SHAPE -> ShapeError, FMOE_ERR_PROTOCOL -> ProtocolError,
//   FMOE_ERR_TRANSPORT -> TransportError, FMOE_ERR_CUDA -> std::runtime_error.
#pragma once

#include <stdexcept>

namespace fmoe {

// Bad shapes, k, expert indices or configuration.
struct ShapeError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

// Plans, payload sizes or worlds that disagree between ranks.
struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// The communicator failed (NCCL error, peer timeout).
struct TransportError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

}  // namespace fmoe
