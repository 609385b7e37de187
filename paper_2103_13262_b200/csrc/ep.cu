// ep.cu -- expert parallelism over NCCL (collectives.cpp:69-265).
// Not wired yet: the single-GPU layer is the round-1 target; EP entry points
// report a ProtocolError until fmoe_comm_init has been implemented.
#include "layer.cuh"

namespace fmoe_b200 {

struct Layer::Ep {};

void Layer::ep_alloc() {}
void Layer::ep_forward(const void*, void*) {
  protocol_error("forward: expert parallelism needs fmoe_comm_init (not available in this build)");
}
void Layer::ep_backward(const void*, void*) {
  protocol_error("backward: expert parallelism needs fmoe_comm_init (not available in this build)");
}

}  // namespace fmoe_b200

extern "C" {
int fmoe_comm_unique_id(void*, int64_t) {
  fmoe_b200::g_last_error = "NCCL communicator not available in this build";
  return FMOE_ERR_TRANSPORT;
}
int fmoe_comm_init(fmoe_ctx*, const void*, int64_t, int, int) {
  fmoe_b200::g_last_error = "NCCL communicator not available in this build";
  return FMOE_ERR_TRANSPORT;
}
}
