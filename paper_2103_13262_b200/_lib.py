"""ctypes binding of libfmoe_b200.so (the C-ABI in include/fmoe_b200.h).

The product path always runs through this library; there is no fallback.  If
the shared object is missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FMOE_B200_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("FMOE_B200_LIB") or os.path.join(HERE, "libfmoe_b200.so")

F64, F32, BF16 = 0, 1, 2
OK, ERR_SHAPE, ERR_PROTOCOL, ERR_TRANSPORT, ERR_CUDA = 0, 1, 2, 3, 4


class FmoeError(RuntimeError):
    code = ERR_CUDA


class ShapeError(FmoeError, ValueError):
    """fmoe::ShapeError (errors.hpp:8-11)"""

    code = ERR_SHAPE


class ProtocolError(FmoeError):
    """fmoe::ProtocolError (errors.hpp:13-17)"""

    code = ERR_PROTOCOL


class TransportError(FmoeError):
    """fmoe::TransportError (errors.hpp:19-23)"""

    code = ERR_TRANSPORT


class CudaError(FmoeError):
    code = ERR_CUDA


_ERRORS = {ERR_SHAPE: ShapeError, ERR_PROTOCOL: ProtocolError, ERR_TRANSPORT: TransportError,
           ERR_CUDA: CudaError}

i64 = C.c_int64
vp = C.c_void_p
i32p = C.POINTER(C.c_int32)


class Plan(C.Structure):
    _fields_ = [("n_b", i64), ("k", i64), ("n_experts", i64), ("align", i64), ("capacity", i64),
                ("counts", vp), ("offsets", vp), ("src_row", vp), ("slot", vp),
                ("inverse_pos", vp), ("tile_expert", vp), ("n_tiles", vp), ("scratch", vp)]


class ExpertParams(C.Structure):
    _fields_ = [("w1", vp), ("b1", vp), ("w2", vp), ("b2", vp)]


class ExpertGrads(C.Structure):
    _fields_ = [("d_w1", vp), ("d_b1", vp), ("d_w2", vp), ("d_b2", vp)]


class LayerConfig(C.Structure):
    _fields_ = [("n_b", i64), ("d_m", i64), ("d_h", i64), ("k", i64), ("n_e_local", i64),
                ("world_size", i64), ("rank", i64), ("seed", C.c_uint64), ("dtype", C.c_int)]


EXPORTS = [
    "fmoe_last_error", "fmoe_version", "fmoe_ctx_create", "fmoe_ctx_destroy", "fmoe_ctx_set_stream",
    "fmoe_ctx_launches", "fmoe_ctx_check", "fmoe_ctx_profile", "fmoe_ctx_profile_read", "fmoe_ctx_profile_step_ms",
    "fmoe_ctx_clock_probe",
    "fmoe_ctx_clock_probe_read", "fmoe_gate_fwd", "fmoe_gate_bwd", "fmoe_plan_sizes",
    "fmoe_plan_build", "fmoe_scatter", "fmoe_gather_combine", "fmoe_scatter_bwd",
    "fmoe_gather_combine_bwd", "fmoe_experts_fwd", "fmoe_experts_bwd", "fmoe_layer_create",
    "fmoe_layer_destroy", "fmoe_layer_init_weights", "fmoe_layer_params", "fmoe_layer_grads",
    "fmoe_layer_routing", "fmoe_layer_fwd", "fmoe_layer_bwd", "fmoe_moe_fwd", "fmoe_moe_bwd", "fmoe_layer_step_host",
    "fmoe_comm_unique_id", "fmoe_comm_init", "fmoe_comm_attach", "fmoe_world_create", "fmoe_world_destroy",
    "fmoe_ctx_join_world", "fmoe_exchange_counts", "fmoe_ep_layout", "fmoe_a2a_rows",
    "fmoe_a2a_rows_reverse", "fmoe_allreduce_sum", "fmoe_matmul", "fmoe_softmax_rows", "fmoe_topk_rows",
    "fmoe_experts_fwd_cached", "fmoe_experts_bwd_cached", "fmoe_layer_train_step", "fmoe_layer_sync_masters",
    "fmoe_layer_fwd_routed", "fmoe_layer_routing_grad", "fmoe_layer_set_ep_exchange",
    "fmoe_layer_ep_exchange_fused", "fmoe_ep_routes", "fmoe_layer_peer_blob", "fmoe_layer_peer_connect",
    "fmoe_checkpoint_info", "fmoe_layer_load_checkpoint", "fmoe_layer_save_checkpoint",
    "fmoe_layer_step_host_async", "fmoe_layer_step_host_wait", "fmoe_cast", "fmoe_layer_keep_preact",
    "fmoe_layer_activations",
]


class CkptInfo(C.Structure):
    _fields_ = [("n_b", i64), ("d_m", i64), ("d_h", i64), ("k", i64), ("n_e_local", i64), ("world_size", i64),
                ("experts_total", i64), ("seed", C.c_uint64)]


class ExchangePlanC(C.Structure):
    _fields_ = [("world", i64), ("rank", i64), ("local_experts", i64), ("send_counts", vp),
                ("recv_counts", vp), ("send_total", i64), ("recv_total", i64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2103_13262_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    lib.fmoe_last_error.restype = C.c_char_p
    lib.fmoe_version.restype = C.c_char_p
    lib.fmoe_ctx_launches.restype = i64
    lib.fmoe_ctx_launches.argtypes = [vp]
    sig = {
        "fmoe_ctx_create": [C.c_int, vp, C.POINTER(vp)],
        "fmoe_ctx_destroy": [vp],
        "fmoe_ctx_set_stream": [vp, vp],
        "fmoe_ctx_check": [vp],
        "fmoe_ctx_profile": [vp, C.c_int],
        "fmoe_ctx_profile_read": [vp, C.POINTER(C.c_float), C.c_int, C.POINTER(C.c_int)],
        "fmoe_ctx_profile_step_ms": [vp, C.POINTER(C.c_float), C.c_int],
        "fmoe_ctx_clock_probe": [vp, C.c_int],
        "fmoe_ctx_clock_probe_read": [vp, C.POINTER(C.c_double), C.POINTER(C.c_int)],
        "fmoe_gate_fwd": [vp, C.c_int, vp, vp, i64, i64, i64, i64, vp, vp, vp],
        "fmoe_gate_bwd": [vp, C.c_int, vp, vp, vp, vp, vp, i64, i64, i64, i64, vp, vp],
        "fmoe_plan_sizes": [i64, i64, i64, i64, C.POINTER(i64), C.POINTER(i64)],
        "fmoe_plan_build": [vp, vp, C.POINTER(Plan), C.c_int],
        "fmoe_scatter": [vp, C.c_int, vp, i64, C.POINTER(Plan), vp],
        "fmoe_gather_combine": [vp, C.c_int, vp, i64, C.POINTER(Plan), vp, vp],
        "fmoe_scatter_bwd": [vp, C.c_int, vp, i64, C.POINTER(Plan), vp],
        "fmoe_gather_combine_bwd": [vp, C.c_int, vp, vp, i64, C.POINTER(Plan), vp, vp, vp],
        "fmoe_experts_fwd": [vp, C.c_int, C.POINTER(Plan), i64, i64, ExpertParams, vp, vp, vp],
        "fmoe_experts_bwd": [vp, C.c_int, C.POINTER(Plan), i64, i64, ExpertParams, vp, vp, vp, vp,
                             ExpertGrads],
        "fmoe_layer_create": [vp, C.POINTER(LayerConfig), C.POINTER(vp)],
        "fmoe_layer_destroy": [vp],
        "fmoe_layer_init_weights": [vp],
        "fmoe_layer_params": [vp, C.POINTER(vp), C.POINTER(ExpertParams)],
        "fmoe_layer_grads": [vp, C.POINTER(vp), C.POINTER(ExpertGrads)],
        "fmoe_layer_routing": [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(Plan)],
        "fmoe_layer_fwd": [vp, vp, vp],
        "fmoe_moe_fwd": [vp, vp, vp],
        "fmoe_moe_bwd": [vp, vp, vp],
        "fmoe_layer_bwd": [vp, vp, vp],
        "fmoe_layer_fwd_routed": [vp, vp, vp, vp, vp],
        "fmoe_layer_routing_grad": [vp, C.POINTER(vp)],
        "fmoe_layer_set_ep_exchange": [vp, C.c_int],
        "fmoe_layer_peer_blob": [vp, vp, i64, C.POINTER(i64)],
        "fmoe_layer_peer_connect": [vp, vp, i64],
        "fmoe_checkpoint_info": [C.c_char_p, C.POINTER(CkptInfo)],
        "fmoe_layer_load_checkpoint": [vp, C.c_char_p],
        "fmoe_layer_save_checkpoint": [vp, C.c_char_p],
        "fmoe_ep_routes": [C.c_int, C.c_int, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp],
        "fmoe_layer_ep_exchange_fused": [vp, C.POINTER(C.c_int)],
        "fmoe_cast": [vp, C.c_int, vp, C.c_int, vp, i64],
        "fmoe_layer_keep_preact": [vp, C.c_int],
        "fmoe_layer_activations": [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)],
        "fmoe_world_create": [C.c_int, C.POINTER(vp)],
        "fmoe_world_destroy": [vp],
        "fmoe_ctx_join_world": [vp, vp, C.c_int],
        "fmoe_exchange_counts": [vp, vp, i64, C.POINTER(ExchangePlanC)],
        "fmoe_ep_layout": [C.c_int, i64, i64, vp, vp, vp, vp, vp, vp],
        "fmoe_a2a_rows": [vp, C.c_int, vp, i64, C.POINTER(ExchangePlanC), vp],
        "fmoe_a2a_rows_reverse": [vp, C.c_int, vp, i64, C.POINTER(ExchangePlanC), vp],
        "fmoe_layer_step_host": [vp, vp, vp, vp, vp],
        "fmoe_layer_step_host_async": [vp, vp, vp, vp, vp],
        "fmoe_layer_step_host_wait": [vp],
        "fmoe_comm_unique_id": [vp, i64],
        "fmoe_comm_init": [vp, vp, i64, C.c_int, C.c_int],
        "fmoe_comm_attach": [vp, vp],
        "fmoe_allreduce_sum": [vp, C.c_int, vp, i64, vp, i64],
        "fmoe_layer_train_step": [vp, vp, vp, C.c_double, C.POINTER(C.c_double)],
        "fmoe_layer_sync_masters": [vp],
        "fmoe_matmul": [vp, C.c_int, vp, vp, i64, i64, i64, vp],
        "fmoe_softmax_rows": [vp, C.c_int, vp, i64, i64, vp],
        "fmoe_topk_rows": [vp, C.c_int, vp, i64, i64, i64, vp, vp],
        "fmoe_experts_fwd_cached": [vp, C.c_int, C.POINTER(Plan), i64, i64, ExpertParams, vp, vp, vp, vp],
        "fmoe_experts_bwd_cached": [vp, C.c_int, C.POINTER(Plan), i64, i64, ExpertParams, vp, vp, vp, vp, vp,
                                    ExpertGrads],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc != OK:
        msg = lib.fmoe_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, FmoeError)(msg)
