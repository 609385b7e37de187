"""Python host of the B200 MoE-layer hot path, mirroring the reference's C++
operator / layer API (include/fmoe/{gate,dispatch,expert,moe_layer}.hpp) on
device tensors.  Every call goes through the C-ABI (libfmoe_b200.so);
PyTorch only provides device memory and the current CUDA stream.

dtype follows the input tensors: torch.float64 selects the parity mode
(reference accumulation order), torch.float32 the SIMT fp32 path and
torch.bfloat16 the tcgen05 tensor-core product path (fp32 scores/gradients).
Indices are int32 on device (the reference's int64 are widened by callers).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import torch

from . import _lib
from ._lib import BF16, F32, F64, ExpertGrads, ExpertParams, LayerConfig, Plan, check, lib
from ._lib import ProtocolError, ShapeError, TransportError  # noqa: F401

_DT = {torch.float64: F64, torch.float32: F32, torch.bfloat16: BF16}


def dtype_code(t: torch.dtype) -> int:
    if t not in _DT:
        raise ShapeError(f"unsupported dtype {t}")
    return _DT[t]


def score_dtype(t: torch.dtype) -> torch.dtype:
    return torch.float64 if t == torch.float64 else torch.float32


def grad_dtype(t: torch.dtype) -> torch.dtype:
    return torch.float32 if t == torch.bfloat16 else t


def _p(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev(t: torch.Tensor) -> torch.Tensor:
    if not t.is_cuda:
        raise ShapeError("tensors must live on a CUDA device (no CPU fallback)")
    return t.contiguous()


# ------------------------------------------------------------------ context
class Context:
    """fmoe_ctx bound to a device; follows torch's current stream per call."""

    _by_device: dict = {}

    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        check(lib.fmoe_ctx_create(device, None, C.byref(h)))
        self.h = h

    @classmethod
    def get(cls, device=None) -> "Context":
        if device is None:
            device = torch.cuda.current_device()
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        c = cls._by_device.get(device)
        if c is None:
            c = cls._by_device[device] = cls(device)
        check(lib.fmoe_ctx_set_stream(c.h, C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))
        return c

    @property
    def launches(self) -> int:
        return int(lib.fmoe_ctx_launches(self.h))

    def check(self):
        check(lib.fmoe_ctx_check(self.h))

    def use_current_stream(self):
        check(lib.fmoe_ctx_set_stream(self.h, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))
        return self

    def join_world(self, world: "World", rank: int):
        """In-process expert-parallel world (InProcWorld analogue, one host thread per rank)."""
        check(lib.fmoe_ctx_join_world(self.h, world.h, rank))

    def init_nccl(self, dist, world: int, rank: int):
        """NCCL communicator over NVLink; the 128-byte id travels through torch.distributed."""
        buf = (C.c_char * 128)()
        if rank == 0:
            check(lib.fmoe_comm_unique_id(buf, 128))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0)
        idb = (C.c_char * 128).from_buffer_copy(obj[0])
        check(lib.fmoe_comm_init(self.h, idb, 128, world, rank))

    def attach_nccl(self, comm: int):
        """Borrow an existing ncclComm_t (an integer handle, one rank per GPU);
        world and rank come from the communicator, which the caller keeps."""
        check(lib.fmoe_comm_attach(self.h, C.c_void_p(comm)))


class World:
    """fmoe_world: `world` ranks of one process (tests, single-GPU EP runs)."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(lib.fmoe_world_create(world, C.byref(h)))
        self.h, self.world = h, world

    def __del__(self):
        if getattr(self, "h", None) is not None and lib is not None:
            lib.fmoe_world_destroy(self.h)
            self.h = None


# ----------------------------------------------------- EP collectives (L2)
@dataclass
class ExchangePlan:
    """ExchangePlan (collectives.hpp:16-33)."""

    rank: int
    world: int
    local_experts: int
    send_counts: "np.ndarray"  # [world, local_experts]
    recv_counts: "np.ndarray"  # [world, local_experts]
    send_total: int
    recv_total: int

    def local_expert_rows(self):
        return self.recv_counts.sum(axis=0)

    def c(self):
        import numpy as np

        self._s = np.ascontiguousarray(self.send_counts.reshape(-1), dtype=np.int64)
        self._r = np.ascontiguousarray(self.recv_counts.reshape(-1), dtype=np.int64)
        return _lib.ExchangePlanC(self.world, self.rank, self.local_experts, self._s.ctypes.data,
                                  self._r.ctypes.data, self.send_total, self.recv_total)


def exchange_counts(local_counts, ctx: Context) -> ExchangePlan:
    """exchange_counts (collectives.hpp:39-40) over ctx's transport."""
    import numpy as np

    lc = np.ascontiguousarray(np.asarray(local_counts, dtype=np.int64).reshape(-1))
    s = np.zeros_like(lc)
    r = np.zeros_like(lc)
    p = _lib.ExchangePlanC(0, 0, 0, s.ctypes.data, r.ctypes.data, 0, 0)
    check(lib.fmoe_exchange_counts(ctx.h, lc.ctypes.data, lc.size, C.byref(p)))
    w, el = p.world, p.local_experts
    return ExchangePlan(p.rank, w, el, s.reshape(w, el), r.reshape(w, el), p.send_total, p.recv_total)


def all_to_all_rows(xs: torch.Tensor, plan: ExchangePlan, ctx: Context) -> torch.Tensor:
    """all_to_all_rows (collectives.hpp:41-47)."""
    xs = _dev(xs)
    if xs.shape[0] != plan.send_total:
        raise ProtocolError(f"all_to_all_rows: input rows {xs.shape[0]} != planned send total {plan.send_total}")
    out = torch.empty(plan.recv_total, xs.shape[1], dtype=xs.dtype, device=xs.device)
    pc = plan.c()
    check(lib.fmoe_a2a_rows(ctx.h, dtype_code(xs.dtype), _p(xs), xs.shape[1], C.byref(pc), _p(out)))
    return out


def all_to_all_rows_reverse(ys: torch.Tensor, plan: ExchangePlan, ctx: Context) -> torch.Tensor:
    """all_to_all_rows_reverse (collectives.hpp:48-50)."""
    ys = _dev(ys)
    if ys.shape[0] != plan.recv_total:
        raise ProtocolError(f"all_to_all_rows_reverse: input rows {ys.shape[0]} != planned recv total")
    out = torch.empty(plan.send_total, ys.shape[1], dtype=ys.dtype, device=ys.device)
    pc = plan.c()
    check(lib.fmoe_a2a_rows_reverse(ctx.h, dtype_code(ys.dtype), _p(ys), ys.shape[1], C.byref(pc), _p(out)))
    return out


def allreduce_sum(m: torch.Tensor, group, ctx: Context) -> torch.Tensor:
    """allreduce_sum (collectives.hpp:52-53): sum over the sorted rank list
    `group` in ascending rank order (identical bytes on every member).  Every
    rank of ctx's world must enter the call.  fp64 / fp32."""
    import numpy as np

    m = _dev(m).contiguous()
    out = m.clone()
    g = np.ascontiguousarray(np.asarray(list(group), dtype=np.int32))
    check(lib.fmoe_allreduce_sum(ctx.h, dtype_code(m.dtype), _p(out), out.numel(), g.ctypes.data, g.size))
    return out


def ep_layout(world: int, local_experts: int, align: int, send_counts, recv_counts):
    """Host layout of one exchange through the library (fmoe_ep_layout):
    (send_off [E], chunk_off [el, W], block_off [el+1], rows [el])."""
    import numpy as np

    e = world * local_experts
    s = np.ascontiguousarray(np.asarray(send_counts, np.int64).reshape(-1))
    r = np.ascontiguousarray(np.asarray(recv_counts, np.int64).reshape(-1))
    so = np.zeros(e, np.int64)
    co = np.zeros(e, np.int64)
    bo = np.zeros(local_experts + 1, np.int64)
    rows = np.zeros(local_experts, np.int64)
    check(lib.fmoe_ep_layout(world, local_experts, align, s.ctypes.data, r.ctypes.data, so.ctypes.data,
                             co.ctypes.data, bo.ctypes.data, rows.ctypes.data))
    return so, co.reshape(local_experts, world), bo, rows


def ep_routes(world: int, rank: int, local_experts: int, align: int, counts):
    """Host arithmetic of the fused peer-memory exchange (fmoe_ep_routes) from
    the all-gathered counts [world, world*local_experts]: (send_off, chunk_off
    [el, W], block_off, rows, g_rank [E], g_delta [E], route [3, el, W])."""
    import numpy as np

    e = world * local_experts
    c = np.ascontiguousarray(np.asarray(counts, np.int64).reshape(world, e))
    so = np.zeros(e, np.int64)
    co = np.zeros(e, np.int64)
    bo = np.zeros(local_experts + 1, np.int64)
    rows = np.zeros(local_experts, np.int64)
    gr = np.zeros(e, np.int32)
    gd = np.zeros(e, np.int64)
    rt = np.zeros(3 * e, np.int32)
    check(lib.fmoe_ep_routes(world, rank, local_experts, align, c.ctypes.data, so.ctypes.data, co.ctypes.data,
                             bo.ctypes.data, rows.ctypes.data, gr.ctypes.data, gd.ctypes.data, rt.ctypes.data))
    return so, co.reshape(local_experts, world), bo, rows, gr, gd, rt.reshape(3, local_experts, world)


def checkpoint_info(path: str) -> dict:
    """Header of a reference checkpoint file (fmoe_checkpoint_info)."""
    info = _lib.CkptInfo()
    check(lib.fmoe_checkpoint_info(str(path).encode(), C.byref(info)))
    return {k: int(getattr(info, k)) for k, _ in info._fields_}


def _ctx(t: torch.Tensor) -> Context:
    return Context.get(t.device)


# ---------------------------------------------------------- dense primitives
def _simt(t: torch.Tensor, who: str) -> None:
    if t.dtype not in (torch.float64, torch.float32):
        raise ShapeError(f"{who}: fp64 or fp32 only")


def matmul(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """matmul (matrix.hpp:77; matrix.cpp:96-119): one fma chain per element over
    the inner index ascending from +0.0 -- the kernel the fp64/fp32 gate uses."""
    a, b = _dev(a).contiguous(), _dev(b).contiguous()
    _simt(a, "matmul")
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0] or a.dtype != b.dtype:
        raise ShapeError(f"matmul: shapes {tuple(a.shape)} x {tuple(b.shape)}")
    c = torch.empty(a.shape[0], b.shape[1], dtype=a.dtype, device=a.device)
    check(lib.fmoe_matmul(_ctx(a).h, dtype_code(a.dtype), _p(a), _p(b), a.shape[0], a.shape[1], b.shape[1], _p(c)))
    return c


def softmax_rows(a: torch.Tensor) -> torch.Tensor:
    """softmax_rows (matrix.cpp:155-170), the gate's softmax."""
    a = _dev(a).contiguous()
    _simt(a, "softmax_rows")
    out = torch.empty_like(a)
    check(lib.fmoe_softmax_rows(_ctx(a).h, dtype_code(a.dtype), _p(a), a.shape[0], a.shape[1], _p(out)))
    return out


def topk_rows(a: torch.Tensor, k: int):
    """topk_rows (matrix.cpp:172-189): (indices int32, values), largest first,
    ties -> lower column."""
    a = _dev(a).contiguous()
    _simt(a, "topk_rows")
    idx = torch.empty(a.shape[0], max(k, 0), dtype=torch.int32, device=a.device)
    val = torch.empty(a.shape[0], max(k, 0), dtype=a.dtype, device=a.device)
    check(lib.fmoe_topk_rows(_ctx(a).h, dtype_code(a.dtype), _p(a), a.shape[0], a.shape[1], k, _p(idx), _p(val)))
    return idx, val


# --------------------------------------------------------------------- gate
@dataclass
class GateOutput:
    """gate.hpp:17-21"""

    scores: torch.Tensor         # [n_b, E] post-softmax (fp64 for fp64, else fp32)
    topk_indices: torch.Tensor   # [n_b, k] int32
    topk_scores: torch.Tensor    # [n_b, k]


def gate_forward(x: torch.Tensor, w_g: torch.Tensor, k: int) -> GateOutput:
    """gate_forward (gate.hpp:23-27, gate.cpp:23-35)."""
    x, w_g = _dev(x), _dev(w_g)
    if x.dim() != 2 or w_g.dim() != 2 or x.shape[1] != w_g.shape[0]:
        raise ShapeError(f"gate_forward: x cols {x.shape[-1]} != gate rows {w_g.shape[0]}")
    if w_g.dtype != x.dtype:
        raise ShapeError("gate_forward: dtype mismatch")
    n, d = x.shape
    e = w_g.shape[1]
    sd = score_dtype(x.dtype)
    scores = torch.empty(n, e, dtype=sd, device=x.device)
    idx = torch.empty(n, max(k, 0), dtype=torch.int32, device=x.device)
    vals = torch.empty(n, max(k, 0), dtype=sd, device=x.device)
    check(lib.fmoe_gate_fwd(_ctx(x).h, dtype_code(x.dtype), _p(x), _p(w_g), n, d, e, k, _p(scores),
                            _p(idx), _p(vals)))
    return GateOutput(scores, idx, vals)


@dataclass
class GateGrads:
    d_wg: torch.Tensor
    d_x: torch.Tensor


def gate_backward(x, w_g, out: GateOutput, d_topk_scores) -> GateGrads:
    """gate_backward (gate.hpp:34-38, gate.cpp:37-65)."""
    x, w_g = _dev(x), _dev(w_g)
    n, d = x.shape
    e = w_g.shape[1]
    k = out.topk_indices.shape[1]
    if out.scores.shape != (n, e):
        raise ShapeError("gate_backward: scores shape mismatch")
    if tuple(d_topk_scores.shape) != (n, k):
        raise ShapeError("gate_backward: upstream gradient shape mismatch")
    sd = score_dtype(x.dtype)
    d_wg = torch.empty(d, e, dtype=sd, device=x.device)
    d_x = torch.empty(n, d, dtype=x.dtype, device=x.device)
    check(lib.fmoe_gate_bwd(_ctx(x).h, dtype_code(x.dtype), _p(x), _p(w_g), _p(_dev(out.scores)),
                            _p(_dev(out.topk_indices)), _p(_dev(d_topk_scores.to(sd))), n, d, e, k,
                            _p(d_wg), _p(d_x)))
    return GateGrads(d_wg, d_x)


# ----------------------------------------------------------------- dispatch
@dataclass
class DispatchPlan:
    """DispatchPlan (dispatch.hpp:15-24) on device.  With align=1 the layout is
    exactly the reference's; align=128 pads each expert block to a tensor-core
    tile (padding rows have src_row == -1)."""

    n_b: int
    k: int
    num_experts: int
    align: int
    capacity: int
    counts: torch.Tensor
    offsets: torch.Tensor        # [E+1]
    expanded_src_row: torch.Tensor
    expanded_slot: torch.Tensor
    inverse_pos: torch.Tensor    # [n_b, k]
    tile_expert: torch.Tensor
    n_tiles: torch.Tensor
    scratch: torch.Tensor
    _c: Plan = field(default=None, repr=False)

    @property
    def c(self) -> Plan:
        if self._c is None:
            self._c = Plan(self.n_b, self.k, self.num_experts, self.align, self.capacity,
                           self.counts.data_ptr(), self.offsets.data_ptr(),
                           self.expanded_src_row.data_ptr(), self.expanded_slot.data_ptr(),
                           self.inverse_pos.data_ptr(), self.tile_expert.data_ptr(),
                           self.n_tiles.data_ptr(), self.scratch.data_ptr())
        return self._c


def alloc_plan(n_b: int, k: int, num_experts: int, align: int = 1, device=None) -> DispatchPlan:
    cap, scr = C.c_int64(), C.c_int64()
    check(lib.fmoe_plan_sizes(n_b, k, num_experts, align, C.byref(cap), C.byref(scr)))
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    z = lambda m: torch.empty(max(m, 1), dtype=torch.int32, device=dev)  # noqa: E731
    return DispatchPlan(n_b, k, num_experts, align, cap.value, z(num_experts)[:num_experts],
                        z(num_experts + 1), z(cap.value)[:cap.value], z(cap.value)[:cap.value],
                        z(n_b * k)[:n_b * k].view(n_b, k), z(cap.value // 128 + 1), z(1),
                        torch.empty(scr.value, dtype=torch.uint8, device=dev))


def build_plan(topk_indices: torch.Tensor, num_experts: int, align: int = 1,
               validate: bool = True, plan: Optional[DispatchPlan] = None) -> DispatchPlan:
    """build_plan (dispatch.hpp:28, dispatch.cpp:10-47).  Out-of-range indices
    raise ShapeError (validate=True costs one host sync)."""
    idx = _dev(topk_indices).to(torch.int32)
    n_b, k = idx.shape
    if plan is None:
        plan = alloc_plan(n_b, k, num_experts, align, idx.device)
    check(lib.fmoe_plan_build(_ctx(idx).h, _p(idx), C.byref(plan.c), 1 if validate else 0))
    return plan


def scatter(x: torch.Tensor, plan: DispatchPlan) -> torch.Tensor:
    """scatter (dispatch.cpp:49-59)."""
    x = _dev(x)
    if x.shape[0] != plan.n_b:
        raise ShapeError("scatter: input rows != plan batch size")
    out = torch.empty(plan.capacity, x.shape[1], dtype=x.dtype, device=x.device)
    check(lib.fmoe_scatter(_ctx(x).h, dtype_code(x.dtype), _p(x), x.shape[1], C.byref(plan.c), _p(out)))
    return out


def gather_combine(ys: torch.Tensor, plan: DispatchPlan, topk_scores: torch.Tensor) -> torch.Tensor:
    """gather_combine (dispatch.cpp:61-78)."""
    ys = _dev(ys)
    if ys.shape[0] != plan.capacity:
        raise ShapeError("gather_combine: ys rows != n_b * k")
    if tuple(topk_scores.shape) != (plan.n_b, plan.k):
        raise ShapeError("gather_combine: topk_scores shape mismatch")
    w = _dev(topk_scores.to(score_dtype(ys.dtype)))
    out = torch.empty(plan.n_b, ys.shape[1], dtype=ys.dtype, device=ys.device)
    check(lib.fmoe_gather_combine(_ctx(ys).h, dtype_code(ys.dtype), _p(ys), ys.shape[1], C.byref(plan.c),
                                  _p(w), _p(out)))
    return out


def scatter_backward(d_xs: torch.Tensor, plan: DispatchPlan) -> torch.Tensor:
    """scatter_backward (dispatch.cpp:80-95)."""
    d_xs = _dev(d_xs)
    if d_xs.shape[0] != plan.capacity:
        raise ShapeError("scatter_backward: rows != n_b * k")
    out = torch.empty(plan.n_b, d_xs.shape[1], dtype=d_xs.dtype, device=d_xs.device)
    check(lib.fmoe_scatter_bwd(_ctx(d_xs).h, dtype_code(d_xs.dtype), _p(d_xs), d_xs.shape[1],
                               C.byref(plan.c), _p(out)))
    return out


def gather_combine_backward(d_y, ys, plan: DispatchPlan, topk_scores):
    """gather_combine_backward (dispatch.cpp:97-126) -> (d_ys, d_topk_scores)."""
    d_y, ys = _dev(d_y), _dev(ys)
    if d_y.shape[0] != plan.n_b:
        raise ShapeError("gather_combine_backward: d_y rows != n_b")
    if ys.shape[0] != plan.capacity:
        raise ShapeError("gather_combine_backward: ys rows != n_b * k")
    if d_y.shape[1] != ys.shape[1]:
        raise ShapeError("gather_combine_backward: column mismatch")
    sd = score_dtype(ys.dtype)
    w = _dev(topk_scores.to(sd))
    d_ys = torch.empty_like(ys)
    d_w = torch.empty(plan.n_b, plan.k, dtype=sd, device=ys.device)
    check(lib.fmoe_gather_combine_bwd(_ctx(ys).h, dtype_code(ys.dtype), _p(d_y), _p(ys), ys.shape[1],
                                      C.byref(plan.c), _p(w), _p(d_ys), _p(d_w)))
    return d_ys, d_w


# ------------------------------------------------------------------ experts
@dataclass
class Experts:
    """Stacked ExpertParams (expert.hpp:15-21): w1 [E,d,h], b1 [E,h], w2 [E,h,d], b2 [E,d]."""

    w1: torch.Tensor
    b1: torch.Tensor
    w2: torch.Tensor
    b2: torch.Tensor

    def c(self) -> ExpertParams:
        return ExpertParams(self.w1.data_ptr(), self.b1.data_ptr(), self.w2.data_ptr(), self.b2.data_ptr())


@dataclass
class ExpertGradsT:
    d_w1: torch.Tensor
    d_b1: torch.Tensor
    d_w2: torch.Tensor
    d_b2: torch.Tensor


def multi_expert_forward(xs: torch.Tensor, plan: DispatchPlan, experts: Experts):
    """multi_expert_forward (expert.hpp:47-53) -> (ys, hidden)."""
    xs = _dev(xs)
    e, d, h = experts.w1.shape
    if e != plan.num_experts:
        raise ShapeError("multi_expert_forward: counts and experts disagree")
    ys = torch.empty(plan.capacity, d, dtype=xs.dtype, device=xs.device)
    hidden = torch.empty(plan.capacity, h, dtype=xs.dtype, device=xs.device)
    check(lib.fmoe_experts_fwd(_ctx(xs).h, dtype_code(xs.dtype), C.byref(plan.c), d, h, experts.c(),
                               _p(xs), _p(hidden), _p(ys)))
    return ys, hidden


def multi_expert_backward(d_ys, xs, hidden, plan: DispatchPlan, experts: Experts):
    """multi_expert_backward (expert.hpp:60-64) -> (d_xs, ExpertGradsT)."""
    d_ys, xs, hidden = _dev(d_ys), _dev(xs), _dev(hidden)
    e, d, h = experts.w1.shape
    gd = grad_dtype(xs.dtype)
    g = ExpertGradsT(torch.empty(e, d, h, dtype=gd, device=xs.device),
                     torch.empty(e, h, dtype=gd, device=xs.device),
                     torch.empty(e, h, d, dtype=gd, device=xs.device),
                     torch.empty(e, d, dtype=gd, device=xs.device))
    d_xs = torch.empty_like(xs)
    check(lib.fmoe_experts_bwd(_ctx(xs).h, dtype_code(xs.dtype), C.byref(plan.c), d, h, experts.c(),
                               _p(xs), _p(hidden), _p(d_ys), _p(d_xs),
                               ExpertGrads(g.d_w1.data_ptr(), g.d_b1.data_ptr(), g.d_w2.data_ptr(),
                                           g.d_b2.data_ptr())))
    return d_xs, g


# -------------------------------------------------------------------- layer
@dataclass
class MoEConfig:
    """MoEConfig (moe_layer.hpp:17-27)."""

    n_b: int
    d_m: int
    d_h: int
    k: int
    n_e_local: int
    world_size: int = 1
    seed: int = 0

    def total_experts(self) -> int:
        return self.n_e_local * self.world_size


class MoELayer:
    """One rank's MoE layer on a B200 (MoELayerState + forward/backward,
    moe_layer.hpp:31-75).  Parameters and gradients live on device and are
    exposed as torch views; activations are cached inside the layer."""

    def __init__(self, config: MoEConfig, rank: int = 0, dtype: torch.dtype = torch.bfloat16,
                 device=None, init: bool = True, ctx: Optional[Context] = None):
        self.config = config
        self.rank = rank
        self.dtype = dtype
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        # each layer owns a context (its stream and, under EP, its transport)
        self.ctx = (ctx if ctx is not None else Context(dev.index)).use_current_stream()
        cfg = LayerConfig(config.n_b, config.d_m, config.d_h, config.k, config.n_e_local,
                          config.world_size, rank, config.seed, dtype_code(dtype))
        h = C.c_void_p()
        check(lib.fmoe_layer_create(self.ctx.h, C.byref(cfg), C.byref(h)))
        self.h = h
        if init:
            self.init_weights()
        self._views()

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and lib is not None:
            lib.fmoe_layer_destroy(h)
            self.h = None

    def init_weights(self):
        """init_state (moe_layer.cpp:28-45): the reference's generators."""
        check(lib.fmoe_layer_init_weights(self.h))

    def load_checkpoint(self, path: str):
        """Gate + this rank's experts from a reference checkpoint file
        (FMOE-CKPT v1, checkpoint.cpp:94-122), rounded once to the layer dtype."""
        check(lib.fmoe_layer_load_checkpoint(self.h, str(path).encode()))

    def save_checkpoint(self, path: str):
        """All weights in the reference's checkpoint format (world_size 1)."""
        check(lib.fmoe_layer_save_checkpoint(self.h, str(path).encode()))

    def connect(self, dist):
        """Expert parallelism over NCCL: one process per GPU, torch.distributed
        carries the communicator id (world/rank from the layer's config)."""
        self.ctx.init_nccl(dist, self.config.world_size, self.rank)

    def join(self, world: World):
        """Expert parallelism inside one process (one host thread per rank)."""
        self.ctx.join_world(world, self.rank)

    def connect_peers(self, dist):
        """bf16 expert parallelism over NVLink peer memory with the peer
        buffers exchanged through torch.distributed (any backend, gloo
        included): no device transport is needed afterwards."""
        n = C.c_int64()
        check(lib.fmoe_layer_peer_blob(self.h, None, 0, C.byref(n)))
        buf = (C.c_char * n.value)()
        check(lib.fmoe_layer_peer_blob(self.h, buf, n.value, C.byref(n)))
        blobs = [None] * self.config.world_size
        dist.all_gather_object(blobs, bytes(buf))
        allb = C.create_string_buffer(b"".join(blobs), n.value * len(blobs))
        check(lib.fmoe_layer_peer_connect(self.h, allb, n.value))

    def set_ep_exchange(self, mode: str):
        """'peer' (default): the expert-parallel row exchanges are fused into
        the scatter / expert-GEMM epilogues over NVLink peer memory;
        'transport': grouped send/recv through the transport.  Before the
        first forward, identically on every rank."""
        code = {"peer": 0, "transport": 1}.get(mode)
        if code is None:
            raise ShapeError(f"set_ep_exchange: unknown mode {mode!r}")
        check(lib.fmoe_layer_set_ep_exchange(self.h, code))

    @property
    def ep_exchange_fused(self) -> bool:
        """True when the last forward ran the fused peer-memory exchange."""
        v = C.c_int()
        check(lib.fmoe_layer_ep_exchange_fused(self.h, C.byref(v)))
        return bool(v.value)

    def _views(self):
        c = self.config
        e, el, d, hh = c.total_experts(), c.n_e_local, c.d_m, c.d_h
        wg = C.c_void_p()
        ep = ExpertParams()
        check(lib.fmoe_layer_params(self.h, C.byref(wg), C.byref(ep)))
        dwg = C.c_void_p()
        eg = ExpertGrads()
        check(lib.fmoe_layer_grads(self.h, C.byref(dwg), C.byref(eg)))
        t = self.dtype
        bt = torch.float32 if t == torch.bfloat16 else t
        gt = grad_dtype(t)
        st = score_dtype(t)
        v = lambda ptr, shape, dt: _wrap(ptr, shape, dt, self.device, self)  # noqa: E731
        self.w_g = v(wg.value, (d, e), t)
        self.experts = Experts(v(ep.w1, (el, d, hh), t), v(ep.b1, (el, hh), bt), v(ep.w2, (el, hh, d), t),
                               v(ep.b2, (el, d), bt))
        self.d_wg = v(dwg.value, (d, e), st)
        self.grads = ExpertGradsT(v(eg.d_w1, (el, d, hh), gt), v(eg.d_b1, (el, hh), gt),
                                  v(eg.d_w2, (el, hh, d), gt), v(eg.d_b2, (el, d), gt))

    def routing(self):
        """(topk_idx [n,k] int32, topk_scores [n,k], scores [n,E], plan)."""
        c = self.config
        i, w, s = C.c_void_p(), C.c_void_p(), C.c_void_p()
        p = Plan()
        check(lib.fmoe_layer_routing(self.h, C.byref(i), C.byref(w), C.byref(s), C.byref(p)))
        st = score_dtype(self.dtype)
        e = c.total_experts()
        idx = _wrap(i.value, (c.n_b, c.k), torch.int32, self.device, self)
        vals = _wrap(w.value, (c.n_b, c.k), st, self.device, self)
        scores = _wrap(s.value, (c.n_b, e), st, self.device, self)
        return idx, vals, scores, p

    def forward(self, x: torch.Tensor, y: Optional[torch.Tensor] = None) -> torch.Tensor:
        """forward (moe_layer.cpp:67-110).  x must stay alive until backward()."""
        x = _dev(x)
        if x.shape != (self.config.n_b, self.config.d_m) or x.dtype != self.dtype:
            raise ShapeError(f"forward: expected x [{self.config.n_b}, {self.config.d_m}] {self.dtype}")
        if y is None:
            y = torch.empty_like(x)
        self.ctx.use_current_stream()
        check(lib.fmoe_layer_fwd(self.h, _p(x), _p(y)))
        self._x = x
        return y

    def forward_routed(self, x: torch.Tensor, topk_idx: torch.Tensor, topk_scores: torch.Tensor,
                       y: Optional[torch.Tensor] = None) -> torch.Tensor:
        """forward with injected routing (the reference's build_plan fed a
        sampled IndexMatrix, dispatch.hpp:28): no gate.
        topk_idx [n_b, k] int32, topk_scores [n_b, k] in the score dtype.  The
        next backward() returns d_x = scatter_backward(d_xs) and leaves
        d(topk_scores) in routing_grad()."""
        x = _dev(x)
        c = self.config
        if x.shape != (c.n_b, c.d_m) or x.dtype != self.dtype:
            raise ShapeError(f"forward_routed: expected x [{c.n_b}, {c.d_m}] {self.dtype}")
        idx = _dev(topk_idx)
        sc = _dev(topk_scores)
        if idx.shape != (c.n_b, c.k) or idx.dtype != torch.int32:
            raise ShapeError(f"forward_routed: expected topk_idx [{c.n_b}, {c.k}] int32")
        if sc.shape != (c.n_b, c.k) or sc.dtype != score_dtype(self.dtype):
            raise ShapeError(f"forward_routed: expected topk_scores [{c.n_b}, {c.k}] {score_dtype(self.dtype)}")
        if y is None:
            y = torch.empty_like(x)
        self.ctx.use_current_stream()
        check(lib.fmoe_layer_fwd_routed(self.h, _p(x), _p(idx), _p(sc), _p(y)))
        self._x, self._routing_in = x, (idx, sc)
        return y

    def routing_grad(self) -> torch.Tensor:
        """d(topk_scores) [n_b, k] of the last backward (gather_combine_backward's d_w)."""
        c = self.config
        p = C.c_void_p()
        check(lib.fmoe_layer_routing_grad(self.h, C.byref(p)))
        return _wrap(p.value, (c.n_b, c.k), score_dtype(self.dtype), self.device, self)

    def backward(self, dy: torch.Tensor, dx: Optional[torch.Tensor] = None) -> torch.Tensor:
        """backward (moe_layer.cpp:112-142): returns d_x; parameter gradients
        land in self.d_wg / self.grads."""
        dy = _dev(dy)
        if dx is None:
            dx = torch.empty_like(dy)
        self.ctx.use_current_stream()
        check(lib.fmoe_layer_bwd(self.h, _p(dy), _p(dx)))
        return dx

    def train_step(self, x: torch.Tensor, target: torch.Tensor, lr: float) -> float:
        """train_step (moe_layer.cpp:144-205) on device: forward, MSE against
        target, backward, (EP) gradient sync, SGD.  Returns the world-average
        loss (one host sync)."""
        x, target = _dev(x), _dev(target)
        shape = (self.config.n_b, self.config.d_m)
        if x.shape != shape or target.shape != shape or x.dtype != self.dtype or target.dtype != self.dtype:
            raise ShapeError(f"train_step: expected x and target [{shape[0]}, {shape[1]}] {self.dtype}")
        self.ctx.use_current_stream()
        loss = C.c_double()
        check(lib.fmoe_layer_train_step(self.h, _p(x), _p(target), float(lr), C.byref(loss)))
        self._x = x
        return loss.value

    def sync_masters(self):
        """Re-widen the fp32 master weights of bf16 training from the bf16
        parameters (after writing self.w_g / self.experts by hand)."""
        check(lib.fmoe_layer_sync_masters(self.h))

    def step_host(self, x_host: torch.Tensor, dy_host: Optional[torch.Tensor], y_host: torch.Tensor,
                  dx_host: Optional[torch.Tensor] = None):
        """Host-buffer forward(+backward) through fmoe_layer_step_host."""
        self.ctx.use_current_stream()
        check(lib.fmoe_layer_step_host(self.h, _p(x_host), _p(dy_host), _p(y_host), _p(dx_host)))

    def step_host_async(self, x_host: torch.Tensor, dy_host: Optional[torch.Tensor], y_host: torch.Tensor,
                        dx_host: Optional[torch.Tensor] = None):
        """Enqueue a host-buffer forward(+backward) (fmoe_layer_step_host_async):
        the next step's uploads overlap this step's kernels.  Host buffers must
        stay untouched until wait_host()."""
        self.ctx.use_current_stream()
        check(lib.fmoe_layer_step_host_async(self.h, _p(x_host), _p(dy_host), _p(y_host), _p(dx_host)))

    def wait_host(self):
        """Wait for every step_host_async submitted so far."""
        check(lib.fmoe_layer_step_host_wait(self.h))


def _wrap(ptr: int, shape, dtype, device, owner):
    """A torch view of library-owned device memory (kept alive by `owner`)."""
    n = 1
    for s in shape:
        n *= s
    esz = torch.empty((), dtype=dtype).element_size()
    t = _from_ptr(ptr, n * esz, device).view(dtype)[:n].view(*shape)
    t._fmoe_owner = owner
    return t


def _from_ptr(ptr: int, nbytes: int, device) -> torch.Tensor:
    class _Holder:
        pass

    h = _Holder()
    h.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
    return torch.as_tensor(h, device=device)


def launches() -> int:
    return Context.get().launches


def version() -> str:
    return lib.fmoe_version().decode()
