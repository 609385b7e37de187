"""Expert parallelism on one B200: W ranks as host threads of this process
(the reference's run_world_inproc pattern, test_support.hpp:96-120), each
with its own context, stream and MoE layer, joined to an fmoe_world whose
transport moves rows with device copies.  The data path (count exchange,
global_scatter into aligned receive blocks, grouped experts, global_gather,
gradients on the same routes) is the one the NCCL transport drives.

Checks: the EP result equals the single-worker result on the
rank-major concatenated batch bit-for-bit (deterministic kernels, receive
order == the single worker's stable order); per-rank gate gradients equal
the single worker's on the rank's own rows; f64 matches the reference's
InProcWorld golden within the exp-ulp tolerance.
"""
import os
import threading

import numpy as np
import pytest
import torch

from tests.gpu_util import dev, host

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def fm():
    import paper_2103_13262_b200 as m

    return m


def run_world(fm, world, cfg, dtype, xs, dys, exchange="peer", steps=1):
    """One thread per rank; returns per-rank dicts of host arrays (last step)."""
    w = fm.World(world)
    out = [None] * world
    errs = [None] * world

    def body(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                layer = fm.MoELayer(cfg, rank=r, dtype=dtype)
                layer.join(w)
                layer.set_ep_exchange(exchange)
                x = xs[r].to(device="cuda", dtype=dtype)
                dy = dys[r].to(device="cuda", dtype=dtype)
                for _ in range(steps):
                    y = layer.forward(x)
                    dx = layer.backward(dy)
                s.synchronize()
                out[r] = dict(y=y.cpu(), dx=dx.cpu(), dwg=layer.d_wg.cpu(), dw1=layer.grads.d_w1.cpu(),
                              db1=layer.grads.d_b1.cpu(), dw2=layer.grads.d_w2.cpu(), db2=layer.grads.d_b2.cpu(),
                              idx=layer.routing()[0].cpu(), fused=layer.ep_exchange_fused)
                del layer
        except Exception as e:  # surfaced below
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=100)
    for e in errs:
        if e is not None:
            raise e
    return out


def single(fm, cfg, dtype, x, dy):
    layer = fm.MoELayer(cfg, dtype=dtype)
    y = layer.forward(x.to(device="cuda", dtype=dtype))
    dx = layer.backward(dy.to(device="cuda", dtype=dtype))
    torch.cuda.synchronize()
    return dict(y=y.cpu(), dx=dx.cpu(), dwg=layer.d_wg.cpu(), dw1=layer.grads.d_w1.cpu(), db1=layer.grads.d_b1.cpu(),
                dw2=layer.grads.d_w2.cpu(), db2=layer.grads.d_b2.cpu())


def check_ep_equals_single(fm, world, n, d, h, el, k, dtype, seed=3, exchange="peer", steps=1):
    g = torch.Generator().manual_seed(seed)
    xs = [(torch.rand(n, d, generator=g) * 2 - 1).to(dtype) for _ in range(world)]
    dys = [(torch.rand(n, d, generator=g) * 2 - 1).to(dtype) for _ in range(world)]
    ep = run_world(fm, world, fm.MoEConfig(n, d, h, k, el, world, seed), dtype, xs, dys, exchange, steps)
    # bf16 + peer: the fused exchange (scatter / epilogues over peer memory) ran
    assert all(o["fused"] == (dtype == torch.bfloat16 and exchange == "peer") for o in ep)
    ref = single(fm, fm.MoEConfig(n * world, d, h, k, el * world, 1, seed), dtype, torch.cat(xs), torch.cat(dys))
    assert torch.equal(torch.cat([o["y"] for o in ep]), ref["y"])
    assert torch.equal(torch.cat([o["dx"] for o in ep]), ref["dx"])
    for key in ("dw1", "db1", "dw2", "db2"):
        assert torch.equal(torch.cat([o[key] for o in ep]), ref[key]), key
    for r in range(world):  # each rank differentiates the gate on its own rows
        own = single(fm, fm.MoEConfig(n, d, h, k, el * world, 1, seed), dtype, xs[r], dys[r])
        assert torch.equal(ep[r]["dwg"], own["dwg"])


@pytest.mark.parametrize("exchange", ["peer", "transport"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_ep_bf16_equals_single_worker(fm, world, exchange):
    check_ep_equals_single(fm, world, n=512, d=128, h=256, el=4, k=2, dtype=torch.bfloat16, exchange=exchange)


@pytest.mark.parametrize("exchange", ["peer", "transport"])
def test_ep_bf16_skewed_and_empty_experts(fm, exchange):
    """k=1 with few tokens: some experts receive nothing from some (or all) ranks."""
    check_ep_equals_single(fm, 4, n=40, d=64, h=128, el=2, k=1, dtype=torch.bfloat16, seed=11, exchange=exchange)


def test_ep_bf16_pair_tiles_repeated_steps(fm):
    """>= 1024 rows per local expert: 256-row blocks and CTA-pair GEMMs on the
    fused path; three steps in a row reuse the peer buffers and epoch flags."""
    check_ep_equals_single(fm, 2, n=4096, d=128, h=256, el=4, k=2, dtype=torch.bfloat16, seed=5, steps=3)


@pytest.mark.parametrize("world", [2, 4])
def test_ep_f64_equals_single_worker(fm, world):
    check_ep_equals_single(fm, world, n=48, d=16, h=24, el=2, k=2, dtype=torch.float64)


@pytest.mark.parametrize("name", ["dist_w2", "dist_w4"])
def test_ep_f64_vs_reference_golden(fm, orc, name):
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    seed, world, n, d, h, el, k = (int(v) for v in g["meta"])
    xs = [torch.from_numpy(orc.seeded_matrix(seed, 200 + r, n, d)) for r in range(world)]
    dys = [torch.from_numpy(orc.seeded_matrix(seed, 300 + r, n, d)) for r in range(world)]
    ep = run_world(fm, world, fm.MoEConfig(n, d, h, k, el, world, seed), torch.float64, xs, dys)
    # bit-identical to the reference's InProcWorld run (glibc exp included)
    same = lambda a, b: a.tobytes() == np.ascontiguousarray(b).tobytes()  # noqa: E731
    assert same(torch.cat([o["y"] for o in ep]).numpy(), g["y"])
    assert same(torch.cat([o["dx"] for o in ep]).numpy(), g["dx"])
    for key in ("dw1", "db1", "dw2", "db2"):
        assert same(torch.cat([o[key] for o in ep]).numpy(), g[key]), key
    for r in range(world):
        assert same(ep[r]["dwg"].numpy(), g["dwg"][r])


def test_exchange_operators_hand_example(fm):
    """exchange_counts / all_to_all_rows(_reverse) (test_comm.cpp:87-104, 170-246)."""
    world = 2
    w = fm.World(world)
    res = [None] * world
    errs = [None] * world
    counts = [[3, 5], [2, 4]]

    def body(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = fm.Context(0).use_current_stream()
                ctx.join_world(w, r)
                plan = fm.exchange_counts(counts[r], ctx)
                rows = sum(counts[r])
                xs = torch.arange(rows * 2, dtype=torch.float64, device="cuda").view(rows, 2) + 100 * r
                got = fm.all_to_all_rows(xs, plan, ctx)
                back = fm.all_to_all_rows_reverse(got, plan, ctx)
                s.synchronize()
                res[r] = (plan, xs.cpu(), got.cpu(), back.cpu())
        except Exception as e:
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join(timeout=120) for t in th]
    for e in errs:
        if e is not None:
            raise e
    p0, p1 = res[0][0], res[1][0]
    assert p0.recv_counts.tolist() == [[3], [2]] and p0.recv_total == 5 and p0.send_total == 8
    assert p1.recv_counts.tolist() == [[5], [4]] and p1.recv_total == 9 and p1.send_total == 6
    # rank 0 receives its own first 3 rows then rank 1's first 2 rows
    assert torch.equal(res[0][2], torch.cat([res[0][1][:3], res[1][1][:2]]))
    assert torch.equal(res[1][2], torch.cat([res[0][1][3:], res[1][1][2:]]))
    for r in range(world):  # exact inverse routing
        assert torch.equal(res[r][3], res[r][1])


def test_ep_needs_transport(fm):
    layer = fm.MoELayer(fm.MoEConfig(16, 64, 64, 1, 4, 2, 0), rank=0, dtype=torch.bfloat16)
    with pytest.raises(fm.ProtocolError):
        layer.forward(torch.zeros(16, 64, dtype=torch.bfloat16, device="cuda"))


def _threads(fm, world, body):
    w = fm.World(world)
    res, errs = [None] * world, [None] * world

    def run(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = fm.Context(0).use_current_stream()
                ctx.join_world(w, r)
                res[r] = body(r, ctx)
                s.synchronize()
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join(timeout=150) for t in th]
    return res, errs


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_allreduce_sum_ascending_rank_order(fm, dtype):
    """allreduce_sum (collectives.cpp:266-292; test_comm.cpp:256-292): the sum is
    accumulated in ascending rank order and every member gets the same bytes."""
    world = 4
    g = torch.Generator().manual_seed(5)
    ms = [torch.rand(7, 5, generator=g, dtype=torch.float64).to(dtype) * 10 ** r for r in range(world)]
    groups = {0: [0, 1, 2, 3], 1: [0, 1, 2, 3], 2: [0, 1, 2, 3], 3: [0, 1, 2, 3]}

    def body(r, ctx):
        full = fm.allreduce_sum(ms[r].cuda(), groups[r], ctx).cpu()
        # data-parallel style subgroups {0, 2} and {1, 3}
        sub = fm.allreduce_sum(ms[r].cuda(), [r % 2, r % 2 + 2], ctx).cpu()
        return full, sub

    res, errs = _threads(fm, world, body)
    for e in errs:
        if e is not None:
            raise e
    want = ((ms[0] + ms[1]) + ms[2]) + ms[3]
    for r in range(world):
        assert torch.equal(res[r][0], want)
        assert torch.equal(res[r][1], ms[r % 2] + ms[r % 2 + 2])


def test_allreduce_sum_detects_shape_mismatch(fm):
    """Ranks contributing different sizes raise ProtocolError on every member
    (test_comm.cpp:294-316)."""
    def body(r, ctx):
        return fm.allreduce_sum(torch.ones(3 + r, dtype=torch.float64, device="cuda"), [0, 1], ctx)

    res, errs = _threads(fm, 2, body)
    assert all(isinstance(e, fm.ProtocolError) for e in errs), errs


def test_allreduce_sum_rejects_bad_groups(fm):
    def body(r, ctx):
        out = []
        for grp in ([], [1, 0], [1 - r]):
            try:
                fm.allreduce_sum(torch.ones(2, dtype=torch.float64, device="cuda"), grp, ctx)
                out.append(None)
            except fm.ProtocolError as e:
                out.append(e)
        return out

    res, errs = _threads(fm, 2, body)
    assert errs == [None, None]
    for r in range(2):
        assert all(isinstance(e, fm.ProtocolError) for e in res[r]), res[r]


def test_nccl_transport_single_rank(fm):
    """The NCCL transport initialises (one rank: NCCL refuses two ranks on one
    GPU) and carries the operator-level collectives through it."""
    import ctypes as C

    from paper_2103_13262_b200 import _lib

    ctx = fm.Context(0)
    uid = (C.c_char * 128)()
    _lib.check(_lib.lib.fmoe_comm_unique_id(uid, 128))
    _lib.check(_lib.lib.fmoe_comm_init(ctx.h, uid, 128, 1, 0))
    plan = fm.exchange_counts([3, 1, 4], ctx)
    assert plan.world == 1 and plan.recv_counts.tolist() == [[3, 1, 4]]
    buf = torch.arange(6, dtype=torch.float32, device="cuda").reshape(2, 3)
    out = fm.allreduce_sum(buf.clone(), [0], ctx=ctx)
    assert torch.equal(out.cpu(), buf.cpu())


def test_nccl_attach_borrowed_communicator(fm):
    """fmoe_comm_attach: a communicator the host already owns (made here
    through libnccl itself) carries the collectives; world / rank are read from
    it and it is still usable by its owner after the context is gone."""
    import ctypes as C

    from paper_2103_13262_b200 import _lib

    class UniqueId(C.Structure):  # ncclUniqueId: 128 bytes, passed by value
        _fields_ = [("internal", C.c_char * 128)]

    nccl = C.CDLL("libnccl.so.2")  # the process's (already loaded) libnccl
    nccl.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, UniqueId, C.c_int]
    uid = UniqueId()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    try:
        ctx = fm.Context(0)
        ctx.attach_nccl(comm.value)
        plan = fm.exchange_counts([2, 0, 5], ctx)
        assert plan.world == 1 and plan.rank == 0 and plan.recv_counts.tolist() == [[2, 0, 5]]
        buf = torch.arange(6, dtype=torch.float64, device="cuda").reshape(3, 2)
        assert torch.equal(fm.allreduce_sum(buf.clone(), [0], ctx=ctx).cpu(), buf.cpu())
        del ctx
        n = C.c_int()
        assert nccl.ncclCommCount(comm, C.byref(n)) == 0 and n.value == 1  # not destroyed by the context
    finally:
        nccl.ncclCommDestroy(comm)
    with pytest.raises(fm.ShapeError):
        fm.Context(0).attach_nccl(0)


def test_ep_routed_equals_single_worker(fm):
    """Injected (Zipf) routing under expert parallelism (cfg5 at N>1): the
    fused exchange gives the single worker's results on the concatenated batch."""
    from paper_2103_13262_b200.workloads import zipf_routing

    W, n, d, h, el, k = 2, 1024, 128, 256, 8, 1
    g = torch.Generator().manual_seed(8)
    xs = [(torch.rand(n, d, generator=g) * 2 - 1).bfloat16() for _ in range(W)]
    dys = [(torch.rand(n, d, generator=g) * 2 - 1).bfloat16() for _ in range(W)]
    routes = [zipf_routing(n, el * W, k, 1.0, seed=30 + r) for r in range(W)]
    world = fm.World(W)
    out, errs = [None] * W, [None] * W

    def body(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, el, W, 9), rank=r, dtype=torch.bfloat16)
                layer.join(world)
                idx = torch.as_tensor(routes[r][0], device="cuda")
                sc = torch.as_tensor(routes[r][1], device="cuda")
                y = layer.forward_routed(xs[r].cuda(), idx, sc)
                dx = layer.backward(dys[r].cuda())
                s.synchronize()
                out[r] = (y.cpu(), dx.cpu(), layer.grads.d_w2.cpu(), layer.routing_grad().cpu(),
                          layer.ep_exchange_fused)
                del layer
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(W)]
    [t.start() for t in th]
    [t.join(timeout=120) for t in th]
    for e in errs:
        if e is not None:
            raise e
    single = fm.MoELayer(fm.MoEConfig(n * W, d, h, k, el * W, 1, 9), dtype=torch.bfloat16)
    idx = torch.as_tensor(np.concatenate([r[0] for r in routes]), device="cuda")
    sc = torch.as_tensor(np.concatenate([r[1] for r in routes]), device="cuda")
    y = single.forward_routed(torch.cat(xs).cuda(), idx, sc)
    dx = single.backward(torch.cat(dys).cuda())
    torch.cuda.synchronize()
    assert all(o[4] for o in out)
    assert torch.equal(torch.cat([o[0] for o in out]), y.cpu())
    assert torch.equal(torch.cat([o[1] for o in out]), dx.cpu())
    assert torch.equal(torch.cat([o[2] for o in out]), single.grads.d_w2.cpu())
    assert torch.equal(torch.cat([o[3] for o in out]), single.routing_grad().cpu())
