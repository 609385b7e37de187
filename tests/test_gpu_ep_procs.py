"""Expert parallelism across PROCESSES: two ranks, one process each, sharing
the one GPU of the test box -- the one-process-per-GPU deployment minus the
second GPU.  The peer buffers are exchanged through torch.distributed/gloo
(fmoe_layer_peer_connect), mapped with CUDA IPC, and the phases are ordered
by epoch flags written into peer memory and awaited with stream memory
operations: exactly the cross-process code path of an 8-GPU run.  The result
must equal the single-worker layer on the concatenated batch bit for bit.
"""
import os
import socket
import traceback

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N, D, H, EL, K, SEED, STEPS = 2048, 128, 256, 4, 2, 7, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(world):
    g = torch.Generator().manual_seed(SEED)
    xs = [(torch.rand(N, D, generator=g) * 2 - 1).bfloat16() for _ in range(world)]
    dys = [(torch.rand(N, D, generator=g) * 2 - 1).bfloat16() for _ in range(world)]
    return xs, dys


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2103_13262_b200 as fm

        xs, dys = _inputs(world)
        layer = fm.MoELayer(fm.MoEConfig(N, D, H, K, EL, world, SEED), rank=rank, dtype=torch.bfloat16)
        layer.connect_peers(dist)
        x, dy = xs[rank].cuda(), dys[rank].cuda()
        for _ in range(STEPS):
            y = layer.forward(x)
            dx = layer.backward(dy)
        torch.cuda.synchronize()
        # plain numpy through the queue (bf16 as its raw 16-bit patterns)
        out = dict(y=y.cpu().view(torch.int16).numpy(), dx=dx.cpu().view(torch.int16).numpy(),
                   dw1=layer.grads.d_w1.cpu().numpy(), db2=layer.grads.d_b2.cpu().numpy(),
                   fused=layer.ep_exchange_fused)
        dist.barrier()  # peers stop writing into this rank before it frees its buffers
        del layer
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


def test_ep_two_processes_peer_memory():
    import paper_2103_13262_b200 as fm

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, err = q.get(timeout=240)
        assert err is None, f"rank {r}:\n{err}"
        res[r] = out
    for p in procs:
        p.join(timeout=60)
    xs, dys = _inputs(world)
    single = fm.MoELayer(fm.MoEConfig(N * world, D, H, K, EL * world, 1, SEED), dtype=torch.bfloat16)
    y = single.forward(torch.cat(xs).cuda())
    dx = single.backward(torch.cat(dys).cuda())
    torch.cuda.synchronize()
    assert all(res[r]["fused"] for r in range(world))
    cat = lambda key: np.concatenate([res[r][key] for r in range(world)])  # noqa: E731
    assert np.array_equal(cat("y"), y.cpu().view(torch.int16).numpy())
    assert np.array_equal(cat("dx"), dx.cpu().view(torch.int16).numpy())
    assert np.array_equal(cat("dw1"), single.grads.d_w1.cpu().numpy())
    assert np.array_equal(cat("db2"), single.grads.d_b2.cpu().numpy())
