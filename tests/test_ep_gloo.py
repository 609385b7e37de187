"""Expert parallelism on CPU: world_size 2 and 4 over torch.distributed/gloo.

Each process is one rank.  Routing comes from the oracle on the rank's own
seeded tokens; the count exchange and the token exchange run over gloo, laid
out by the library's own host layout code (fmoe_ep_layout, the same function
the NCCL path uses).  Checked against the reference: the received rows equal
all_to_all_rows (collectives.cpp:146-203) and the full EP forward/backward
through this layout reproduces the reference's InProcWorld golden outputs
bit-for-bit (tests/golden/dist_w*.npz).
"""
import os
import socket
import traceback

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(rank, world, el, send_counts, recv_counts, send_buf, align, d):
    """Token all-to-all over gloo laid out by fmoe_ep_layout."""
    import paper_2103_13262_b200 as fm

    so, co, bo, rows = fm.ep_layout(world, el, align, send_counts, recv_counts)
    recv = np.zeros((bo[-1], d))
    ops, keep = [], []
    for p in range(world):
        for e in range(el):
            g = p * el + e
            ns, nr = int(send_counts.reshape(-1)[g]), int(recv_counts.reshape(-1)[g])
            if p == rank:
                recv[co[e, p]:co[e, p] + nr] = send_buf[so[g]:so[g] + ns]
                continue
            if ns:
                t = torch.from_numpy(np.ascontiguousarray(send_buf[so[g]:so[g] + ns]))
                keep.append(t)
                ops.append(dist.P2POp(dist.isend, t, p))
            if nr:
                t = torch.empty(nr, d, dtype=torch.float64)
                keep.append((t, e, p))
                ops.append(dist.P2POp(dist.irecv, t, p))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for item in keep:
        if isinstance(item, tuple):
            t, e, p = item
            recv[co[e, p]:co[e, p] + t.shape[0]] = t.numpy()
    return recv, so, co, bo, rows


def _reverse(rank, world, el, send_counts, recv_counts, recv_buf, so, co, d):
    n_send = int(send_counts.sum())
    out = np.zeros((n_send, d))
    ops, keep = [], []
    for p in range(world):
        for e in range(el):
            g = p * el + e
            ns, nr = int(send_counts.reshape(-1)[g]), int(recv_counts.reshape(-1)[g])
            if p == rank:
                out[so[g]:so[g] + ns] = recv_buf[co[e, p]:co[e, p] + nr]
                continue
            if nr:
                t = torch.from_numpy(np.ascontiguousarray(recv_buf[co[e, p]:co[e, p] + nr]))
                keep.append(t)
                ops.append(dist.P2POp(dist.isend, t, p))
            if ns:
                t = torch.empty(ns, d, dtype=torch.float64)
                keep.append((t, g))
                ops.append(dist.P2POp(dist.irecv, t, p))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for item in keep:
        if isinstance(item, tuple):
            t, g = item
            out[so[g]:so[g] + t.shape[0]] = t.numpy()
    return out


def _fused_push(rank, world, el, align, counts_all, send_buf, d):
    """The fused global_scatter (peer.cuh) emulated over gloo: every send row
    goes to rank g_rank[g] at receive row (position + g_delta[g]) as
    fmoe_ep_routes lays it out."""
    import paper_2103_13262_b200 as fm

    so, co, bo, rows, gr, gd, rt = fm.ep_routes(world, rank, el, align, counts_all)
    e = world * el
    dest_rank = np.repeat(gr, counts_all[rank])
    dest_row = np.arange(send_buf.shape[0]) + np.repeat(gd, counts_all[rank])
    out = [torch.from_numpy(np.ascontiguousarray(np.c_[dest_row[dest_rank == p], send_buf[dest_rank == p]]))
           for p in range(world)]
    got = [None] * world
    dist.all_gather_object(got, out)
    recv = np.zeros((bo[-1], d))
    for s in range(world):
        blk = got[s][rank].numpy()
        recv[blk[:, 0].astype(np.int64)] = blk[:, 1:]
    return recv, (so, co, bo, rows, gr, gd, rt)


def _fused_home(rank, world, el, counts_all, recv_buf, routes, d):
    """The fused global_gather (the fc2 / dgrad-fc1 epilogue route): receive
    chunk (e, s) goes back to rank s at route[2][e, s] + offset."""
    so, co, bo, rows, gr, gd, rt = routes
    out = [[] for _ in range(world)]
    for e in range(el):
        for s in range(world):
            start, n, dst = int(rt[0, e, s]), int(rt[1, e, s]), int(rt[2, e, s])
            if n:
                out[s].append(np.c_[np.arange(dst, dst + n), recv_buf[start:start + n]])
    out = [torch.from_numpy(np.concatenate(o) if o else np.zeros((0, d + 1))) for o in out]
    got = [None] * world
    dist.all_gather_object(got, out)
    home = np.zeros((int(counts_all[rank].sum()), d))
    for s in range(world):
        blk = got[s][rank].numpy()
        home[blk[:, 0].astype(np.int64)] = blk[:, 1:]
    return home


def _worker(rank, world, port, name, align, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import orc

        g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
        seed, W, n, d, h, el, k = (int(v) for v in g["meta"])
        assert W == world
        e = el * world
        w = orc.init_state(seed, d, h, e)
        xs_all = [orc.seeded_matrix(seed, 200 + r, n, d) for r in range(world)]
        dys_all = [orc.seeded_matrix(seed, 300 + r, n, d) for r in range(world)]
        x, dy = xs_all[rank], dys_all[rank]
        scores, idx, vals = orc.gate_forward(x, w["wg"], k)
        plan = orc.build_plan(idx, e)
        xs_send = orc.scatter(x, plan)
        # count exchange (C1) over gloo
        counts = torch.from_numpy(plan["counts"].astype(np.int64))
        recv = torch.empty_like(counts)
        dist.all_to_all_single(recv, counts, [el] * world, [el] * world)
        send_counts = plan["counts"].reshape(world, el)
        recv_counts = recv.numpy().reshape(world, el)
        assert np.array_equal(recv_counts, g["recv_counts"][rank].reshape(world, el))
        # token exchange (C2) with the library's layout
        xs_recv, so, co, bo, rows = _exchange(rank, world, el, send_counts, recv_counts, xs_send, align, d)
        # reference order of the received rows (collectives.cpp:146-203)
        all_counts = []
        for r in range(world):
            _, ir, _ = orc.gate_forward(xs_all[r], w["wg"], k)
            all_counts.append(orc.build_plan(ir, e)["counts"])
        sends_all = []
        for r in range(world):
            _, ir, _ = orc.gate_forward(xs_all[r], w["wg"], k)
            sends_all.append(orc.scatter(xs_all[r], orc.build_plan(ir, e)))
        want = orc.all_to_all_rows(sends_all, np.stack(all_counts), rank)
        dense = np.concatenate([xs_recv[bo[j]:bo[j] + rows[j]] for j in range(el)])
        assert dense.tobytes() == want.tobytes()
        assert all(not xs_recv[bo[j] + rows[j]:bo[j + 1]].any() for j in range(el))  # zero padding
        # the fused peer-memory routes (fmoe_ep_routes) land every row where the
        # transport exchange does, from the all-gathered counts alone
        cl = [torch.zeros(world * el, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(cl, torch.from_numpy(plan["counts"].astype(np.int64)))
        counts_all = torch.stack(cl).numpy()
        xs_fused, routes = _fused_push(rank, world, el, align, counts_all, xs_send, d)
        assert xs_fused.tobytes() == xs_recv.tobytes()
        assert np.array_equal(routes[0], so) and np.array_equal(routes[1], co) and np.array_equal(routes[2], bo)
        # experts on the received blocks, reverse exchange (C3), combine
        ys_recv = np.zeros_like(xs_recv)
        cache = []
        for j in range(el):
            gl = rank * el + j
            blk = xs_recv[bo[j]:bo[j] + rows[j]]
            yj, pre, hid = orc.expert_forward(blk, w["w1"][gl], w["b1"][gl], w["w2"][gl], w["b2"][gl])
            ys_recv[bo[j]:bo[j] + rows[j]] = yj
            cache.append((pre, hid))
        ys_send = _reverse(rank, world, el, send_counts, recv_counts, ys_recv, so, co, d)
        assert _fused_home(rank, world, el, counts_all, ys_recv, routes, d).tobytes() == ys_send.tobytes()
        y = orc.gather_combine(ys_send, plan, vals)
        assert y.tobytes() == g["y"][rank * n:(rank + 1) * n].tobytes()
        # backward through the same routes
        d_ys_send, d_w = orc.gather_combine_backward(dy, ys_send, plan, vals)
        d_ys_recv, *_ = _exchange(rank, world, el, send_counts, recv_counts, d_ys_send, align, d)
        d_xs_recv = np.zeros_like(xs_recv)
        for j in range(el):
            gl = rank * el + j
            a, c = bo[j], rows[j]
            dxj, gr = orc.expert_backward(d_ys_recv[a:a + c], xs_recv[a:a + c], cache[j][0], cache[j][1],
                                          w["w1"][gl], w["w2"][gl])
            d_xs_recv[a:a + c] = dxj
            for key in ("dw1", "db1", "dw2", "db2"):
                assert gr[key].tobytes() == g[key][gl].tobytes(), key
        d_xs_send = _reverse(rank, world, el, send_counts, recv_counts, d_xs_recv, so, co, d)
        dxs = orc.scatter_backward(d_xs_send, plan)
        d_wg, gdx = orc.gate_backward(x, w["wg"], scores, idx, d_w)
        assert d_wg.tobytes() == g["dwg"][rank].tobytes()
        assert (dxs + gdx).tobytes() == g["dx"][rank * n:(rank + 1) * n].tobytes()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, None))
    except Exception:
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("name,world", [("dist_w2", 2), ("dist_w4", 4)])
@pytest.mark.parametrize("align", [1, 128])
def test_ep_exchange_over_gloo(name, world, align):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, align, q)) for r in range(world)]
    for p in procs:
        p.start()
    errs = {}
    for _ in range(world):
        r, e = q.get(timeout=240)
        errs[r] = e
    for p in procs:
        p.join(timeout=60)
    bad = {r: e for r, e in errs.items() if e}
    assert not bad, "\n".join(f"rank {r}:\n{e}" for r, e in bad.items())
