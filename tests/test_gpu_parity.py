"""GPU parity: the sm_100a kernels through the C-ABI vs the oracle.

Bar (SURVEY §8c parity protocol):
  * integers (routing, counts, offsets, positions): bit-exact;
  * FMOE_F64 parity mode: bit-exact on every operator whose reference
    arithmetic has no transcendental (plan, permutes, expert pool, gate
    backward given the scores); softmax scores within 4 ulp (CUDA exp vs
    glibc exp), top-k exact;
  * FMOE_BF16 product path vs the oracle fed the same bf16-rounded values:
    outputs rel-L2 <= 1e-2, gradients rel-L2 <= 2e-2, routing exact on
    well-separated tokens.
"""
import numpy as np
import pytest
import torch

from tests.gpu_util import beq, bf16_round, dev, host, random_assignment, rel_l2, well_separated_rows

pytestmark = pytest.mark.gpu

TOL_Y_BF16 = 1e-2
TOL_G_BF16 = 2e-2


@pytest.fixture(scope="module")
def fm():
    import paper_2103_13262_b200 as m

    return m


# ------------------------------------------------------------------ plan
PLAN_CASES = [(3, 2, 3), (1, 1, 1), (5, 1, 3), (777, 2, 16), (4096, 2, 64), (5000, 3, 7), (20000, 1, 256),
              (65536, 2, 64)]


@pytest.mark.parametrize("n,k,e", PLAN_CASES)
def test_plan_bit_exact(fm, orc, n, k, e):
    rng = np.random.default_rng(n * 31 + k * 7 + e)
    idx = random_assignment(rng, n, k, e) if n < 6000 else rng.integers(0, e, (n, k))
    want = orc.build_plan(idx, e)
    p = fm.build_plan(dev(idx, torch.int32), e, align=1)
    assert beq(host(p.counts).astype(np.int64), want["counts"])
    assert beq(host(p.offsets)[:e].astype(np.int64), want["offsets"])
    assert host(p.offsets)[e] == n * k
    assert beq(host(p.expanded_src_row).astype(np.int64), want["src_row"])
    assert beq(host(p.expanded_slot).astype(np.int64), want["slot"])
    assert beq(host(p.inverse_pos).astype(np.int64), want["inverse_pos"])


def test_plan_hand_example(fm):
    # test_dispatch.cpp:35-51
    p = fm.build_plan(dev([[1, 2], [0, 1], [1, 0]], torch.int32), 3)
    assert host(p.counts).tolist() == [2, 3, 1]
    assert host(p.offsets).tolist() == [0, 2, 5, 6]
    assert host(p.expanded_src_row).tolist() == [1, 2, 0, 1, 2, 0]
    assert host(p.expanded_slot).tolist() == [0, 1, 0, 1, 0, 1]
    assert host(p.inverse_pos).tolist() == [[2, 5], [0, 3], [4, 1]]


@pytest.mark.parametrize("align", [128, 256])
@pytest.mark.parametrize("n,k,e", [(777, 2, 16), (4096, 2, 64), (20000, 1, 256), (300, 2, 40)])
def test_plan_aligned_layout(fm, orc, n, k, e, align):
    """aligned plans: same stable order inside each block, blocks start on tiles."""
    rng = np.random.default_rng(5 + n)
    p_ = 1.0 / np.arange(1, e + 1)
    idx = np.stack([rng.choice(e, size=k, replace=False, p=p_ / p_.sum()) for _ in range(n)])
    want = orc.build_plan(idx, e)
    p = fm.build_plan(dev(idx, torch.int32), e, align=align)
    counts = host(p.counts).astype(np.int64)
    off = host(p.offsets).astype(np.int64)
    assert beq(counts, want["counts"])
    assert (off % align == 0).all()
    assert np.array_equal(np.diff(off), (counts + align - 1) // align * align)
    inv = host(p.inverse_pos).astype(np.int64)
    e_of = idx
    assert np.array_equal(inv - off[e_of], want["inverse_pos"] - want["offsets"][e_of])
    src = host(p.expanded_src_row)
    for g in range(e):
        pad = src[off[g] + counts[g]: off[g + 1]]
        assert (pad == -1).all()
    n_tiles = int(host(p.n_tiles)[0])
    assert n_tiles == off[e] // 128
    te = host(p.tile_expert)[:n_tiles]
    assert np.array_equal(te, np.repeat(np.arange(e), np.diff(off) // 128))


def test_plan_golden_zipf(fm):
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "plan_zipf.npz"))
    p = fm.build_plan(dev(g["idx"], torch.int32), 64)
    assert beq(host(p.inverse_pos).astype(np.int64), g["inverse_pos"])
    assert beq(host(p.expanded_src_row).astype(np.int64), g["src_row"])


@pytest.mark.parametrize("bad", [3, -1])
def test_plan_rejects_out_of_range(fm, bad):
    with pytest.raises(fm.ShapeError):
        fm.build_plan(dev([[0], [bad]], torch.int32), 3)
    # the error flag is consumed: a valid plan afterwards is fine
    fm.build_plan(dev([[0], [2]], torch.int32), 3)


def test_empty_experts_legal(fm):
    # test_dispatch.cpp:286-298
    idx = np.ones((4, 1), np.int64)
    p = fm.build_plan(dev(idx, torch.int32), 3)
    assert host(p.counts).tolist() == [0, 4, 0]
    x = dev(np.random.default_rng(38).uniform(-1, 1, (4, 3)))
    xs = fm.scatter(x, p)
    y = fm.gather_combine(xs, p, torch.ones(4, 1, dtype=torch.float64, device="cuda"))
    assert beq(host(y), host(x))


# -------------------------------------------------------------- permutes
@pytest.mark.parametrize("n,k,e,d", [(37, 2, 5, 16), (300, 3, 8, 33), (1000, 2, 16, 128), (64, 1, 4, 7)])
def test_permutes_f64_bit_exact(fm, orc, n, k, e, d):
    rng = np.random.default_rng(n + d)
    idx = random_assignment(rng, n, k, e)
    plan_o = orc.build_plan(idx, e)
    p = fm.build_plan(dev(idx, torch.int32), e)
    x = rng.uniform(-1, 1, (n, d))
    w = rng.uniform(0, 1, (n, k))
    ys = rng.uniform(-1, 1, (n * k, d))
    dy = rng.uniform(-1, 1, (n, d))
    assert beq(host(fm.scatter(dev(x), p)), orc.scatter(x, plan_o))
    assert beq(host(fm.gather_combine(dev(ys), p, dev(w))), orc.gather_combine(ys, plan_o, w))
    assert beq(host(fm.scatter_backward(dev(ys), p)), orc.scatter_backward(ys, plan_o))
    d_ys, d_w = fm.gather_combine_backward(dev(dy), dev(ys), p, dev(w))
    o_dys, o_dw = orc.gather_combine_backward(dy, ys, plan_o, w)
    assert beq(host(d_ys), o_dys)
    assert beq(host(d_w), o_dw)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_permutes_low_precision(fm, orc, dtype):
    rng = np.random.default_rng(7)
    n, k, e, d = 2000, 2, 16, 256
    idx = random_assignment(rng, n, k, e)
    plan_o = orc.build_plan(idx, e)
    x = bf16_round(rng.uniform(-1, 1, (n, d)))
    w = rng.uniform(0, 1, (n, k)).astype(np.float32).astype(np.float64)
    ys = bf16_round(rng.uniform(-1, 1, (n * k, d)))
    dy = bf16_round(rng.uniform(-1, 1, (n, d)))
    for align in (1, 128):
        p = fm.build_plan(dev(idx, torch.int32), e, align=align)
        inv = host(p.inverse_pos).astype(np.int64)
        ysa = np.zeros((p.capacity, d))
        ysa[inv.reshape(-1)] = ys[plan_o["inverse_pos"].reshape(-1)]
        xs = host(fm.scatter(dev(x, dtype), p))
        assert beq(xs[inv.reshape(-1)], x[np.repeat(np.arange(n), k)])  # copies are exact
        if align == 128:
            src = host(p.expanded_src_row)
            assert (xs[: host(p.offsets)[-1]][src[: host(p.offsets)[-1]] == -1] == 0).all()
        y = host(fm.gather_combine(dev(ysa, dtype), p, dev(w, torch.float32)))
        tol = 1e-6 if dtype == torch.float32 else 1e-2
        assert rel_l2(y, orc.gather_combine(ys, plan_o, w)) < tol
        dx = host(fm.scatter_backward(dev(ysa, dtype), p))
        assert rel_l2(dx, orc.scatter_backward(ys, plan_o)) < tol
        d_ys, d_w = fm.gather_combine_backward(dev(dy, dtype), dev(ysa, dtype), p, dev(w, torch.float32))
        o_dys, o_dw = orc.gather_combine_backward(dy, ys, plan_o, w)
        assert rel_l2(host(d_ys)[inv.reshape(-1)], o_dys[plan_o["inverse_pos"].reshape(-1)]) < tol
        assert rel_l2(host(d_w), o_dw) < 1e-5
        if align == 128:  # padding rows of d_ys are zero (the wgrad contract)
            src = host(p.expanded_src_row)
            end = host(p.offsets)[-1]
            assert (host(d_ys)[:end][src[:end] == -1] == 0).all()


# ------------------------------------------------------------------- gate
@pytest.mark.parametrize("n,d,e,k", [(37, 16, 5, 2), (300, 64, 16, 3), (2048, 128, 64, 2), (50, 8, 1, 1)])
def test_gate_f64(fm, orc, n, d, e, k):
    rng = np.random.default_rng(n + e)
    x = rng.uniform(-1, 1, (n, d))
    wg = rng.uniform(-0.1, 0.1, (d, e))
    s_o, i_o, v_o = orc.gate_forward(x, wg, k)
    out = fm.gate_forward(dev(x), dev(wg), k)
    s = host(out.scores)
    # the parity mode computes exp as glibc does (glibc_exp.cuh): scores, and
    # therefore the routing, are bit-identical to the reference's
    assert beq(s, s_o)
    assert beq(host(out.topk_indices).astype(np.int64), i_o)
    assert beq(host(out.topk_scores), v_o)
    # backward given identical scores is exp-free: bit-exact
    dt = rng.uniform(-1, 1, (n, k))
    gw_o, gx_o = orc.gate_backward(x, wg, s_o, i_o, dt)
    g = fm.gate_backward(dev(x), dev(wg), fm.GateOutput(dev(s_o), dev(i_o, torch.int32), dev(v_o)), dev(dt))
    assert beq(host(g.d_wg), gw_o)
    assert beq(host(g.d_x), gx_o)


def test_softmax_f64_is_glibc_bitwise(fm, orc):
    """FMOE_F64 softmax_rows == the oracle's (glibc exp, matrix.cpp:155-170) bit
    for bit on 4M values spanning exp's whole domain: ordinary logits, rows
    whose spread reaches the rescaled |x| >= 512 path, subnormal and zero
    results (x - max down to -1500)."""
    rng = np.random.default_rng(5)
    rows, cols = 16384, 256
    a = rng.uniform(-1, 1, (rows, cols)) * rng.choice([1.0, 30.0, 600.0, 1500.0], size=(rows, 1))
    got = host(fm.softmax_rows(dev(a)))
    want = orc.softmax_rows(a)
    assert beq(got, want)


def test_gate_uniform_tie_break(fm):
    # test_gate.cpp:54-64: zero weights -> uniform scores, indices [0, 1]
    x = dev(np.random.default_rng(2).uniform(-1, 1, (5, 3)))
    out = fm.gate_forward(x, torch.zeros(3, 4, dtype=torch.float64, device="cuda"), 2)
    assert np.allclose(host(out.scores), 0.25)
    assert host(out.topk_indices).tolist() == [[0, 1]] * 5


@pytest.mark.parametrize("n,d,e,k", [(1000, 128, 64, 2), (3000, 256, 16, 1), (513, 64, 128, 2),
                                     (256, 128, 256, 1), (700, 64, 64, 9)])
def test_gate_bf16(fm, orc, n, d, e, k):
    rng = np.random.default_rng(n * 3 + e)
    x = bf16_round(rng.uniform(-1, 1, (n, d)))
    wg = bf16_round(rng.uniform(-0.1, 0.1, (d, e)))
    s_o, i_o, v_o = orc.gate_forward(x, wg, k)
    out = fm.gate_forward(dev(x, torch.bfloat16), dev(wg, torch.bfloat16), k)
    s = host(out.scores)
    assert np.abs(s - s_o).max() < 1e-5
    ok = well_separated_rows(s_o, k)
    assert ok.sum() >= min(100, n // 10)
    assert np.array_equal(host(out.topk_indices)[ok], i_o[ok])
    assert np.abs(host(out.topk_scores)[ok] - v_o[ok]).max() < 1e-5
    dt = rng.uniform(-1, 1, (n, k))
    gw_o, gx_o = orc.gate_backward(x, wg, s_o, i_o, dt)
    g = fm.gate_backward(dev(x, torch.bfloat16), dev(wg, torch.bfloat16),
                         fm.GateOutput(dev(s_o, torch.float32), dev(i_o, torch.int32), dev(v_o, torch.float32)),
                         dev(dt, torch.float32))
    assert rel_l2(host(g.d_wg), gw_o) < TOL_G_BF16
    assert rel_l2(host(g.d_x), gx_o) < TOL_G_BF16


# ---------------------------------------------------------------- experts
def _blocks(orc, rng, n, k, e):
    """Zipf-skewed distinct selections; the last expert stays empty (empty
    blocks are legal, SPEC.md dispatch design decisions)."""
    p = 1.0 / np.arange(1, e)
    p /= p.sum()
    return np.stack([rng.choice(e - 1, size=k, replace=False, p=p) for _ in range(n)]).astype(np.int64)


@pytest.mark.parametrize("n,k,e,d,h", [(40, 2, 4, 8, 12), (300, 2, 6, 32, 48), (97, 1, 3, 5, 7)])
def test_experts_f64_bit_exact(fm, orc, n, k, e, d, h):
    rng = np.random.default_rng(n + h)
    idx = _blocks(orc, rng, n, k, e)
    po = orc.build_plan(idx, e)
    p = fm.build_plan(dev(idx, torch.int32), e)
    w = orc.init_state(123, d, h, e)
    xs = rng.uniform(-1, 1, (n * k, d))
    d_ys = rng.uniform(-1, 1, (n * k, d))
    ex = fm.Experts(dev(w["w1"]), dev(w["b1"]), dev(w["w2"]), dev(w["b2"]))
    ys, hid = fm.multi_expert_forward(dev(xs), p, ex)
    d_xs, g = fm.multi_expert_backward(dev(d_ys), dev(xs), hid, p, ex)
    ys_h, dxs_h = host(ys), host(d_xs)
    for gi in range(e):
        a, c = po["offsets"][gi], po["counts"][gi]
        y_o, pre_o, hid_o = orc.expert_forward(xs[a:a + c], w["w1"][gi], w["b1"][gi], w["w2"][gi], w["b2"][gi])
        assert beq(ys_h[a:a + c], y_o)
        assert beq(host(hid)[a:a + c], hid_o)
        dx_o, go = orc.expert_backward(d_ys[a:a + c], xs[a:a + c], pre_o, hid_o, w["w1"][gi], w["w2"][gi])
        assert beq(dxs_h[a:a + c], dx_o)
        assert beq(host(g.d_w1[gi]), go["dw1"]) and beq(host(g.d_b1[gi]), go["db1"])
        assert beq(host(g.d_w2[gi]), go["dw2"]) and beq(host(g.d_b2[gi]), go["db2"])


@pytest.mark.parametrize("align", [128, 256])  # 128: one-CTA tiles; 256: CTA-pair (cta_group::2) tiles
@pytest.mark.parametrize("n,k,e,d,h", [(512, 2, 8, 128, 256), (3000, 2, 16, 64, 192), (1500, 1, 8, 256, 512),
                                       (700, 2, 4, 320, 448)])
def test_experts_bf16_vs_torch_fp32(fm, orc, n, k, e, d, h, align):
    """Grouped tcgen05 GEMM (fc1/fc2, dgrad, wgrad) vs a plain PyTorch fp32
    reference of the same op on the same bf16 values."""
    rng = np.random.default_rng(n + d)
    idx = _blocks(orc, rng, n, k, e)
    p = fm.build_plan(dev(idx, torch.int32), e, align=align)
    w1 = torch.randn(e, d, h, device="cuda").mul(0.05).bfloat16()
    w2 = torch.randn(e, h, d, device="cuda").mul(0.05).bfloat16()
    b1 = torch.randn(e, h, device="cuda").mul(0.1)
    b2 = torch.randn(e, d, device="cuda").mul(0.1)
    x = torch.randn(n, d, device="cuda").bfloat16()
    xs = fm.scatter(x, p)
    ex = fm.Experts(w1, b1, w2, b2)
    ys, hid = fm.multi_expert_forward(xs, p, ex)
    dy = torch.randn(n, d, device="cuda").bfloat16()
    d_ys_full, _ = fm.gather_combine_backward(dy, ys, p, torch.ones(n, k, device="cuda"))
    d_xs, g = fm.multi_expert_backward(d_ys_full, xs, hid, p, ex)
    torch.cuda.synchronize()
    off = host(p.offsets).astype(np.int64)
    cnt = host(p.counts).astype(np.int64)
    for gi in range(e):
        a, c = int(off[gi]), int(cnt[gi])
        xe = xs[a:a + c].float()
        pre = xe @ w1[gi].float() + b1[gi]
        he = torch.relu(pre)
        assert rel_l2(host(hid[a:a + c]), host(he)) < 1e-2
        ye = hid[a:a + c].float() @ w2[gi].float() + b2[gi]
        assert rel_l2(host(ys[a:a + c]), host(ye)) < 1e-2
        dye = d_ys_full[a:a + c].float()
        dh = (dye @ w2[gi].float().t()) * (hid[a:a + c].float() > 0)
        ref_dw2 = hid[a:a + c].float().t() @ dye
        ref_db2 = dye.sum(0)
        assert rel_l2(host(g.d_w2[gi]), host(ref_dw2)) < 1e-3 if c else (host(g.d_w2[gi]) == 0).all()
        assert rel_l2(host(g.d_b2[gi]), host(ref_db2)) < 1e-3 if c else (host(g.d_b2[gi]) == 0).all()
        dpre_bf = dh.bfloat16().float()
        ref_dw1 = xe.t() @ dpre_bf
        assert rel_l2(host(g.d_w1[gi]), host(ref_dw1)) < 1e-2 if c else (host(g.d_w1[gi]) == 0).all()
        ref_dx = dpre_bf @ w1[gi].float().t()
        assert rel_l2(host(d_xs[a:a + c]), host(ref_dx)) < 1e-2


# ------------------------------------------------------------------ layer
def _layer_io(orc, seed, n, d):
    return orc.seeded_matrix(seed, 102, n, d), orc.seeded_matrix(seed, 103, n, d)


@pytest.mark.parametrize("name", ["layer_a", "layer_b", "layer_c"])
def test_layer_f64_vs_golden(fm, orc, name):
    import os

    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", name + ".npz")))
    seed, n, d, h, e, k = (int(v) for v in g["meta"])
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, seed), dtype=torch.float64)
    w = orc.init_state(seed, d, h, e)
    assert beq(host(layer.w_g), w["wg"]) and beq(host(layer.experts.w1), w["w1"])
    x, dy = _layer_io(orc, seed, n, d)
    xt = dev(x)
    y = layer.forward(xt)
    dx = layer.backward(dev(dy))
    idx, vals, scores, _ = layer.routing()
    assert np.array_equal(host(idx), g["idx"])
    for got, key in ((y, "y"), (dx, "dx"), (layer.d_wg, "dwg"), (layer.grads.d_w1, "dw1"),
                     (layer.grads.d_b1, "db1"), (layer.grads.d_w2, "dw2"), (layer.grads.d_b2, "db2")):
        assert beq(host(got), g[key]), key  # bit-identical to the reference (glibc exp included)


# (16384, 128, 256, 8, 2): >= 1024 rows per expert -> 256-row blocks, CTA-pair GEMMs
@pytest.mark.parametrize("n,d,h,e,k", [(512, 128, 256, 16, 2), (4096, 256, 512, 32, 2), (1000, 64, 128, 8, 1),
                                       (16384, 128, 256, 8, 2)])
def test_layer_bf16_vs_oracle(fm, orc, n, d, h, e, k):
    seed = 42
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, seed), dtype=torch.bfloat16)
    x, dy = _layer_io(orc, seed, n, d)
    x, dy = bf16_round(x), bf16_round(dy)
    y = layer.forward(dev(x, torch.bfloat16))
    dx = layer.backward(dev(dy, torch.bfloat16))
    torch.cuda.synchronize()
    w = dict(wg=host(layer.w_g), w1=host(layer.experts.w1), b1=host(layer.experts.b1),
             w2=host(layer.experts.w2), b2=host(layer.experts.b2))
    o = orc.moe_forward_backward(x, dy, k, **w)
    idx = host(layer.routing()[0]).astype(np.int64)
    ok = well_separated_rows(o["scores"], k)
    assert np.array_equal(idx[ok], o["idx"][ok])
    same = (idx == o["idx"]).all(axis=1)
    assert same.mean() > 0.98
    assert rel_l2(host(y)[same], o["y"][same]) < TOL_Y_BF16
    assert rel_l2(host(dx)[same], o["dx"][same]) < TOL_G_BF16
    if same.all():
        for a, key in ((layer.d_wg, "dwg"), (layer.grads.d_w1, "dw1"), (layer.grads.d_b1, "db1"),
                       (layer.grads.d_w2, "dw2"), (layer.grads.d_b2, "db2")):
            assert rel_l2(host(a), o[key]) < TOL_G_BF16, key


def test_layer_bf16_deterministic(fm):
    """Run-to-run bitwise determinism (no atomics in any reduction)."""
    n, d, h, e, k = 2048, 128, 256, 16, 2
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 5), dtype=torch.bfloat16)
    x = torch.randn(n, d, device="cuda").bfloat16()
    dy = torch.randn(n, d, device="cuda").bfloat16()
    outs = []
    for _ in range(2):
        y = layer.forward(x).clone()
        dx = layer.backward(dy).clone()
        outs.append([y, dx, layer.d_wg.clone(), layer.grads.d_w1.clone(), layer.grads.d_b1.clone()])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_layer_step_host(fm):
    n, d, h, e, k = 1024, 128, 256, 16, 2
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 9), dtype=torch.bfloat16)
    x = torch.randn(n, d).bfloat16().pin_memory()
    dy = torch.randn(n, d).bfloat16().pin_memory()
    y = torch.empty(n, d, dtype=torch.bfloat16).pin_memory()
    dx = torch.empty(n, d, dtype=torch.bfloat16).pin_memory()
    layer.step_host(x, dy, y, dx)
    y2 = layer.forward(x.cuda())
    dx2 = layer.backward(dy.cuda())
    assert torch.equal(y, y2.cpu()) and torch.equal(dx, dx2.cpu())


def test_layer_step_host_async_pipeline(fm):
    """Back-to-back async host steps (uploads of step t+1 under the kernels of
    step t, two device buffer sets) give every step's eager results."""
    n, d, h, e, k = 1024, 128, 256, 16, 2
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 9), dtype=torch.bfloat16)
    steps = 5
    xs = [torch.randn(n, d).bfloat16().pin_memory() for _ in range(steps)]
    dys = [torch.randn(n, d).bfloat16().pin_memory() for _ in range(steps)]
    ys = [torch.empty(n, d, dtype=torch.bfloat16).pin_memory() for _ in range(steps)]
    dxs = [torch.empty(n, d, dtype=torch.bfloat16).pin_memory() for _ in range(steps)]
    for i in range(steps):
        layer.step_host_async(xs[i], dys[i], ys[i], dxs[i])
    layer.wait_host()
    for i in range(steps):
        y = layer.forward(xs[i].cuda())
        dx = layer.backward(dys[i].cuda())
        assert torch.equal(ys[i], y.cpu()) and torch.equal(dxs[i], dx.cpu()), i


def test_layer_shape_errors(fm):
    with pytest.raises(fm.ShapeError):
        fm.MoELayer(fm.MoEConfig(8, 64, 64, 3, 2, 1, 0), dtype=torch.float64)  # k > E
    with pytest.raises(fm.ShapeError):
        fm.MoELayer(fm.MoEConfig(8, 60, 64, 1, 8, 1, 0), dtype=torch.bfloat16)  # d % 64
    with pytest.raises(fm.ShapeError):
        fm.gate_forward(torch.zeros(4, 3, dtype=torch.float64, device="cuda"),
                        torch.zeros(4, 2, dtype=torch.float64, device="cuda"), 1)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_dense_primitives_compose_to_the_gate(fm, dtype):
    """matmul -> softmax_rows -> topk_rows reproduce gate_forward bit for bit
    (test_gate.cpp:66-82) and matmul is the reference's fma chain."""
    g = torch.Generator().manual_seed(11)
    x = (torch.rand(300, 70, generator=g, dtype=torch.float64) * 2 - 1).to(dtype).cuda()
    w = (torch.rand(70, 24, generator=g, dtype=torch.float64) * 0.2 - 0.1).to(dtype).cuda()
    out = fm.gate_forward(x, w, 3)
    logits = fm.matmul(x, w)
    s = fm.softmax_rows(logits)
    idx, val = fm.topk_rows(s, 3)
    assert torch.equal(out.scores, s)
    assert torch.equal(out.topk_indices, idx)
    assert torch.equal(out.topk_scores, val)
    if dtype == torch.float64:  # the reference's fma chain (oracle matmul, matrix.cpp:56-88)
        from oracle import orc

        assert np.array_equal(logits.cpu().numpy(), orc.matmul(x.cpu().numpy(), w.cpu().numpy()))
    with pytest.raises(fm.ShapeError):
        fm.topk_rows(s, 25)
    with pytest.raises(fm.ShapeError):
        fm.matmul(x, x)


# ----------------------------------------------- full-size properties (cfg2)
def test_permutes_full_size_round_trips(fm):
    """BASELINE cfg2 size (65536 tokens, d=1024, 64 experts, top-2, 256-row
    blocks): size-independent identities that hold bit for bit --
    scatter_backward(scatter(x)) == k*x and gather_combine(scatter(x), 1/k) == x
    (halving, doubling and the two-term sums are exact in fp32 and bf16)."""
    n, d, e, k = 65536, 1024, 64, 2
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    x = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    first = torch.randint(0, e, (n, 1), device="cuda", generator=g)
    step = torch.randint(1, e, (n, 1), device="cuda", generator=g)
    idx = torch.cat([first, (first + step) % e], dim=1)  # two distinct experts per token
    p = fm.build_plan(idx.int(), e, align=256)
    xs = fm.scatter(x, p)
    assert torch.equal(fm.scatter_backward(xs, p), x * 2)
    half = torch.full((n, k), 0.5, device="cuda")
    assert torch.equal(fm.gather_combine(xs, p, half), x)
    counts = p.counts.cpu().long()
    assert int(counts.sum()) == n * k and (host(p.offsets) % 256 == 0).all()


# --------------------------------------------------------- fp32 layer (§8c)
@pytest.mark.parametrize("n,d,h,e,k,seed", [(512, 64, 128, 8, 2, 21),      # 128-row blocks, single CTAs
                                             (4096, 128, 320, 8, 2, 22),   # 256-row blocks, CTA pairs, h % 256 != 0
                                             (1000, 192, 256, 16, 3, 23)])  # ragged experts, k = 3
def test_layer_f32_vs_oracle(fm, orc, n, d, h, e, k, seed):
    """FMOE_F32 against the oracle fed the same fp32 values: outputs
    max-abs-err <= 1e-5 * max|ref|, gradients rel-L2 <= 1e-4 (SURVEY §8c
    parity protocol (3)), routing exact on well-separated tokens.  The expert
    GEMMs run on the tensor cores (bf16x3 split products, f32x.cu) over
    aligned expert blocks; the gate stays on the SIMT fp32 kernels."""
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, seed), dtype=torch.float32)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    x = f32(orc.seeded_matrix(seed, 102, n, d))
    dy = f32(orc.seeded_matrix(seed, 103, n, d))
    y = layer.forward(dev(x, torch.float32))
    dx = layer.backward(dev(dy, torch.float32))
    torch.cuda.synchronize()
    w = dict(wg=host(layer.w_g), w1=host(layer.experts.w1), b1=host(layer.experts.b1), w2=host(layer.experts.w2),
             b2=host(layer.experts.b2))
    o = orc.moe_forward_backward(x, dy, k, **w)
    idx = host(layer.routing()[0]).astype(np.int64)
    ok = well_separated_rows(o["scores"], k)
    assert np.array_equal(idx[ok], o["idx"][ok])
    same = (idx == o["idx"]).all(axis=1)
    assert same.all()
    assert np.abs(host(y) - o["y"]).max() <= 1e-5 * np.abs(o["y"]).max()
    assert rel_l2(host(dx), o["dx"]) <= 1e-4
    for a, key in ((layer.d_wg, "dwg"), (layer.grads.d_w1, "dw1"), (layer.grads.d_b1, "db1"),
                   (layer.grads.d_w2, "dw2"), (layer.grads.d_b2, "db2")):
        assert rel_l2(host(a), o[key]) <= 1e-4, key
