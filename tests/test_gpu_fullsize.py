"""BASELINE-size checks of the bf16 product path (full sizes
through size-independent properties, fp32 recomputation on samples):

* cfg2 (65536 tokens, d=1024, h=4096, 64 experts, top-2) and cfg3's per-GPU
  layer shape (16384 tokens, d=2048, h=8192, 8 experts):
  - gate routing on a token sample equals the fp64 oracle gate on
    well-separated rows, scores within bf16-input tolerance;
  - outputs y, d(topk_scores) and d_x (expert path + the gate's softmax
    Jacobian and d_x, gate.cpp:44-63) on a token sample, recomputed per token
    in fp32 from the GPU's routing;
  - dW1, dW2, d_b1 of four experts (first, last, heaviest, lightest) against
    fp32 recomputation over ALL of each expert's rows (expert.cpp:41-55);
  - d_b2 of every expert, and the full d x E gate gradient d_wg against
    x^T dz over every token (gate.cpp:52-62);
  - one bf16 train_step: SGD on the fp32 masters applied bit for bit to the
    GPU's gradients, and those gradients within tolerance of the fp32
    recomputation driven by the MSE d_y (moe_layer.cpp:144-205).
Tolerances are SURVEY §8c's bf16 rule: outputs rel-L2 <= 1e-2, gradients
<= 2e-2.
"""
import numpy as np
import pytest
import torch

from tests.gpu_util import beq, dev, host, rel_l2, well_separated_rows

pytestmark = pytest.mark.gpu

Y_TOL, G_TOL = 1e-2, 2e-2


@pytest.fixture(scope="module")
def fm():
    import paper_2103_13262_b200 as m

    return m


def _bf(t):
    """Round to bf16 as the GPU stores the tensor, back to fp32."""
    return t.bfloat16().float()


def _inputs(n, d, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    dy = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    return x, dy


def _sample_refs(layer, x, dy, rows):
    """Per-token fp32 recomputation on `rows` from the GPU's routing: y,
    d(topk_scores) and d_x including the gate path.  Pairs are grouped by
    expert so each expert's weights are widened once."""
    idx, vals, scores, _ = layer.routing()
    k = idx.shape[1]
    w1, b1, w2, b2 = layer.experts.w1, layer.experts.b1, layer.experts.w2, layer.experts.b2
    R, d = len(rows), x.shape[1]
    xr, dyr = x[rows].float(), dy[rows].float()
    ir, vr = idx[rows].long(), vals[rows].float()
    y_ref = torch.zeros(R, d, device="cuda")
    dw_ref = torch.zeros(R, k, device="cuda")
    dxs_sum = torch.zeros(R, d, device="cuda")
    for e in torch.unique(ir).tolist():
        ri, sj = (ir == e).nonzero(as_tuple=True)
        W1, W2 = w1[e].float(), w2[e].float()
        hid = _bf(torch.relu(xr[ri] @ W1 + b1[e].float()))
        ys = _bf(hid @ W2 + b2[e].float())
        wv = vr[ri, sj].unsqueeze(1)
        y_ref.index_add_(0, ri, wv * ys)
        dw_ref[ri, sj] = (dyr[ri] * ys).sum(1)
        dys = _bf(wv * dyr[ri])
        dpre = _bf((dys @ W2.t()) * (hid > 0))
        dxs_sum.index_add_(0, ri, _bf(dpre @ W1.t()))
    # gate: ds = d_w scattered into the selected columns, dz = s (ds - <ds, s>),
    # d_x += dz Wg^T (dz rounded to bf16 as the GPU's tensor-core operand)
    s = scores[rows].float()
    ds = torch.zeros_like(s).scatter_add_(1, ir, dw_ref)
    dz = s * (ds - (ds * s).sum(1, keepdim=True))
    dx_ref = dxs_sum + _bf(dz) @ layer.w_g.float().t()
    return y_ref, dw_ref, dx_ref


def _expert_grad_refs(layer, x, dy, experts):
    """dW1, dW2, d_b1 of `experts` in fp32 over every row routed to them."""
    idx, vals, _, _ = layer.routing()
    w1, b1, w2 = layer.experts.w1, layer.experts.b1, layer.experts.w2
    out = {}
    for e in experts:
        ti, sj = (idx.long() == e).nonzero(as_tuple=True)
        X = x[ti].float()
        hid = _bf(torch.relu(X @ w1[e].float() + b1[e].float()))
        dys = _bf(vals[ti, sj].float().unsqueeze(1) * dy[ti].float())
        dpre = _bf((dys @ w2[e].float().t()) * (hid > 0))
        out[e] = dict(dw2=hid.t() @ dys, dw1=X.t() @ dpre, db1=dpre.sum(0), rows=len(ti))
    return out


def _gate_dwg_ref(layer, x):
    """d_wg = x^T dz over every token, dz from the GPU's scores and d_w."""
    idx, _, scores, _ = layer.routing()
    s = scores.float()
    ds = torch.zeros_like(s).scatter_add_(1, idx.long(), layer.routing_grad().float())
    dz = s * (ds - (ds * s).sum(1, keepdim=True))
    return x.float().t() @ dz


def _check_grads(fm, orc, layer, x, dy, seed, sample):
    n, d = x.shape
    e = layer.config.total_experts()
    k = layer.config.k
    idx, vals, scores, _ = layer.routing()
    rng = np.random.default_rng(seed)
    rows = torch.as_tensor(np.sort(rng.choice(n, sample, replace=False)), device="cuda")
    # gate on the sample: fp64 oracle on the same bf16 inputs / weights
    s_o, i_o, _ = orc.gate_forward(host(x[rows]), host(layer.w_g), k)
    ok = well_separated_rows(s_o, k)
    assert ok.mean() > 0.5
    assert np.array_equal(host(idx[rows]).astype(np.int64)[ok], i_o[ok])
    assert rel_l2(host(scores[rows]), s_o) < Y_TOL
    # d_b2[e] = sum over slots routed to e of w * dy (expert.cpp:43-45), every token
    dys = _bf(vals.unsqueeze(-1) * dy.float().unsqueeze(1))  # [n, k, d]
    db2 = torch.zeros(e, d, device="cuda").index_add_(0, idx.reshape(-1).long(), dys.reshape(-1, d))
    assert rel_l2(host(layer.grads.d_b2), host(db2)) < G_TOL
    del dys, db2
    # first, last, heaviest, lightest expert: weight gradients over all their rows
    counts = torch.bincount(idx.reshape(-1).long(), minlength=e)
    pick = sorted({0, e - 1, int(counts.argmax()), int(counts.argmin())})
    for ex, r in _expert_grad_refs(layer, x, dy, pick).items():
        assert r["rows"] == int(counts[ex])
        for key, got in (("dw2", layer.grads.d_w2[ex]), ("dw1", layer.grads.d_w1[ex]), ("db1", layer.grads.d_b1[ex])):
            err = rel_l2(host(got), host(r[key]))
            assert err < G_TOL, (ex, key, err)
    # the whole gate gradient
    assert rel_l2(host(layer.d_wg), host(_gate_dwg_ref(layer, x))) < G_TOL
    return rows


def _check_layer(fm, orc, n, d, h, e, k, seed, sample=256):
    torch.cuda.empty_cache()
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, seed), dtype=torch.bfloat16)
    x, dy = _inputs(n, d, seed)
    y = layer.forward(x)
    dx = layer.backward(dy)
    torch.cuda.synchronize()
    rows = _check_grads(fm, orc, layer, x, dy, seed, sample)
    y_ref, dw_ref, dx_ref = _sample_refs(layer, x, dy, rows)
    assert rel_l2(host(y[rows]), host(y_ref)) < Y_TOL
    assert rel_l2(host(layer.routing_grad()[rows]), host(dw_ref)) < G_TOL
    assert rel_l2(host(dx[rows]), host(dx_ref)) < G_TOL
    assert torch.isfinite(dx).all()
    return layer


def test_cfg2_full_size(fm, orc):
    _check_layer(fm, orc, 65536, 1024, 4096, 64, 2, seed=21)


def test_cfg3_layer_shape(fm, orc):
    _check_layer(fm, orc, 16384, 2048, 8192, 8, 2, seed=22, sample=128)


def test_cfg2_train_step(fm, orc):
    """One bf16 train_step at cfg2: d_y = 2 (y - t) / numel (moe_layer.cpp:
    153-158); the parameters after the step are the SGD update of the fp32
    masters (widened from the bf16 weights) by the step's own gradients, bit
    for bit (param_sync.cpp:63-66); the gradients match fp32 recomputation."""
    n, d, h, e, k, seed, lr = 65536, 1024, 4096, 64, 2, 23, 1000.0  # large enough to move bf16 weights
    torch.cuda.empty_cache()
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, seed), dtype=torch.bfloat16)
    x, t = _inputs(n, d, seed)
    y = layer.forward(x).clone()
    before = dict(wg=layer.w_g.clone(), w1=layer.experts.w1.clone(), w2=layer.experts.w2.clone(),
                  b1=layer.experts.b1.clone(), b2=layer.experts.b2.clone())
    loss = layer.train_step(x, t, lr)
    torch.cuda.synchronize()
    diff = y.float() - t.float()
    assert abs(loss - float((diff.double() ** 2).mean())) <= 1e-6 * abs(loss)
    dy = (2.0 * diff / (n * d)).bfloat16()
    g = layer.grads

    def sgd(param, grad):  # fmaf(-lr, g, p) (exact product, one rounding), emulated in fp64
        return (param.double() + (-lr) * grad.double()).float()

    for key, got, grad in (("wg", layer.w_g, layer.d_wg), ("w1", layer.experts.w1, g.d_w1),
                           ("w2", layer.experts.w2, g.d_w2), ("b1", layer.experts.b1, g.d_b1),
                           ("b2", layer.experts.b2, g.d_b2)):
        want = sgd(before[key], grad).to(got.dtype)  # bf16 weights: RN of the fp32 master
        # fp64-then-fp32 can differ from one fp32 rounding only on an exact tie
        assert (got != want).float().mean().item() < 1e-5, key
        assert not torch.equal(got, before[key]), key  # the step moved the parameter group
    # the step's gradients, recomputed from d_y in fp32 (weights before the step)
    ref = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, seed), dtype=torch.bfloat16)
    ref.forward(x)
    ref.backward(dy)
    torch.cuda.synchronize()
    for a, b in ((ref.d_wg, layer.d_wg), (ref.grads.d_w1, g.d_w1), (ref.grads.d_w2, g.d_w2)):
        assert torch.equal(a, b)  # the step's backward is the layer's backward
    _check_grads(fm, orc, ref, x, dy, seed, 128)


def test_cfg5_full_size(fm, orc):
    """cfg5 at its BASELINE size: 262144 tokens, 256 experts, top-1, d=1024,
    h=4096, Zipf s=1.  Plan bit-exact; outputs and data gradients on a token
    sample; bias gradients through per-expert sums; dW1 / dW2 of the hot
    expert (16 % of the tokens) and of a tail expert over all their rows."""
    from paper_2103_13262_b200.workloads import zipf_routing

    n, d, h, e, k = 262144, 1024, 4096, 256, 1
    torch.cuda.empty_cache()
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 42), dtype=torch.bfloat16)
    idx, sc = zipf_routing(n, e, k, 1.0, seed=7)
    x, dy = _inputs(n, d, 7)
    it, st = dev(idx, torch.int32), dev(sc, torch.float32)
    y = layer.forward_routed(x, it, st)
    dx = layer.backward(dy)
    torch.cuda.synchronize()
    # plan: bit-exact against the oracle's build_plan on the same IndexMatrix
    want = orc.build_plan(idx.astype(np.int64), e)
    _, _, _, plan = layer.routing()
    counts = host(fm.api._wrap(plan.counts, (e,), torch.int32, x.device, layer)).astype(np.int64)
    assert beq(counts, want["counts"])
    assert counts[0] > 0.15 * n  # the skew is real: ~16% of tokens on expert 0
    # token sample: y_i = w_i * expert_{e_i}(x_i); dx_i = ((w_i dy_i) W2^T * mask) W1^T
    rng = np.random.default_rng(0)
    rows = torch.as_tensor(np.sort(rng.choice(n, 512, replace=False)), device="cuda")
    y_ref, dw_ref, _ = _sample_refs(layer, x, dy, rows)
    assert rel_l2(host(y[rows]), host(y_ref)) < Y_TOL
    assert rel_l2(host(layer.routing_grad()[rows]), host(dw_ref)) < G_TOL
    # injected routing: d_x is scatter_backward alone (no gate)
    w1, w2, b1 = layer.experts.w1, layer.experts.w2, layer.experts.b1
    dx_ref = torch.zeros(len(rows), d, device="cuda")
    ir = it[rows, 0].long()
    for ex in torch.unique(ir).tolist():
        ri = (ir == ex).nonzero(as_tuple=True)[0]
        hid = _bf(torch.relu(x[rows[ri]].float() @ w1[ex].float() + b1[ex].float()))
        dys = _bf(st[rows[ri], 0:1] * dy[rows[ri]].float())
        dpre = _bf((dys @ w2[ex].float().t()) * (hid > 0))
        dx_ref[ri] = dpre @ w1[ex].float().t()
    assert rel_l2(host(dx[rows]), host(dx_ref)) < G_TOL
    # d_b2[e] = sum over e's tokens of w_i * dy_i (expert.cpp:43-45)
    dys_all = _bf(st * dy.float())
    db2 = torch.zeros(e, d, device="cuda").index_add_(0, it[:, 0].long(), dys_all)
    assert rel_l2(host(layer.grads.d_b2), host(db2)) < G_TOL
    del dys_all, db2
    # weight gradients of the hot expert and a tail expert over all their rows
    for ex, r in _expert_grad_refs(layer, x, dy, [0, 200]).items():
        for key, got in (("dw2", layer.grads.d_w2[ex]), ("dw1", layer.grads.d_w1[ex]), ("db1", layer.grads.d_b1[ex])):
            err = rel_l2(host(got), host(r[key]))
            assert err < G_TOL, (ex, key, err)
