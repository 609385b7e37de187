"""Edge cases of the bf16 product path against the oracle (empty
and ragged inputs, extreme routing parameters): n_b = 0 and 1, batches that
are not multiples of a GEMM tile, k = E (every expert selected), the smallest
dims, E > 256 (the logits-then-softmax gate path), k up to 8."""
import numpy as np
import pytest
import torch

from tests.gpu_util import bf16_round, dev, host, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fm():
    import paper_2103_13262_b200 as m

    return m


def _run(fm, orc, n, d, h, e, k, seed=7, check_grads=True):
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, seed), dtype=torch.bfloat16)
    x = bf16_round(orc.seeded_matrix(seed, 102, max(n, 1), d))[:n]
    dy = bf16_round(orc.seeded_matrix(seed, 103, max(n, 1), d))[:n]
    y = layer.forward(dev(x, torch.bfloat16))
    dx = layer.backward(dev(dy, torch.bfloat16))
    torch.cuda.synchronize()
    assert y.shape == (n, d) and dx.shape == (n, d)
    if n == 0:
        return layer, None, None, None
    w = dict(wg=host(layer.w_g), w1=host(layer.experts.w1), b1=host(layer.experts.b1), w2=host(layer.experts.w2),
             b2=host(layer.experts.b2))
    o = orc.moe_forward_backward(x, dy, k, **w)
    idx = host(layer.routing()[0]).astype(np.int64)
    same = (np.sort(idx, 1) == np.sort(o["idx"], 1)).all(axis=1) if k == e else (idx == o["idx"]).all(axis=1)
    assert same.mean() > 0.9
    assert rel_l2(host(y)[same], o["y"][same]) < 1e-2
    assert rel_l2(host(dx)[same], o["dx"][same]) < 2e-2
    if check_grads and same.all():
        for a, key in ((layer.grads.d_w1, "dw1"), (layer.grads.d_b2, "db2")):
            assert rel_l2(host(a), o[key]) < 2e-2, key
    return layer, y, dx, o


def test_empty_batch(fm, orc):
    layer, *_ = _run(fm, orc, 0, 64, 64, 8, 2)
    assert not host(layer.grads.d_w1).any() and not host(layer.d_wg).any()


@pytest.mark.parametrize("n", [1, 3, 129, 1000])
def test_ragged_batches(fm, orc, n):
    _run(fm, orc, n, 64, 128, 8, 2)


def test_every_expert_selected(fm, orc):
    _run(fm, orc, 300, 64, 64, 8, 8)


def test_top8_of_64(fm, orc):
    _run(fm, orc, 512, 128, 128, 64, 8)


def test_more_than_256_experts(fm, orc):
    _run(fm, orc, 2048, 64, 64, 512, 2, check_grads=False)


@pytest.mark.parametrize("dtype,e,k", [(torch.bfloat16, 16, 2), (torch.bfloat16, 64, 3), (torch.bfloat16, 128, 2),
                                       (torch.bfloat16, 512, 2), (torch.float64, 16, 2), (torch.float32, 16, 3)])
def test_nan_token_row_routes_like_the_reference(fm, orc, dtype, e, k):
    """A NaN in one token makes that row's softmax all-NaN; the reference's
    stable sort then keeps column order (matrix.cpp:172-189), so the row picks
    experts 0..k-1 with NaN scores.  Every index stays in [0, E), the NaN stays
    in its own row, and the other rows equal a run where that row is finite."""
    n, d, h, seed, bad = 300, 64, 64, 11, 5
    x = bf16_round(orc.seeded_matrix(seed, 102, n, d))
    dy = bf16_round(orc.seeded_matrix(seed, 103, n, d))
    xn = x.copy()
    xn[bad, 7] = np.nan
    outs = []
    for xi in (xn, x):
        layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, seed), dtype=dtype)
        y = layer.forward(dev(xi, dtype))
        dx = layer.backward(dev(dy, dtype))
        torch.cuda.synchronize()
        outs.append((host(layer.routing()[0]).astype(np.int64), host(y), host(dx)))
    (idx, y, dx), (idx0, y0, dx0) = outs
    assert ((idx >= 0) & (idx < e)).all()
    assert (idx[bad] == np.arange(k)).all()
    assert np.isnan(y[bad]).all()
    keep = np.ones(n, bool)
    keep[bad] = False
    assert (idx[keep] == idx0[keep]).all()
    assert np.array_equal(y[keep], y0[keep])
    assert np.isfinite(y[keep]).all()
