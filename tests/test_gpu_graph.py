"""The single-GPU bf16 layer step has no host synchronisation and no
allocation, so a whole forward+backward captures into one CUDA graph
(torch.cuda.graph around the C-ABI calls) and replays bit-identically to the
eager step -- the launch-free way to drive it from a training loop."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_layer_step_graph_replay_is_bitwise_eager():
    import paper_2103_13262_b200 as fm

    n, d, h, e, k = 4096, 256, 512, 16, 2
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 3), dtype=torch.bfloat16)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, d, device="cuda", generator=g).bfloat16()
    dy = torch.randn(n, d, device="cuda", generator=g).bfloat16()
    y, dx = torch.empty_like(x), torch.empty_like(x)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up (kernel attributes, lazy setup) outside the capture
        layer.forward(x, y)
        layer.backward(dy, dx)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        layer.forward(x, y)
        layer.backward(dy, dx)
    eager_y, eager_dx = layer.forward(x).clone(), layer.backward(dy).clone()
    eager_dw1 = layer.grads.d_w1.clone()
    y.zero_()
    dx.zero_()
    layer.grads.d_w1.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, eager_y) and torch.equal(dx, eager_dx)
    assert torch.equal(layer.grads.d_w1, eager_dw1)
    # new inputs in the captured buffers flow through the replay
    x.copy_(torch.randn(n, d, device="cuda", generator=g).bfloat16())
    graph.replay()
    ref_y = layer.forward(x.clone()).clone()
    torch.cuda.synchronize()
    assert torch.equal(y, ref_y)
