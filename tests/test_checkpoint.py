"""Weight checkpoints in the reference's format (FMOE-CKPT v1,
checkpoint.hpp:10-16, checkpoint.cpp:63-122).

CPU: the library's header reader on files written by the reference itself,
and its error behaviour (ProtocolError on missing / malformed files, as
test_moe_layer.cpp:325-331).  GPU: reference file -> device layer (f64 bit for
bit, bf16 rounded once), device layer -> file -> reference loader bit for bit,
an expert-parallel rank loads its slice, and the shape / world checks.
"""
import os

import numpy as np
import pytest
import torch


@pytest.fixture(scope="module")
def fm():
    import paper_2103_13262_b200 as m

    return m


def test_header_of_reference_file(fm, ref, tmp_path):
    w = ref.init_state(9, 16, 24, 6, 2)
    path = str(tmp_path / "ref.ckpt")
    ref.save_checkpoint(path, w, n_b=33, k=2, n_e_local=3, world=2, seed=9)
    info = fm.checkpoint_info(path)
    assert info == dict(n_b=33, d_m=16, d_h=24, k=2, n_e_local=3, world_size=2, experts_total=6, seed=9)
    assert os.path.getsize(path) == 10 + 4 + 8 * 8 + (16 + 16 * 6 * 8) + 6 * 4 * 16 + 6 * 8 * (2 * 16 * 24 + 24 + 16)


def test_bad_files_raise_protocol_error(fm, tmp_path):
    with pytest.raises(fm.ProtocolError):
        fm.checkpoint_info(str(tmp_path / "missing.ckpt"))
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"NOT-A-CKPT" + b"\0" * 64)
    with pytest.raises(fm.ProtocolError):
        fm.checkpoint_info(str(bad))


def _weights(layer):
    f = lambda t: t.detach().cpu().double().numpy()  # noqa: E731
    return dict(wg=f(layer.w_g), w1=f(layer.experts.w1), b1=f(layer.experts.b1), w2=f(layer.experts.w2),
                b2=f(layer.experts.b2))


@pytest.mark.gpu
def test_reference_file_into_device_layer(fm, ref, orc, tmp_path):
    d, h, e, k, seed = 64, 128, 8, 2, 17  # bf16 layers need multiples of 64
    w = orc.init_state(seed, d, h, e)
    w = {key: v + 0.25 for key, v in w.items()}  # not what init_weights would produce
    path = str(tmp_path / "w.ckpt")
    ref.save_checkpoint(path, w, n_b=64, k=k, seed=seed)
    f64 = fm.MoELayer(fm.MoEConfig(64, d, h, k, e, 1, 0), dtype=torch.float64)
    f64.load_checkpoint(path)
    got = _weights(f64)
    for key in w:
        assert got[key].tobytes() == w[key].tobytes(), key
    bf = fm.MoELayer(fm.MoEConfig(64, d, h, k, e, 1, 0), dtype=torch.bfloat16)
    bf.load_checkpoint(path)
    got = _weights(bf)
    rb = lambda a: torch.as_tensor(a).float().bfloat16().double().numpy()  # noqa: E731
    for key in ("wg", "w1", "w2"):
        assert np.array_equal(got[key], rb(w[key])), key
    for key in ("b1", "b2"):  # fp32 biases on the product path
        assert np.array_equal(got[key], w[key].astype(np.float32).astype(np.float64)), key


@pytest.mark.gpu
def test_device_layer_into_reference_loader(fm, ref, tmp_path):
    n, d, h, e, k = 128, 32, 48, 8, 2
    layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 5), dtype=torch.float64)
    x = torch.rand(n, d, dtype=torch.float64, device="cuda")
    layer.train_step(x, torch.rand_like(x), 0.05)  # weights no longer init_state's
    path = str(tmp_path / "dev.ckpt")
    layer.save_checkpoint(path)
    hdr, w = ref.load_checkpoint(path)
    assert hdr == dict(n_b=n, d_m=d, d_h=h, k=k, n_e_local=e, world_size=1, seed=5)
    got = _weights(layer)
    for key in w:
        assert got[key].tobytes() == w[key].tobytes(), key
    # and back into a fresh layer
    other = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 99), dtype=torch.float64)
    other.load_checkpoint(path)
    for key, v in _weights(other).items():
        assert v.tobytes() == got[key].tobytes(), key


@pytest.mark.gpu
def test_expert_parallel_rank_loads_its_slice(fm, orc, ref, tmp_path):
    d, h, el, world, k = 16, 32, 2, 4, 2
    w = orc.init_state(3, d, h, el * world)
    path = str(tmp_path / "ep.ckpt")
    ref.save_checkpoint(path, w, n_b=8, k=k, seed=3)
    for r in range(world):
        layer = fm.MoELayer(fm.MoEConfig(8, d, h, k, el, world, 3), rank=r, dtype=torch.float64)
        layer.load_checkpoint(path)
        got = _weights(layer)
        assert got["wg"].tobytes() == w["wg"].tobytes()
        for key in ("w1", "b1", "w2", "b2"):
            assert got[key].tobytes() == w[key][r * el:(r + 1) * el].tobytes(), key
        with pytest.raises(fm.ShapeError):  # an EP rank holds only its slice
            layer.save_checkpoint(str(tmp_path / "no.ckpt"))


@pytest.mark.gpu
def test_shape_mismatch(fm, orc, ref, tmp_path):
    w = orc.init_state(3, 16, 32, 4)
    path = str(tmp_path / "s.ckpt")
    ref.save_checkpoint(path, w)
    layer = fm.MoELayer(fm.MoEConfig(8, 16, 64, 1, 4, 1, 3), dtype=torch.float64)
    with pytest.raises(fm.ShapeError):
        layer.load_checkpoint(path)
    with pytest.raises(fm.ProtocolError):
        layer.load_checkpoint(str(tmp_path / "missing.ckpt"))


@pytest.mark.gpu
def test_truncated_file_fails_on_every_rank(fm, orc, ref, tmp_path):
    """A rank whose own experts precede the cut still rejects the file, as the
    reference loader does (the skipped experts are checked against the length)."""
    d, h, el, world, k = 16, 32, 2, 2, 2
    w = orc.init_state(3, d, h, el * world)
    path = tmp_path / "full.ckpt"
    ref.save_checkpoint(str(path), w, n_b=8, k=k, seed=3)
    cut = tmp_path / "cut.ckpt"
    cut.write_bytes(path.read_bytes()[:-8 * (h * d)])  # the last expert's w2 is short
    for r in range(world):
        layer = fm.MoELayer(fm.MoEConfig(8, d, h, k, el, world, 3), rank=r, dtype=torch.float64)
        with pytest.raises(fm.ProtocolError):
            layer.load_checkpoint(str(cut))


@pytest.mark.gpu
def test_bf16_training_resumes_from_fp32_masters(fm, tmp_path):
    """bf16 training updates fp32 masters; a checkpoint keeps them, so a run
    resumed from the file continues bit for bit like the uninterrupted one."""
    n, d, h, e, k, lr = 256, 64, 128, 8, 2, 0.05
    g = torch.Generator().manual_seed(4)
    xs = [torch.rand(n, d, generator=g).bfloat16().cuda() for _ in range(5)]
    ts = [torch.rand(n, d, generator=g).bfloat16().cuda() for _ in range(5)]
    a = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 21), dtype=torch.bfloat16)
    for i in range(3):
        a.train_step(xs[i], ts[i], lr)
    path = str(tmp_path / "bf.ckpt")
    a.save_checkpoint(path)
    b = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 0), dtype=torch.bfloat16)
    b.load_checkpoint(path)
    for i in range(3, 5):
        la, lb = a.train_step(xs[i], ts[i], lr), b.train_step(xs[i], ts[i], lr)
        assert la == lb
    for key, v in _weights(a).items():
        assert v.tobytes() == _weights(b)[key].tobytes(), key
