"""The reference's own C++ unit tests, compiled unchanged against the B200
drop-in (include/fmoe/*.hpp + libfmoe_dropin.so over the C-ABI).

tests/dropin/Makefile builds proj/tests/test_{tensor,gate,dispatch,expert,
moe_layer,comm,param_sync}.cpp from the reference checkout with a minimal doctest stand-in
(tests/dropin/doctest.h); the binaries travel to the GPU box with the
snapshot.  Every operator they call runs on the GPU in the FMOE_F64 parity mode.

Every test case runs (the checkpoint round trip included: the drop-in reads
and writes the reference's file format).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "dropin", "_bin")
LIB = os.path.join(ROOT, "paper_2103_13262_b200", "libfmoe_dropin.so")
SUITES = ["test_tensor", "test_gate", "test_dispatch", "test_expert", "test_moe_layer", "test_comm",
          "test_param_sync"]
# test_comm.cpp's wire-codec and TCP cases (lines 17-86, 297-395) exercise the
# reference's framed-byte transport, which the B200 drop-in does not have (rows
# move over NCCL / device copies; SURVEY §2, §8 put the codec and TCP out of
# scope).  They are skipped on both libraries; every exchange_counts,
# all_to_all_rows(_reverse) and allreduce_sum case runs.
EXCLUDE = {"test_comm": ["frame encoding", "frame decoding", "row payloads survive the wire",
                         "detects shape mismatch", "tcp transport", "tcp rendezvous", "hostfile parsing"]}


def test_dropin_library_exports_reference_api():
    assert os.path.exists(LIB), "build() did not produce libfmoe_dropin.so"
    syms = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    for name in ["fmoe::gate_forward(", "fmoe::gate_backward(", "fmoe::build_plan(", "fmoe::scatter(",
                 "fmoe::gather_combine(", "fmoe::scatter_backward(", "fmoe::gather_combine_backward(",
                 "fmoe::multi_expert_forward(", "fmoe::multi_expert_backward(", "fmoe::expert_forward(",
                 "fmoe::expert_backward(", "fmoe::forward(", "fmoe::backward(", "fmoe::naive_forward(",
                 "fmoe::init_state(", "fmoe::train_step(", "fmoe::exchange_counts(", "fmoe::all_to_all_rows(",
                 "fmoe::all_to_all_rows_reverse(", "fmoe::allreduce_sum(", "fmoe::matmul(", "fmoe::softmax_rows(",
                 "fmoe::topk_rows(", "fmoe::InProcWorld::transport("]:
        assert name in syms, name
    # the drop-in computes through the product library, never the checker
    deps = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "libfmoe_b200.so" in deps and "orc" not in deps and "fmoe_ref" not in deps


def _run(exe, exclude):
    args = [exe] + (["--exclude=" + ",".join(exclude)] if exclude else [])
    r = subprocess.run(args, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    failed_cases = sorted(line.split("] ", 1)[1].split(" (")[0] for line in r.stdout.splitlines()
                          if line.startswith("[ FAIL ]"))
    failed_checks = sorted(line.split(": FAILED")[0].rsplit("/", 1)[-1] for line in out.splitlines()
                           if ": FAILED" in line)
    summary = [line for line in r.stdout.splitlines() if line.startswith("test cases:")]
    return r.returncode, failed_cases, failed_checks, summary, out


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_tests_pass_on_dropin(suite):
    """The drop-in passes exactly what the reference library passes on the same
    test source: identical failing assertions (the reference itself fails
    test_tensor.cpp:42,51,56 -- its naive loop is unfused, its matmul fused)."""
    exe, ref = os.path.join(BIN, suite), os.path.join(BIN, "ref_" + suite)
    if not os.path.exists(exe) or not os.path.exists(ref):
        pytest.skip("reference unit tests were not compiled (build() needs the reference checkout)")
    ex = EXCLUDE.get(suite, [])
    rc, cases, checks, summary, out = _run(exe, ex)
    rrc, rcases, rchecks, rsummary, rout = _run(ref, ex)
    print("drop-in  :", summary, cases, checks)
    print("reference:", rsummary, rcases, rchecks)
    assert summary, out[-3000:]
    assert (cases, checks) == (rcases, rchecks), out[-3000:]
    assert rc == rrc
    if suite not in ("test_tensor", "test_comm"):  # the reference fails test_tensor.cpp:42,51,56, test_comm.cpp:119
        assert rc == 0 and "0 failed" in summary[0], out[-3000:]


def _fast_route_dump(tmp_path, tag, env, shape=("512", "128", "256", "8")):
    """Sections of fast_route's dump: y, scores, top-k scores, expert outputs,
    the E expert caches (input, preact, hidden), d_x, d_wg, the E expert
    gradients (d_w1, d_b1, d_w2, d_b2), the edited-cache d_x and d_wg, three
    losses, the parameters after training, and the last forward."""
    import numpy as np

    exe = os.path.join(BIN, "fast_route")
    if not os.path.exists(exe):
        pytest.skip("fast_route was not compiled (build() needs the reference checkout for tests/dropin)")
    out = str(tmp_path / f"{tag}.bin")
    r = subprocess.run([exe, out, *shape], capture_output=True, text=True, timeout=600,
                       env={**os.environ, **env})
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
    raw = np.fromfile(out, dtype=np.float64)
    secs, i = [], 0
    while i < raw.size:
        n = int(raw[i])
        secs.append(raw[i + 1:i + 1 + n])
        i += 1 + n
    return raw, secs


@pytest.mark.gpu
def test_dropin_device_route_is_the_composition_bitwise(tmp_path):
    """fmoe::forward / backward / train_step on the device-resident route
    (one device layer, results left on the GPU until read; dropin/fast.cpp)
    produce byte-identical values to the operator composition
    (FMOE_DROPIN_PATH=ops): y, the whole forward cache, d_x, every gradient,
    a backward over an edited copy of the cache (the route must fall back),
    three train_step losses and the parameters they leave, and a forward from
    those device-resident parameters (moe_layer.cpp:67-205)."""
    fast, _ = _fast_route_dump(tmp_path, "fast", {})
    ops, _ = _fast_route_dump(tmp_path, "ops", {"FMOE_DROPIN_PATH": "ops"})
    assert fast.shape == ops.shape and fast.size > 0
    assert fast.tobytes() == ops.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dropin_device_route_reduced_precision(tmp_path, dtype):
    """FMOE_DROPIN_DTYPE=f32 (bf16x6 tensor-core products) / bf16 runs the same
    reference API on the tensor cores.  f32: every section (y, the whole
    cache, d_x, all gradients, losses, trained parameters, last forward)
    within SURVEY 8(c)'s fp32 gradient bound (rel-L2 1e-4) of the f64
    composition.  bf16: SURVEY 8(c)'s bf16 rule compares against the oracle
    fed the ROUNDED values, so both runs start from inputs and weights rounded
    to bf16 (biases to fp32; FAST_ROUTE_ROUND_BF16=1) and the remaining
    difference is the route's bf16 storage of activations with fp32
    accumulation: y and d_x on the tokens whose top-k matches at 1e-2 / 2e-2,
    the gradients, losses and trained parameters at 2e-2, the cache sections
    not at all (a rerouted near-tie token shifts rows)."""
    import numpy as np

    E, k, n, d = 8, 2, 1024, 128
    shape = (str(n), str(d), "256", str(E))
    rnd = {"FAST_ROUTE_ROUND_BF16": "1"} if dtype == "bf16" else {}
    _, low = _fast_route_dump(tmp_path, dtype, {"FMOE_DROPIN_DTYPE": dtype, **rnd}, shape)
    _, ref = _fast_route_dump(tmp_path, "ops", {"FMOE_DROPIN_PATH": "ops", **rnd}, shape)
    n_cache = 4 + 3 * E
    assert len(low) == len(ref) == n_cache + 2 + 4 * E + 2 + 3 + 1 + 4 * E + 1
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))  # noqa: E731
    if dtype == "f32":
        for i, (a, b) in enumerate(zip(low, ref)):
            assert a.shape == b.shape, i
            if b.size and np.linalg.norm(b):
                assert rel(a, b) < 1e-4, (i, rel(a, b))
        return
    top = lambda s: np.sort(np.argsort(-s.reshape(n, E), axis=1, kind="stable")[:, :k], axis=1)  # noqa: E731
    same = (top(low[1]) == top(ref[1])).all(axis=1)
    assert same.mean() > 0.99, same.mean()
    rows = lambda s: s.reshape(n, d)[same]  # noqa: E731
    assert rel(rows(low[0]), rows(ref[0])) < 1e-2                      # y
    assert rel(rows(low[n_cache]), rows(ref[n_cache])) < 2e-2          # d_x
    for i in range(n_cache + 1, len(ref)):
        if i in (n_cache + 1 + 4 * E, n_cache + 2 + 4 * E):           # edited-cache d_x, d_wg (f64 composition)
            continue
        a, b = low[i], ref[i]
        assert a.shape == b.shape, i
        if i == len(ref) - 1:                                          # last forward: matched tokens
            assert rel(rows(a), rows(b)) < 2e-2
        elif b.size and np.linalg.norm(b):
            assert rel(a, b) < 2e-2, (i, rel(a, b))
