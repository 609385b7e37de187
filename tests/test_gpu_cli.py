"""The benchmark CLI (paper_2103_13262_b200/fmoe_bench): the reference's
subcommands and CSV schema (tools/fmoe_bench.cpp:36-37, 94-107) on the GPU.

* bench-local prints the reference header and one row per scenario with the
  reference's FLOP accounting (fmoe_bench.cpp:110-126);
* train-toy in fp64 reproduces the reference's own train-toy trajectory
  (make_toy_task + train_step, oracle/_ref) to a few ulp;
* usage errors exit 2 like the reference.
"""
import csv
import io
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2103_13262_b200", "fmoe_bench")
HEADER = "scenario,n_b,d_m,d_h,n_e,k,world,reps,mean_ms,stddev_ms,gflops"


def run(*args):
    return subprocess.run([EXE, *args], capture_output=True, text=True, timeout=300)


def test_bench_local_csv():
    r = run("bench-local", "--n-b", "2048", "--d-m", "256", "--d-h", "512", "--k", "2", "--n-e", "8,16",
            "--reps", "3", "--warmup", "1")
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if not ln.startswith("#")]
    assert lines[0] == HEADER
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    assert [x["scenario"] for x in rows] == ["moe_batched_forward", "moe_batched_fwdbwd"] * 2
    assert [int(x["n_e"]) for x in rows] == [8, 8, 16, 16]
    for x in rows:
        n, d, h, e, k = (int(x[c]) for c in ("n_b", "d_m", "d_h", "n_e", "k"))
        fwd = 2.0 * n * d * e + 4.0 * n * k * d * h
        fl = fwd if x["scenario"].endswith("forward") else fwd + 4.0 * n * d * e + 8.0 * n * k * d * h
        assert abs(float(x["gflops"]) - fl / (float(x["mean_ms"]) * 1e-3) / 1e9) <= 1e-3 * float(x["gflops"])


def test_train_toy_f64_matches_reference(ref):
    n, d, h, el, k, seed, steps, lr = 64, 16, 24, 4, 2, 42, 6, 0.05
    r = run("train-toy", "--dtype", "f64", "--n-b", str(n), "--d-m", str(d), "--d-h", str(h), "--n-e", str(el),
            "--k", str(k), "--seed", str(seed), "--steps", str(steps), "--lr", str(lr))
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    losses = np.array([float(x["loss"]) for x in rows])
    x, t = ref.toy_task(n, d, h, k, el, 1, seed)
    want = ref.train_steps(x, t, 1, n, h, el, k, seed, steps, lr)["losses"]
    assert np.max(np.abs(losses - want)) <= 1e-13 * max(1.0, abs(want[0])), (losses, want)


def test_usage_errors_exit_2():
    assert run().returncode == 2
    assert run("bench-local", "--bogus", "1").returncode == 2
    assert run("bench-local", "--n-e", "2", "--k", "3").returncode == 2
