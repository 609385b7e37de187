"""bench.py's contract on the GPU: the single-GPU line (every key the driver
reads) and the N>1 path under torchrun.

The multi-rank run uses --shared-gpu (every rank on cuda:0, gloo plumbing, the
fused peer exchange over CUDA IPC) because the test box has one GPU; it runs
the same code as an N-GPU launch from the barrier / max-over-ranks timing to
the expert-parallel step and the host-buffer e2e loop.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "gpu_launches", "clocks", "roofline", "e2e"}


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--workload", "cfg3", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--e2e-steps", "2"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert KEYS <= set(line), KEYS - set(line)
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["value"] > 0
    assert line["gpu_launches"] > 0 and line["roofline"]["bound"] == "tensor"
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert "workload" in line["config"]


@pytest.mark.parametrize("workload", ["cfg3", "cfg5"])
def test_bench_two_ranks_shared_gpu(workload):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--workload", workload, "--steps", "3", "--warmup", "3", "--shared-gpu", "--e2e-steps", "2"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "ep2"
    assert "shared_gpu" in line["config"] and line["value"] > 0 and line["gpu_launches"] > 0
    if workload == "cfg3":
        assert line["e2e"]["value"] > 0
