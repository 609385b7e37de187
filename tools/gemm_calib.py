"""Our grouped expert GEMMs against cuBLAS on the same FLOPs, same box, same
thermal state (cfg2 shapes).  Interleaves R rounds of: K layer steps (stage
events give each expert GEMM's time) and K repetitions of the equivalent
cuBLAS products (torch.matmul / bmm, bf16 in, fp32 accumulate):

  fc1        [N*k, d] @ [d, h]              (dense, the 64 experts' rows stacked)
  fc2        [N*k, h] @ [h, d]
  dgrad_fc2  [N*k, d] @ [d, h]
  dgrad_fc1  [N*k, h] @ [h, d]
  wgrad_fc2  64 x [h, N*k/64] @ [N*k/64, d]   (bmm, bf16 out; ours writes fp32)
  wgrad_fc1  64 x [d, N*k/64] @ [N*k/64, h]

Prints one JSON line per round and a summary (TF/s of each, ratio ours/cuBLAS).
"""
import ctypes as C
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2103_13262_b200 as fm  # noqa: E402
from paper_2103_13262_b200 import _lib  # noqa: E402


def main():
    K = int(os.environ.get("K", "20"))
    R = int(os.environ.get("R", "3"))
    n, d, h, E, k = 65536, 1024, 4096, 64, 2
    rows = n * k
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    out = []
    with torch.cuda.stream(s):
        layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, E, 1, 42), dtype=torch.bfloat16)
        x = (torch.rand(n, d, device="cuda") * 2 - 1).bfloat16()
        dy = (torch.rand(n, d, device="cuda") * 2 - 1).bfloat16()
        y, dx = torch.empty_like(x), torch.empty_like(x)
        A1 = torch.randn(rows, d, device="cuda").bfloat16()
        B1 = torch.randn(d, h, device="cuda").bfloat16()
        A2 = torch.randn(rows, h, device="cuda").bfloat16()
        B2 = torch.randn(h, d, device="cuda").bfloat16()
        per = rows // E
        Hm = torch.randn(E, h, per, device="cuda").bfloat16()
        Dy = torch.randn(E, per, d, device="cuda").bfloat16()
        Xm = torch.randn(E, d, per, device="cuda").bfloat16()
        Dp = torch.randn(E, per, h, device="cuda").bfloat16()
        C1 = torch.empty(rows, h, device="cuda").bfloat16()
        C2 = torch.empty(rows, d, device="cuda").bfloat16()
        W2 = torch.empty(E, h, d, device="cuda").bfloat16()
        W1 = torch.empty(E, d, h, device="cuda").bfloat16()
        cub = {
            "fc1": lambda: torch.matmul(A1, B1, out=C1),
            "fc2": lambda: torch.matmul(A2, B2, out=C2),
            "wgrad_fc2": lambda: torch.bmm(Hm, Dy, out=W2),
            "wgrad_fc1": lambda: torch.bmm(Xm, Dp, out=W1),
        }
        flop = 2.0 * rows * d * h
        for _ in range(3):
            layer.forward(x, y)
            layer.backward(dy, dx)
        for name, f in cub.items():
            f()
        torch.cuda.synchronize()
        for r in range(R):
            clk = bench.Clocks(0)
            clk.region(True)
            _lib.check(_lib.lib.fmoe_ctx_profile(layer.ctx.h, K))
            for _ in range(K):
                layer.forward(x, y)
                layer.backward(dy, dx)
            torch.cuda.synchronize()
            stage = (C.c_float * len(bench.STAGES))()
            done = C.c_int()
            _lib.check(_lib.lib.fmoe_ctx_profile_read(layer.ctx.h, stage, len(bench.STAGES), C.byref(done)))
            _lib.check(_lib.lib.fmoe_ctx_profile(layer.ctx.h, 0))
            ours = {bench.STAGES[i]: stage[i] / max(done.value, 1) for i in range(1, len(bench.STAGES))}
            ck_ours = clk.stop()
            clk = bench.Clocks(0)
            clk.region(True)
            res = {}
            for name, f in cub.items():
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(K):
                    f()
                e1.record(s)
                torch.cuda.synchronize()
                res[name] = e0.elapsed_time(e1) / K
            ck_cub = clk.stop()
            line = {"round": r,
                    "ours_tflops": {g: round(flop / (ours[g] / 1e3) / 1e12, 1) for g in bench.GEMM_STAGES},
                    "cublas_tflops": {g: round(flop / (v / 1e3) / 1e12, 1) for g, v in res.items()},
                    "ours_sm_mhz": ck_ours.get("sm_mhz"), "cublas_sm_mhz": ck_cub.get("sm_mhz"),
                    "ours_power_w": ck_ours.get("power_w_median"), "cublas_power_w": ck_cub.get("power_w_median"),
                    "note": "cuBLAS wgrad writes bf16 (half of our fp32 gradient bytes); ours is the grouped kernel in the layer step"}
            out.append(line)
            print(json.dumps(line), flush=True)
    summ = {}
    for g in ("fc1", "fc2", "wgrad_fc2", "wgrad_fc1"):
        o = statistics.median([ln["ours_tflops"][g] for ln in out])
        c = statistics.median([ln["cublas_tflops"][g] for ln in out])
        summ[g] = {"ours": o, "cublas": c, "ratio": round(o / c, 3)}
    print(json.dumps({"summary": summ}))


if __name__ == "__main__":
    main()
