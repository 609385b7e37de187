#!/usr/bin/env python
"""bench.py -- FastMoE MoE-layer forward+backward tokens/s on B200.

Workload (BASELINE.json configs[1]) at N=1: one MoE layer,
d_model=1024, d_hidden=4096, 64 experts, top-2, 65536 tokens, bf16 storage /
fp32 accumulation, synthetic inputs, weights from the reference's init_state
generators.  A step = forward + backward of the layer (gate, plan, scatter,
grouped expert GEMMs, gather-combine, and every gradient).  At N>1 (torchrun,
one process per GPU) the same layer runs under expert parallelism: its 64
experts sharded 64/N per GPU, 65536 tokens per GPU -- weak scaling of the N=1
workload, so the per-N values compare directly.  --workload cfg3|cfg4|cfg5
runs the other BASELINE configs (cfg3: d=2048/h=8192, 8 experts and 16384
tokens per GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ...]

Timing: W warm-up steps, then exactly K steps bracketed by barrier +
synchronize, timed with CUDA events on the layer's stream, max over ranks.
The working set (inputs + activations + weights, several GB) is far above the
126 MB L2, so no flush is needed between steps.  Per-stage CUDA events are
recorded inside the same timed region (fmoe_ctx_profile) and give the
roofline of the dominant kernel (the tcgen05 grouped GEMM).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer fwd+bwd tokens/s at 1/2/4/8 B200; expert-GEMM % of tensor peak"
UNIT = "tokens/s"
CFG2 = dict(n_b=65536, d_m=1024, d_h=4096, n_e_local=64, k=2)          # 1 GPU
CFG3 = dict(n_b=16384, d_m=2048, d_h=8192, n_e_local=8, k=2)           # EP, per GPU
CFG1 = dict(n_b=8192, d_m=1024, d_h=4096, n_e_local=16, k=2)           # fp32, the reference CPU path's config
CFG4_LAYERS = 12
ZIPF_S = 1.0


def workload_cfg(name: str, world: int) -> dict:
    """Per-GPU shape of a BASELINE workload at `world` GPUs."""
    if name == "cfg1":  # BASELINE configs[0]: the reference's own fp32 config, one GPU
        if world != 1:
            raise SystemExit("cfg1 is the single-GPU fp32 config (BASELINE configs[0])")
        return dict(CFG1)
    if name == "cfg2":  # the cfg2 layer (64 experts in total), 65536 tokens per GPU, sharded over the world
        if CFG2["n_e_local"] % world:
            raise SystemExit("cfg2 needs the world size to divide its 64 experts")
        return dict(CFG2, n_e_local=CFG2["n_e_local"] // world)
    if name == "cfg3":
        return dict(CFG3)
    if name == "cfg4":  # 12-layer stack, 128 experts over the world, 16384 tokens/GPU
        if 128 % world:
            raise SystemExit("cfg4 needs the world size to divide 128 experts")
        return dict(n_b=16384, d_m=1024, d_h=4096, n_e_local=128 // world, k=2)
    if name == "cfg5":  # Zipf routing, 256 experts top-1, 262144 tokens in total
        if 256 % world:
            raise SystemExit("cfg5 needs the world size to divide 256 experts")
        return dict(n_b=262144 // world, d_m=1024, d_h=4096, n_e_local=256 // world, k=1)
    raise SystemExit(f"unknown workload {name}")


SEED = 42
STAGES = ["-", "gate", "plan", "scatter", "fc1", "fc2", "gather_combine", "fwd_bwd_gap",
          "gather_combine_bwd", "dgrad_fc2", "wgrad_fc2", "db2", "dgrad_fc1", "wgrad_fc1", "db1",
          "gate_dwg", "gate_dx_scatter_bwd"]
GEMM_STAGES = ["fc1", "fc2", "dgrad_fc2", "wgrad_fc2", "dgrad_fc1", "wgrad_fc1"]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return dict(hbm=j["hbm_gbs"], tc=j["bf16_tflops"], tc_sus=j.get("bf16_tflops_sustained", j["bf16_tflops"]),
                    src="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, tc=1590.0, tc_sus=1400.0, src="fallback (B200_PROFILING.md)")


# ------------------------------------------------------------------ clocks
class Clocks:
    """SM clock, power and clock-event reasons sampled with NVML every
    `period` seconds on a background thread (nvidia-smi at 100 ms gave one
    sample in a 0.12 s timed region).  `region(True/False)` brackets the timed
    region; the summary covers the samples taken inside it (all samples when
    the region saw fewer than 3)."""
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int, period: float = 0.005):
        import threading

        self.samples, self.in_region, self.err = [], False, None
        self.stop_ev = threading.Event()
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self._nvml_index(device))
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        except Exception as e:  # no NVML: report it, never guess
            self.nv, self.err = None, f"nvml unavailable: {e}"
            return
        self.period = period
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    @staticmethod
    def _nvml_index(device: int) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[device])
            except (ValueError, IndexError):
                pass
        return device

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1e3
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((self.in_region, sm, pw, rs))
            except Exception as e:
                self.err = str(e)
            time.sleep(self.period)

    def region(self, inside: bool):
        self.in_region = inside

    def stop(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err]}
        self.stop_ev.set()
        self.t.join(timeout=2)
        inside = [x for x in self.samples if x[0]]
        use = inside if len(inside) >= 3 else self.samples
        sm = [x[1] for x in use]
        pw = [x[2] for x in use]
        reasons = sorted({n for x in use for n, b in self.bits.items() if x[3] & b})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "sm_mhz_min": min(sm) if sm else None, "sm_mhz_max_seen": max(sm) if sm else None,
                "power_w_median": statistics.median(pw) if pw else None, "power_w_max": max(pw) if pw else None,
                "samples": len(use), "samples_in_timed_region": len(inside),
                "sampler": f"NVML every {self.period * 1e3:.0f} ms", "reasons": reasons}


def tensor_peak(pk: dict, clk: dict):
    """Roofline denominator for the expert GEMM: the burst cuBLAS figure when
    the SM clock sat at its maximum through the timed region, the sustained
    (power-capped, seconds-long) figure when it was held below it.  The clock
    is the one the GEMMs ran at (in-kernel clock64 / globaltimer probe) when
    available -- NVML's clocks.sm reads the maximum while the power-capped
    part runs dense GEMMs at ~1.3-1.5 GHz -- else NVML's median."""
    sm, mx = clk.get("gemm_sm_mhz_effective") or clk.get("sm_mhz"), clk.get("sm_max_mhz")
    if sm and mx and sm >= 0.97 * mx:
        return pk["tc"], "burst (median SM clock at max through the timed region)"
    if sm and mx:
        return pk["tc_sus"], (f"sustained (median SM clock {sm:.0f} of {mx:.0f} MHz under the power cap; "
                              "the burst figure needs the maximum clock)")
    return pk["tc_sus"], "sustained (no clock samples)"


# ------------------------------------------------------------- CPU reference
def cpu_reference(n_tokens: int, cfg: dict, min_seconds: float = 10.0, max_reps: int = 5,
                  workload: str = "cfg2", n_layers: int = 1, e_total: int = 0):
    """The reference's own forward+backward (oracle/_ref, compiled from its
    sources) on the host cores: tokens/s on a bounded token sample of the
    workload's layer (all e_total experts on one worker).  cfg5 feeds the same
    Zipf IndexMatrix to the reference's dispatch + expert pool; cfg4 divides
    the one-layer rate by the stack depth."""
    cores = os.cpu_count() or 1
    os.environ["FMOE_THREADS"] = str(cores)
    from oracle import bindings

    if not bindings.ref_available():
        return None
    e_total = e_total or cfg["n_e_local"]
    so, build = bindings.ref_timing_so()
    lib = C.CDLL(so)
    routed = workload == "cfg5"
    if routed:
        import numpy as np

        from paper_2103_13262_b200.workloads import zipf_routing

        idx, sc = zipf_routing(n_tokens, e_total, cfg["k"], ZIPF_S, seed=7)
        idx64 = np.ascontiguousarray(idx, dtype=np.int64)
        sc64 = np.ascontiguousarray(sc, dtype=np.float64)
        create, step, destroy = lib.ref_bench_routed_create, lib.ref_bench_routed_step, lib.ref_bench_routed_destroy
        create.argtypes = [C.c_uint64] + [C.c_int64] * 5 + [C.c_void_p, C.c_void_p]
        extra = (idx64.ctypes.data, sc64.ctypes.data)
    else:
        create, step, destroy = lib.ref_bench_create, lib.ref_bench_step, lib.ref_bench_destroy
        create.argtypes = [C.c_uint64] + [C.c_int64] * 5
        extra = ()
    create.restype = C.c_void_p
    step.argtypes = [C.c_void_p]
    destroy.argtypes = [C.c_void_p]
    h = create(SEED, n_tokens, cfg["d_m"], cfg["d_h"], e_total, cfg["k"], *extra)
    if not h:
        return None
    try:
        step(h)  # warm-up
        times = []
        t_all = time.perf_counter()
        while len(times) < max_reps and (len(times) < 2 or time.perf_counter() - t_all < min_seconds):
            t0 = time.perf_counter()
            step(h)
            times.append(time.perf_counter() - t0)
    finally:
        destroy(h)
    mean = statistics.mean(times)
    what = ("Zipf-routed dispatch + expert pool (build_plan .. scatter_backward)" if routed
            else "forward+backward")
    stack = f", rate / {n_layers} layers" if n_layers > 1 else ""
    full = n_tokens >= cfg["n_b"]
    return {"value": n_tokens / mean / n_layers, "unit": UNIT, "cores": cores, "kind": "reference",
            "reps": len(times), "tokens_per_rep": n_tokens, "s_per_rep": mean, "build": build,
            "sample": (f"{n_tokens} tokens of d_m={cfg['d_m']} d_h={cfg['d_h']} E={e_total} "
                       f"k={cfg['k']} (" + ("the full workload" if full else "the GPU workload's layer, "
                                            "token-subsampled") + f"), fp64, reference "
                       f"{what}{stack}, warm-up 1 + {len(times)} reps, mean {mean:.2f} s/step, "
                       f"FMOE_THREADS={cores}, built {build}")}


def reference_api_line(cfg: dict, reps: int = 5):
    """tokens/s of fmoe::forward + fmoe::backward (the reference's C++ API)
    through libfmoe_dropin.so, FMOE_F64, via fmoe_bench bench-local --api
    reference (the reference's moe_batched_fwdbwd loop)."""
    exe = os.path.join(ROOT, "paper_2103_13262_b200", "fmoe_bench")
    if not os.path.exists(exe):
        return {"unavailable": "paper_2103_13262_b200/fmoe_bench not built"}
    cmd = [exe, "bench-local", "--api", "reference", "--n-b", str(cfg["n_b"]), "--d-m", str(cfg["d_m"]),
           "--d-h", str(cfg["d_h"]), "--k", str(cfg["k"]), "--n-e", str(cfg["n_e_local"]), "--reps", str(reps),
           "--warmup", "2"]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=600).stdout
    except Exception as e:  # report, never guess
        return {"unavailable": f"fmoe_bench failed: {e}"}
    rows = {r.split(",")[0]: r.split(",") for r in out.splitlines() if r and not r.startswith(("#", "scenario"))}
    if "moe_batched_fwdbwd" not in rows:
        return {"unavailable": "fmoe_bench printed no moe_batched_fwdbwd row: " + out[-300:]}
    ms = float(rows["moe_batched_fwdbwd"][8])
    ms_host = float(rows["moe_batched_fwdbwd_host_results"][8]) if "moe_batched_fwdbwd_host_results" in rows else None
    return {"value": cfg["n_b"] / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
            "value_host_results": cfg["n_b"] / (ms_host / 1e3) if ms_host else None, "ms_per_step_host_results": ms_host,
            "dtype": "f64 (FMOE_F64: bit-identical to the reference and to the drop-in's operator composition)",
            "path": ("fmoe::init_state / forward(x, state, nullptr, &cache) / backward(d_y, cache, state) of the "
                     "reference headers (include/fmoe/moe_layer.hpp) through libfmoe_dropin.so's device-resident "
                     "route: x, d_y uploaded per step, parameters resident, results device-backed Matrices"),
            "value_host_results_note": "the same loop with y and d_x read on the host every step",
            "timing": f"host steady_clock, warm-up 2 + {reps} reps (fmoe_bench bench-local --api reference)"}


def cpu_tokens_for(cores: int) -> int:
    # ~6 s of reference work per rep on 16 host cores at cfg2 (4096 tokens: 64
    # rows per expert, so its per-expert GEMMs are not starved for rows)
    return max(256, min(8192, 256 * cores))


# --------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="default", choices=["default", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5"],
                    help="BASELINE config (SURVEY §8d); default cfg2: its layer at every N (weak scaling); "
                         "cfg1: the reference's fp32 config (8192 tokens, 16 experts) through FMOE_F32")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--graph", action="store_true",
                    help="replay the single-GPU fwd+bwd step as one captured CUDA graph")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="N>1 code-path check on a one-GPU box: every rank on cuda:0, gloo plumbing, peer "
                         "buffers exchanged through it (the fused exchange over CUDA IPC); NOT a scaling number")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.workload == "default":
        args.workload = "cfg2"
    cfg = workload_cfg(args.workload, world)
    if args.impl == "reference":
        return run_reference(args, world, rank, cfg)
    return run_ours(args, world, rank, cfg)


def n_layers_of(workload: str) -> int:
    return CFG4_LAYERS if workload == "cfg4" else 1


def cpu_sample_tokens(workload: str, cores: int) -> int:
    if workload == "cfg1":  # the reference's own config: full size (warm-up 1 + 3 reps)
        return CFG1["n_b"]
    n = cpu_tokens_for(cores)
    return max(256, n // 4) if workload == "cfg4" else n


def run_reference(args, world, rank, cfg):
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    n_tok = cpu_sample_tokens(args.workload, cores)
    reps = 3 if args.workload == "cfg1" else max(2, min(args.steps, 10))
    res = cpu_reference(n_tok, cfg, min_seconds=max(10.0, 2.0 * args.steps), max_reps=reps,
                        workload=args.workload, n_layers=n_layers_of(args.workload),
                        e_total=cfg["n_e_local"] * world)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfmoe_ref.so not built"}))
        return 0
    # a step of this arm = one timed rep of the (sampled) workload: steps and
    # ms_per_step are what actually ran, so steps x ms_per_step fits the run
    line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": res["reps"], "steps_requested": args.steps, "warmup": 1, "higher_is_better": True,
            "ms_per_step": 1e3 * res["s_per_rep"], "tokens_per_step": res["tokens_per_rep"],
            "ms_per_full_workload_step": 1e3 * cfg["n_b"] * world / res["value"], "dtype": "f64", "data": "synthetic",
            "scaling": "weak", "vs_baseline": None,
            "config": {"workload": workload_name(args.workload, cfg, world), **cfg, "world": world},
            "cpu_baseline": res,
            "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def workload_name(workload, cfg, world):
    if workload == "cfg1":
        return ("cfg1: single MoE layer d_model=1024 d_hidden=4096, 16 experts top-2, 8192 tokens, fp32 "
                "(FMOE_F32: gate and permutes in fp32, expert GEMMs as bf16x6 split products on the tensor "
                "cores, fp32 accumulate), fwd+bwd")
    if workload == "cfg2":
        if world == 1:
            return ("cfg2: single MoE layer d_model=1024 d_hidden=4096, 64 experts top-2, 65536 tokens, "
                    "bf16 storage / fp32 accumulate, fwd+bwd")
        return (f"cfg2 layer under expert parallelism: d_model=1024 d_hidden=4096, 64 experts top-2 sharded "
                f"{64 // world} per GPU over {world} GPUs, 65536 tokens per GPU (weak scaling of the N=1 "
                "workload), bf16 storage / fp32 accumulate, fwd+bwd")
    if workload == "cfg3":
        return (f"cfg3: expert-parallel MoE layer d_model=2048 d_hidden=8192, 8 experts/GPU x {world} GPUs, "
                "top-2, 16384 tokens/GPU, fwd+bwd")
    if workload == "cfg4":
        return (f"cfg4: GPT-style MoE FFN stack, {CFG4_LAYERS} chained layers (no residual/norm, as the "
                f"reference), d_model=1024 d_hidden=4096, 128 experts top-2 over {world} GPU(s), "
                "16384 tokens/GPU, fwd through all layers then bwd")
    return (f"cfg5: skewed-gate stress, injected Zipf(s={ZIPF_S}) routing over 256 experts top-1, "
            f"262144 tokens in total ({cfg['n_b']}/GPU), d_model=1024 d_hidden=4096, fwd+bwd")


def run_ours(args, world, rank, cfg):
    import torch

    shared = args.shared_gpu and world > 1
    if world > 1 and not shared:  # NCCL's INIT lines (rings, NVLS, P2P) on stderr, for the scaling runs
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    local = 0 if shared else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def max_over_ranks(v: float) -> float:
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    import paper_2103_13262_b200 as fm
    from paper_2103_13262_b200 import _lib
    from paper_2103_13262_b200.workloads import MoEStack, zipf_routing

    wl = args.workload
    n_layers = n_layers_of(wl)
    n, d, h, el, k = cfg["n_b"], cfg["d_m"], cfg["d_h"], cfg["n_e_local"], cfg["k"]
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        mcfg = fm.MoEConfig(n, d, h, k, el, world, SEED)
        dt = torch.float32 if wl == "cfg1" else torch.bfloat16
        if wl == "cfg4":
            model = MoEStack(mcfg, n_layers, rank=rank, dtype=dt)
            layer0 = model.layers[0]
        else:
            model = layer0 = fm.MoELayer(mcfg, rank=rank, dtype=dt)
        if shared:
            model.connect_peers(dist)
        elif world > 1:
            model.connect(dist)
        g = torch.Generator(device="cuda")
        g.manual_seed(1000 + rank)
        x = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).to(dt)
        dy = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).to(dt)
        es = x.element_size()
        y = torch.empty_like(x)
        dx = torch.empty_like(x)
        if wl == "cfg5":
            ridx, rsc = zipf_routing(n, el * world, k, ZIPF_S, seed=7 + rank)
            ridx = torch.as_tensor(ridx, device="cuda")
            rsc = torch.as_tensor(rsc, device="cuda")

            def step():
                model.forward_routed(x, ridx, rsc, y)
                model.backward(dy, dx)
        else:
            def step():
                model.forward(x, y)
                model.backward(dy, dx)

        clocks = Clocks(local)  # sampled from the warm-up (under load) through the timed region
        for _ in range(max(args.warmup, 3)):
            step()
        eager_step = step
        if args.graph:
            if world > 1 or wl != "cfg2":
                raise SystemExit("--graph: the single-GPU cfg2 step only")
            graph = torch.cuda.CUDAGraph()
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=stream):
                step()
            step = graph.replay
            step()
        ctx = layer0.ctx
        if not args.graph:  # graph replays carry no host-side stage marks; profiled eagerly below
            _lib.check(_lib.lib.fmoe_ctx_profile(ctx.h, args.steps * n_layers))
            _lib.check(_lib.lib.fmoe_ctx_clock_probe(ctx.h, args.steps * n_layers * 6))
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        launches0 = ctx.launches
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        torch.cuda.synchronize()
        clocks.region(True)
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        clocks.region(False)
        clk = clocks.stop()
        t0, t1 = evs[0], evs[-1]
        per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
        if dist:
            dist.barrier()
        launches = ctx.launches - launches0
        if args.graph:  # every replay launches the captured kernels: count them from one eager step
            l0 = ctx.launches
            eager_step()
            launches = (ctx.launches - l0) * args.steps
            _lib.check(_lib.lib.fmoe_ctx_profile(ctx.h, args.steps))
            for _ in range(args.steps):
                eager_step()
        ms = t0.elapsed_time(t1) / args.steps
        ms_sd = statistics.stdev(per_step) if len(per_step) > 1 else 0.0
        stage = (C.c_float * len(STAGES))()
        done = C.c_int()
        _lib.check(_lib.lib.fmoe_ctx_profile_read(ctx.h, stage, len(STAGES), C.byref(done)))
        _lib.check(_lib.lib.fmoe_ctx_profile(ctx.h, 0))
        eff_mhz, probed = C.c_double(0.0), C.c_int(0)
        if not args.graph:
            _lib.check(_lib.lib.fmoe_ctx_clock_probe_read(ctx.h, C.byref(eff_mhz), C.byref(probed)))
            _lib.check(_lib.lib.fmoe_ctx_clock_probe(ctx.h, 0))
        clk["gemm_sm_mhz_effective"] = round(eff_mhz.value, 1) if probed.value else None
        clk["gemm_clock_probe"] = (f"clock64 / globaltimer of CTA 0 over {probed.value} expert-GEMM launches "
                                   "inside the timed region: the SM clock the tensor cores actually ran at")
        # per layer-step averages
        stage_ms = {STAGES[i]: stage[i] / max(done.value, 1) for i in range(1, len(STAGES))}
        if dist:
            ms = max_over_ranks(ms)
        tokens = n * world
        value = tokens / (ms / 1e3)

        # ---- end to end through the public host-buffer entry point (single layers)
        e2e = None
        if wl in ("cfg1", "cfg2", "cfg3"):
            e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
            hx = x.cpu().pin_memory()
            hdy = dy.cpu().pin_memory()
            hy = torch.empty_like(hx).pin_memory()
            hdx = torch.empty_like(hx).pin_memory()
            layer0.step_host(hx, hdy, hy, hdx)
            if dist:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            # the public host-buffer loop: every step uploads x, dy from pinned
            # host memory and downloads y, dx; consecutive steps overlap their
            # copies with each other's kernels (fmoe_layer_step_host_async)
            e0.record(stream)
            for _ in range(e2e_steps):
                layer0.step_host_async(hx, hdy, hy, hdx)
            layer0.wait_host()
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_ms = e0.elapsed_time(e1) / e2e_steps
            # the synchronous call (results back on the host before it returns), for reference
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(3):
                layer0.step_host(hx, hdy, hy, hdx)
            s1.record(stream)
            torch.cuda.synchronize()
            sync_ms = s0.elapsed_time(s1) / 3
            # training-loop variant (reported beside the headline, never instead of
            # it): x arrives from pinned host memory every step (double-buffered
            # upload on a copy stream, overlapping the previous step), d_y is
            # device-resident as the downstream layer would leave it, d_x stays
            # on the device for the upstream layer, and the step's result read
            # back is one fp32 scalar (sum of y, a loss stand-in)
            copy = torch.cuda.Stream()
            xb = [torch.empty_like(x), torch.empty_like(x)]
            up = [torch.cuda.Event(), torch.cuda.Event()]
            used = [torch.cuda.Event(), torch.cuda.Event()]
            res_d = torch.empty(e2e_steps, dtype=torch.float32, device="cuda")
            res_h = torch.empty(e2e_steps, dtype=torch.float32).pin_memory()

            def upload(i):
                with torch.cuda.stream(copy):
                    if i >= 2:
                        copy.wait_event(used[i & 1])
                    xb[i & 1].copy_(hx, non_blocking=True)
                    up[i & 1].record(copy)

            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0_ = torch.cuda.Event(enable_timing=True)
            t1_ = torch.cuda.Event(enable_timing=True)
            t0_.record(stream)
            upload(0)
            for i in range(e2e_steps):
                if i + 1 < e2e_steps:
                    upload(i + 1)
                stream.wait_event(up[i & 1])
                layer0.forward(xb[i & 1], y)
                layer0.backward(dy, dx)
                used[i & 1].record(stream)
                torch.sum(y, dim=(0, 1), dtype=torch.float32, out=res_d[i])
                res_h[i].copy_(res_d[i], non_blocking=True)
            t1_.record(stream)
            torch.cuda.synchronize()
            tl_ms = t0_.elapsed_time(t1_) / e2e_steps
            if dist:
                e2e_ms = max_over_ranks(e2e_ms)
                tl_ms = max_over_ranks(tl_ms)
            # PCIe ceiling of the host-buffer path: x + dy up and y + dx down per
            # step, full duplex, at the copy rates measured here
            # (best of three copies each way: a single copy can read low on a cold mapping)
            h2d_gbs = d2h_gbs = 0.0
            for _ in range(3):
                c0, c1, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                c0.record(stream)
                xb[0].copy_(hx, non_blocking=True)
                c1.record(stream)
                hy.copy_(xb[0], non_blocking=True)
                c2.record(stream)
                torch.cuda.synchronize()
                h2d_gbs = max(h2d_gbs, n * d * es / (c0.elapsed_time(c1) / 1e3) / 1e9)
                d2h_gbs = max(d2h_gbs, n * d * es / (c1.elapsed_time(c2) / 1e3) / 1e9)
            pcie_cap = tokens / max(2 * n * d * es / (h2d_gbs * 1e9), 2 * n * d * es / (d2h_gbs * 1e9))
            e2e = {"value": tokens / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 2 * n * d * es,
                   "d2h_bytes_per_step": 2 * n * d * es,
                   "sync_call_value": tokens / (sync_ms / 1e3),
                   "note": (f"the PCIe traffic of a step ({2 * n * d * es >> 20} MiB each way) hides under the kernels of the "
                            "neighbouring steps, so the host loop runs at the device-resident rate; the "
                            "device-resident loop additionally records its per-stage CUDA events; "
                            "sync_call_value: one fmoe_layer_step_host call per step, results on the host "
                            "before it returns"),
                   "path": ("fmoe_layer_step_host_async x K + wait (pinned host x,dy -> H2D -> fwd+bwd -> "
                            "D2H y,dx every step; copy streams overlap the uploads / downloads with the "
                            "kernels of the same and the neighbouring steps)"),
                   "pcie_ceiling_value": pcie_cap, "h2d_GBps": h2d_gbs, "d2h_GBps": d2h_gbs,
                   "pcie_ceiling_note": ("x, dy in and y, dx out: 2 x n_b x d_m bf16 per direction per step at the "
                                         "H2D / D2H rates measured here cap the host-buffer path at this rate "
                                         "however fast the kernels get (DESIGN.md §6)"),
                   "training_loop": {"value": tokens / (tl_ms / 1e3), "unit": UNIT,
                                     "h2d_bytes_per_step": n * d * es, "d2h_bytes_per_step": 4,
                                     "path": ("MoELayer.forward/backward: x uploaded from pinned host memory each "
                                              "step (copy stream, double-buffered), d_y device-resident, d_x left "
                                              "on the device, one fp32 scalar (sum of y) read back per step")}}

    # cfg1: the same workload through the reference's own C++ API (fmoe::forward
    # + fmoe::backward of include/fmoe/moe_layer.hpp, host Matrix values) served
    # by libfmoe_dropin.so on this GPU in FMOE_F64 -- bit-identical to the
    # reference -- timed by the reference's bench-local loop (host clock)
    ref_api = None
    if wl == "cfg1" and rank == 0:
        ref_api = reference_api_line(cfg)

    pk = peaks()
    peak, peak_why = tensor_peak(pk, clk)
    # expert GEMM FLOPs of one launch (fmoe_bench.cpp:110-126): 2 * rows * d * h,
    # rows = tokens routed to this rank's experts (N*k per rank on average)
    flop_gemm = 2.0 * n * k * d * h
    gemm_ms = [stage_ms[s] for s in GEMM_STAGES]
    avg_launch_ms = sum(gemm_ms) / len(gemm_ms)
    if avg_launch_ms <= 0:  # no per-GEMM stage marks on this path (FMOE_F32_SIMT)
        avg_launch_ms = float("nan")
    # cfg1 (FMOE_F32): each expert GEMM is 6 bf16 passes on the tensor pipe
    # (bf16x6 split products, tc_gemm.cuh / f32x.cu); the roofline counts the
    # pipe's work, algorithmic_fp32_tflops the fp32 FLOPs the layer delivers
    passes = 6 if wl == "cfg1" else 1
    achieved = passes * flop_gemm / (avg_launch_ms / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and wl == "cfg2":
        try:
            traffic = json.load(open(tp)).get("tc_gemm_dram_bytes_per_launch")
        except Exception:
            traffic = None
    s = es
    scatter_bytes = s * d * (n + n * k) + 4 * n * k
    gather_bytes = s * d * (n * k + n) + 8 * n * k
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "ms_per_step_stddev": ms_sd, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if wl == "cfg1" else "bf16",
        "data": "synthetic (uniform[-1,1) inputs; reference init_state weights"
                + ("; injected Zipf routing" if wl == "cfg5" else "") + ")",
        "config": {"workload": workload_name(wl, cfg, world), "n_b_per_gpu": n, "d_m": d, "d_h": h,
                   "experts_per_gpu": el, "experts_total": el * world, "k": k, "layers": n_layers,
                   "parallelism": f"ep{world}" if world > 1 else "single",
                   "l2": "working set several GB >> 126 MB L2; no flush needed",
                   "launch": "one CUDA graph per step" if args.graph else "eager stream launches",
                   **({"shared_gpu": f"all {world} ranks on ONE GPU (code-path check, gloo plumbing, fused "
                                     "peer exchange over CUDA IPC): not a scaling number"} if shared else {})},
        "gpu_launches": launches,
        "clocks": clk,
        "roofline": {"kernel": "tc_gemm_kernel (grouped tcgen05 expert GEMM; fc1, fc2, 2x dgrad, 2x wgrad)",
                     "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "frac_of_burst_peak": achieved / pk["tc"],
                     "frac_of_sustained_peak": achieved / pk["tc_sus"],
                     **({"frac_of_clock_peak": achieved / (148 * 8192 * clk["gemm_sm_mhz_effective"] * 1e6 / 1e12),
                         "clock_peak_note": ("dense bf16 tcgen05 issue rate, 8192 flop/clk/SM x 148 SMs (2.25 PF at "
                                             "1.855 GHz), at the measured GEMM clock")}
                        if clk.get("gemm_sm_mhz_effective") else {}),
                     "frac_of_datasheet_2250": achieved / 2250.0,
                     "flops_per_launch": flop_gemm, "avg_launch_ms": avg_launch_ms, "traffic": traffic,
                     "peak_source": pk["src"] + " bf16, " + peak_why,
                     "per_gemm_tflops": {s_: round(flop_gemm / (stage_ms[s_] / 1e3) / 1e12, 1)
                                         for s_ in GEMM_STAGES if stage_ms[s_] > 0},
                     **({"algorithmic_fp32_tflops": flop_gemm / (avg_launch_ms / 1e3) / 1e12,
                         "bf16_passes_per_gemm": passes,
                         "note": ("FMOE_F32: fp32 operands split into three bf16 planes a0 + a1 + a2, each GEMM = "
                                  "a0*b2 + a2*b0 + a1*b1 + a0*b1 + a1*b0 + a0*b0 on tcgen05 into one fp32 accumulator "
                                  "(6 bf16 passes); 'achieved' counts the "
                                  "tensor pipe's bf16 work, per_gemm_tflops the fp32 FLOPs; stage times include the "
                                  "plane-split passes of the stage's operands")} if passes > 1 else {}),
                     **({"note": ("averaged over the six expert GEMMs; with few rows per expert the weight-gradient "
                                  "launches are bound by writing fp32 gradients (HBM), not by the tensor pipe "
                                  "(profiles/r01h_cfg4_wgrad.md); fc1/fc2/dgrad stages in stages_ms")}
                        if wl in ("cfg4", "cfg5") else {})},
        "stages_ms": {k_: round(v, 4) for k_, v in stage_ms.items()},
        "stages_source": ("eager steps after the graph-replay timed region" if args.graph
                          else "CUDA events inside the timed region"),
        "permute_roofline": {
            "scatter_GBps": scatter_bytes / (stage_ms["scatter"] / 1e3) / 1e9 if stage_ms["scatter"] > 0 else None,
            "gather_combine_GBps": (gather_bytes / (stage_ms["gather_combine"] / 1e3) / 1e9
                                    if stage_ms["gather_combine"] > 0 else None),
            "peak_GBps": pk["hbm"],
        },
    }
    if e2e is not None:
        line["e2e"] = e2e
    if ref_api is not None:
        line["reference_api"] = ref_api
    if world > 1:
        fused = bool(getattr(layer0, "ep_exchange_fused", False))
        st = stage_ms
        line["exchange"] = {
            "path": ("fused: count all-gather + row stores over NVLink peer memory inside the scatter / "
                     "fc2 / gather-combine-backward / dgrad-fc1 kernels" if fused
                     else "transport: grouped ncclSend/ncclRecv per (peer, local expert) chunk between kernels"),
            "fused": fused,
            # what each profiling stage spans under expert parallelism (ep.cu)
            "phases_ms": {"counts_and_layout (C1)": st["plan"],
                          "scatter + global_scatter (C2, incl. waiting for the peers' rows)": st["scatter"],
                          "fc1 + fc2 + global_gather (C3) + gather_combine": st["fc1"] + st["fc2"] + st["gather_combine"],
                          "gather_combine_bwd + d_ys global_scatter (incl. wait)": st["gather_combine_bwd"],
                          "backward experts + d_xs global_gather + gate": sum(st[k_] for k_ in (
                              "dgrad_fc2", "wgrad_fc2", "db2", "dgrad_fc1", "wgrad_fc1", "db1", "gate_dwg",
                              "gate_dx_scatter_bwd"))},
            "nvlink_bytes_per_step_per_gpu": 4 * n * k * d * 2 * (world - 1) // world,
        }
    pr = line["permute_roofline"]
    if world == 1 and pr["scatter_GBps"]:
        pr["scatter_frac"] = pr["scatter_GBps"] / pk["hbm"]
        pr["gather_frac"] = pr["gather_combine_GBps"] / pk["hbm"]
    else:
        pr["note"] = "under EP the scatter / gather stages include the NCCL exchanges"
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        line["cpu_baseline"] = cpu_reference(cpu_sample_tokens(wl, cores), cfg, workload=wl, n_layers=n_layers,
                                             e_total=el * world)
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
