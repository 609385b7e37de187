"""Expert-parallel exchange overhead, measured on ONE GPU.

W ranks run as host threads on the same B200 (the in-process world), each
with its own stream and cfg3 layer slice (BASELINE configs[2]: d_model=2048,
d_hidden=8192, 8 experts per rank, 16384 tokens per rank, top-2).  All ranks
share the GPU, so their sum of work equals one worker holding all W*8 experts
and all W*16384 tokens; the difference between the two timings is what the
expert-parallel machinery costs on top of the computation (count all-gather,
layouts, the exchange -- fused into the scatter / GEMM epilogues, or through
the transport -- and the phase synchronisation).  It is not a multi-GPU
number: NVLink bandwidth does not enter.

  python tools/ep_overhead.py [--world 2] [--steps 10] [--warmup 3]
"""
import argparse
import json
import os
import sys
import threading

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

N, D, H, EL, K, SEED = 16384, 2048, 8192, 8, 2, 42  # cfg3 slice per rank (--workload cfg2: the cfg2 layer)


def time_steps(step, stream, steps, warmup):
    for _ in range(warmup):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream.synchronize()
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def single(fm, world, steps, warmup):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        layer = fm.MoELayer(fm.MoEConfig(N * world, D, H, K, EL * world, 1, SEED), dtype=torch.bfloat16)
        g = torch.Generator(device="cuda").manual_seed(1)
        x = (torch.rand(N * world, D, device="cuda", generator=g) * 2 - 1).bfloat16()
        dy = (torch.rand(N * world, D, device="cuda", generator=g) * 2 - 1).bfloat16()
        y, dx = torch.empty_like(x), torch.empty_like(x)

        def step():
            layer.forward(x, y)
            layer.backward(dy, dx)

        ms = time_steps(step, s, steps, warmup)
    del layer
    torch.cuda.empty_cache()
    return ms


def expert_parallel(fm, world, exchange, steps, warmup):
    w = fm.World(world)
    ms, errs = [0.0] * world, [None] * world
    barrier = threading.Barrier(world)

    def body(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                layer = fm.MoELayer(fm.MoEConfig(N, D, H, K, EL, world, SEED), rank=r, dtype=torch.bfloat16)
                layer.join(w)
                layer.set_ep_exchange(exchange)
                g = torch.Generator(device="cuda").manual_seed(100 + r)
                x = (torch.rand(N, D, device="cuda", generator=g) * 2 - 1).bfloat16()
                dy = (torch.rand(N, D, device="cuda", generator=g) * 2 - 1).bfloat16()
                y, dx = torch.empty_like(x), torch.empty_like(x)

                def step():
                    layer.forward(x, y)
                    layer.backward(dy, dx)

                for _ in range(warmup):
                    step()
                s.synchronize()
                barrier.wait()
                ms[r] = time_steps(step, s, steps, 0)
                s.synchronize()
                barrier.wait()
                del layer
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    for e in errs:
        if e is not None:
            raise e
    torch.cuda.empty_cache()
    return max(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg3", choices=["cfg3", "cfg2"])
    a = ap.parse_args()
    global N, D, H, EL
    if a.workload == "cfg2":  # 65536 tokens per rank, 64 experts in total
        N, D, H, EL = 65536, 1024, 4096, 64 // a.world
    import paper_2103_13262_b200 as fm

    torch.cuda.set_device(0)
    tokens = N * a.world
    base = single(fm, a.world, a.steps, a.warmup)
    fused = expert_parallel(fm, a.world, "peer", a.steps, a.warmup)
    trans = expert_parallel(fm, a.world, "transport", a.steps, a.warmup)
    print(json.dumps({
        "what": f"{a.workload} slices (d={D}, h={H}, {EL} experts and {N} tokens per rank, top-2) as {a.world} ranks "
                "sharing one B200 vs one worker with all experts and tokens; fwd+bwd per step",
        "world": a.world, "steps": a.steps,
        "single_worker_ms": base, "single_worker_tokens_per_s": tokens / base * 1e3,
        "ep_fused_ms": fused, "ep_fused_tokens_per_s": tokens / fused * 1e3,
        "ep_fused_overhead": fused / base - 1.0,
        "ep_transport_ms": trans, "ep_transport_tokens_per_s": tokens / trans * 1e3,
        "ep_transport_overhead": trans / base - 1.0,
    }))


if __name__ == "__main__":
    main()
