"""Summarise ncu output from gpurun_out/ into profiles/ (committed evidence).

  python tools/summarize_ncu.py <round-tag>

Reads gpurun_out/launches.csv (per-launch gpu__time_duration + DRAM bytes of
one bench step, `tools/gpu_profile.sh`) and gpurun_out/prof_tc.ncu-rep (full
capture of the grouped GEMM launches) and writes
  profiles/<tag>_launches.md      per-kernel share of one fwd+bwd step
  profiles/<tag>_tc_gemm_full.md  key metrics of the expert GEMM launches
  profiles/ncu_traffic.json       DRAM bytes per grouped-GEMM launch (bench.py `traffic`)
"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

# issue order of one bf16 single-GPU step (layer.cu): data gradients first
STEP_ORDER = ["gate", "plan_hist", "plan_colscan", "plan_offsets", "plan_rank", "scatter", "fc1", "fc2", "gather_combine",
              "gcb", "dgrad_fc2", "dgrad_fc1", "gate_dx", "scatter_bwd", "wgrad_order", "wgrad_fc2", "db2_colsum",
              "db1_db2_reduce", "wgrad_fc1", "gate_dwg", "gate_dwg_reduce"]


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    return n.replace("fmoe_b200::", "").replace("tc::", "")


def launches(tag):
    rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    h = {k: i for i, k in enumerate(hdr)}
    per = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = int(r[h["ID"]])
        d = per.setdefault(key, {"name": short(r[h["Kernel Name"]]), "grid": r[h["Grid Size"]]})
        d[r[h["Metric Name"]]] = float(r[h["Metric Value"]].replace(",", ""))
    ids = sorted(per)
    # one step = the launches starting at the first gate GEMM (tc_gemm_kernel<64|128|256, 0, 1, 1, 3>)
    first = next(i for i in ids if "tc_gemm_kernel<" in per[i]["name"] and per[i]["name"].endswith(", 3>"))
    # the capture window may start mid-step: rotate so it starts at a gate launch
    # (consecutive steps launch the same sequence)
    after = [per[i] for i in ids if i >= first]
    before = [per[i] for i in ids if i < first]
    extra = len(ids) - len(STEP_ORDER)  # a window longer than a step repeats its first launches
    step = (after + (before[extra:] if 0 < extra <= len(before) else before))[:len(STEP_ORDER)]
    total = sum(s["gpu__time_duration.sum"] for s in step)
    lines = [f"# {tag}: kernel launches of one bench step (cfg2, ncu --clock-control none, serialized)", "",
             "Command: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none python bench.py --steps 2 --warmup 3 --e2e-steps 1` (tools/gpu_profile.sh).  "
             "Per-launch times are cold-cache and serialized; compare shares, not absolutes.", "",
             "| # | stage | kernel | grid | time (us) | share | DRAM read (MB) | DRAM write (MB) |",
             "|---|---|---|---|---|---|---|---|"]
    for j, s in enumerate(step):
        t = s["gpu__time_duration.sum"] / 1e3
        lines.append(f"| {j} | {STEP_ORDER[j] if j < len(STEP_ORDER) else '?'} | `{s['name']}` | {s['grid']} | "
                     f"{t:.1f} | {100 * s['gpu__time_duration.sum'] / total:.1f}% | "
                     f"{s.get('dram__bytes_read.sum', 0) / 1e6:.1f} | {s.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")
    gemm = [s for j, s in enumerate(step) if STEP_ORDER[j] in ("fc1", "fc2", "dgrad_fc2", "wgrad_fc2", "dgrad_fc1", "wgrad_fc1")]
    gt = sum(s["gpu__time_duration.sum"] for s in gemm)
    lines += ["", f"Step total (serialized): {total / 1e3:.1f} us; grouped expert GEMM launches: {gt / 1e3:.1f} us "
              f"= {100 * gt / total:.1f}% of the step."]
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    traffic = sum(s.get("dram__bytes_read.sum", 0) + s.get("dram__bytes_write.sum", 0) for s in gemm) / max(len(gemm), 1)
    return gemm, traffic


def full(tag):
    rep = os.path.join(OUT, "prof_tc.ncu-rep")
    if not os.path.exists(rep):
        return None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    h = {k: i for i, k in enumerate(hdr)}
    keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
            "launch__grid_size", "launch__cluster_dim_x"]
    lines = [f"# {tag}: ncu --set full of the grouped tcgen05 GEMM launches of one step", "",
             "Command: `ncu --set full --clock-control none --import-source on -k regex:tc_gemm` on "
             "`bench.py --steps 1 --warmup 3` (tools/gpu_profile.sh).", "",
             "| launch | " + " | ".join(k.split(".")[0].replace("TPC", "tensor pipe (realtime)") + " "
                                      + k.split(".")[-1] for k in keys) + " |",
             "|---" * (len(keys) + 1) + "|"]
    for r in data:
        name = short(r[h["Kernel Name"]])
        vals = []
        for k in keys:
            v = r[h[k]] if k in h else ""
            u = units[h[k]] if k in h else ""
            vals.append(f"{v} {u}".strip())
        lines.append(f"| `{name}` | " + " | ".join(vals) + " |")
    open(os.path.join(PROF, f"{tag}_tc_gemm_full.md"), "w").write("\n".join(lines) + "\n")
    return len(data)


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    gemm, traffic = launches(tag)
    n = full(tag)
    json.dump({"round": tag, "tc_gemm_dram_bytes_per_launch": traffic,
               "note": "mean of dram__bytes_read.sum + dram__bytes_write.sum over the six expert GEMM launches "
                       "(fc1, fc2, dgrad fc2, wgrad fc2, dgrad fc1, wgrad fc1) of one step, ncu launch list"},
              open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    print("gemm launches", len(gemm), "traffic/launch", traffic, "full rows", n)


if __name__ == "__main__":
    main()
