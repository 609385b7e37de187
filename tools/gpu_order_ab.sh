# weight-gradient tile order A/B (FMOE_WGRAD_ORDER=desc|interleave), same box, interleaved runs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2 3; do
  for wl in ${WLS:-cfg5 cfg2}; do
    for o in desc interleave; do
      steps=10; [ $wl = cfg2 ] && steps=20
      FMOE_WGRAD_ORDER=$o timeout 600 python bench.py --workload $wl --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 3 \
        > gpurun_out/ord_${o}_${wl}_$r.json 2>> gpurun_out/ord.err
      python - "$o" "$wl" "$r" gpurun_out/ord_${o}_${wl}_$r.json >> gpurun_out/ord.log <<'PY'
import json, sys
v, wl, r, f = sys.argv[1:]
try:
    l = json.loads(open(f).read().strip().splitlines()[-1])
    s = l["stages_ms"]
    print(f"{wl} r{r} {v}: {l['value']/1e6:.3f}M ms={l['ms_per_step']:.3f} clk={l['clocks'].get('gemm_sm_mhz_effective')} "
          + " ".join(f"{k}={s[k]:.3f}" for k in ("fc1", "fc2", "dgrad_fc2", "dgrad_fc1", "wgrad_fc2", "wgrad_fc1")))
except Exception as e:
    print(f"{wl} r{r} {v}: failed {e}")
PY
    done
  done
done
