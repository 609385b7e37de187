# Same-box interleaved A/B of variants given as NAME=LIB[,ENV=VAL...] (LIB "-" =
# the in-tree library), printing every stage:
#   bash tools/gpu_ab2.sh "A=- B=paper_2103_13262_b200/_ab/libB.so I=-,FMOE_WGRAD_ORDER=interleave" "cfg2 cfg5" ROUNDS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARS=${1:-"A=-"}; WLS=${2:-"cfg2"}; ROUNDS=${3:-3}
for r in $(seq $ROUNDS); do
  for wl in $WLS; do
    for spec in $VARS; do
      name=${spec%%=*}; rest=${spec#*=}; lib=${rest%%,*}; envs=""
      [ "$rest" != "$lib" ] && envs=$(echo ${rest#*,} | tr ',' ' ')
      libenv=""; [ "$lib" != "-" ] && libenv="FMOE_B200_LIB=$PWD/$lib"
      steps=20; [ $wl = cfg4 ] && steps=5
      env $libenv $envs timeout 600 python bench.py --workload $wl --steps $steps --warmup 3 --no-cpu-baseline \
        --e2e-steps 3 > gpurun_out/ab_${name}_${wl}_$r.json 2>> gpurun_out/ab.err
      python - "$name" "$wl" "$r" gpurun_out/ab_${name}_${wl}_$r.json >> gpurun_out/ab.log <<'PY'
import json, sys
v, wl, r, f = sys.argv[1:]
try:
    l = json.loads(open(f).read().strip().splitlines()[-1])
    s = l["stages_ms"]
    e2e = (l.get("e2e") or {}).get("value")
    print(f"{wl} r{r} {v}: {l['value']/1e6:.3f}M ms={l['ms_per_step']:.3f} gemm_mhz={l['clocks'].get('gemm_sm_mhz_effective')} "
          + (f"e2e={e2e/1e6:.3f}M " if e2e else "")
          + " ".join(f"{k}={1000*x:.1f}" for k, x in s.items()))
except Exception as e:
    print(f"{wl} r{r} {v}: failed {e}")
PY
    done
  done
done
