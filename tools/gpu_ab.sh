# Same-box A/B of library variants (paper_2103_13262_b200/_ab/lib*.so, built with
# make -C paper_2103_13262_b200/csrc OBJ=... OUT=... EXTRA=-D...), interleaved
# so clock drift under the power cap hits every variant alike.
#   bash tools/gpu_ab.sh "B C" "cfg2 cfg4" ROUNDS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARS=${1:-"B"}; WLS=${2:-"cfg2"}; ROUNDS=${3:-3}
for v in $VARS; do
  FMOE_B200_LIB=$PWD/paper_2103_13262_b200/_ab/lib$v.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -q -x \
    > gpurun_out/ab_tests_$v.log 2>&1; echo "tests $v exit $?" >> gpurun_out/ab.log
done
for r in $(seq $ROUNDS); do
  for wl in $WLS; do
    for v in A $VARS; do
      if [ $v = A ]; then unset FMOE_B200_LIB; else export FMOE_B200_LIB=$PWD/paper_2103_13262_b200/_ab/lib$v.so; fi
      steps=20; [ $wl = cfg4 ] && steps=5
      timeout 600 python bench.py --workload $wl --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 3 \
        > gpurun_out/ab_${v}_${wl}_$r.json 2>> gpurun_out/ab.err
      python - "$v" "$wl" "$r" gpurun_out/ab_${v}_${wl}_$r.json >> gpurun_out/ab.log <<'PY'
import json, sys
v, wl, r, f = sys.argv[1:]
try:
    l = json.loads(open(f).read().strip().splitlines()[-1])
    s = l["stages_ms"]
    print(f"{wl} r{r} {v}: {l['value']/1e6:.3f}M ms={l['ms_per_step']:.3f} sm={l['clocks'].get('sm_mhz')} "
          + " ".join(f"{k}={s[k]:.3f}" for k in ("fc1", "fc2", "dgrad_fc2", "dgrad_fc1", "wgrad_fc2", "wgrad_fc1")))
except Exception as e:
    print(f"{wl} r{r} {v}: failed {e}")
PY
    done
  done
done
unset FMOE_B200_LIB
