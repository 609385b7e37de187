cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2 3 4; do
  for v in A P0; do
    if [ $v = P0 ]; then export FMOE_PDL=0; else unset FMOE_PDL; fi
    timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 20 > gpurun_out/e2e_${v}_$r.json 2>/dev/null
    python -c "import json; l=json.loads(open('gpurun_out/e2e_${v}_$r.json').read().strip().splitlines()[-1]); print('$v', $r, round(l['value']/1e6,3), round(l['e2e']['value']/1e6,3), round(l['e2e']['training_loop']['value']/1e6,3), l['clocks']['gemm_sm_mhz_effective'])" >> gpurun_out/e2e_ab.log
  done
done
