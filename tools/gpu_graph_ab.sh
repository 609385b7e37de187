# Timed-region variants on one box, interleaved: captured graph vs eager, with and
# without the stage marks / clock probe (--no-marks: experiment only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2 3; do
  for m in graph eager graphnm eagernm; do
    case $m in graph) extra="";; eager) extra="--eager";; graphnm) extra="--no-marks";; eagernm) extra="--eager --no-marks";; esac
    timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 $extra > gpurun_out/g_${m}_$r.json 2>>gpurun_out/g.err
    python -c "import json,sys; l=json.loads(open('gpurun_out/g_${m}_$r.json').read().strip().splitlines()[-1]); s=l['stages_ms']; print('$m', $r, round(l['ms_per_step'],3), round(l['ms_per_step_stddev'],3), l['gpu_launches'], l['clocks'].get('gemm_sm_mhz_effective'), ' '.join(f'{k}={1000*v:.1f}' for k,v in s.items()))" >> gpurun_out/g.log 2>>gpurun_out/g.err
  done
done
