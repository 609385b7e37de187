# ncu --set full (+ source) of selected grouped-GEMM launches of one cfg2 step.
# tc_gemm launch order per step: gate, fc1, fc2, dgrad_fc2, dgrad_fc1, gate_dx,
# wgrad_fc2, wgrad_fc1, gate_dwg (9 per step); 3 warm-up steps -> skip 27.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s ${TC_SKIP:-28} -c ${TC_COUNT:-2} \
  -o gpurun_out/prof_${TAG:-tc} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_${TAG:-tc}.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_${TAG:-tc}.log
