# Final-build checks: compute-sanitizer memcheck over the GPU suite (minus the
# multi-GB cfg5 case), racecheck of the gate (staged bulk score stores) and
# layer tests, the reference arm and the default bench with their wall times.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
s=$(date +%s); timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err
echo "reference arm (steps 20 warmup 5) wall $(( $(date +%s) - s )) s" >> gpurun_out/walltimes.log
s=$(date +%s); timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "default bench wall $(( $(date +%s) - s )) s" >> gpurun_out/walltimes.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 99 --print-limit 20 python -m pytest \
  tests/test_gpu_parity.py -q -k "gate_bf16 or layer_bf16_vs_oracle" > gpurun_out/racecheck.log 2>&1
echo "exit $?" >> gpurun_out/racecheck.log
bash tools/gpu_memcheck.sh
