# compute-sanitizer synccheck / racecheck over the round-2 code paths: the
# overlapped EP exchange (push kernel, arrival flags, threads-as-ranks), the
# FMOE_F32 bf16x6 GEMMs, the drop-in's device route, the gathered A-loads.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 python -m pytest \
    tests/test_gpu_ep.py tests/test_gpu_parity.py -q -k "f32 or ep or fused or overlap" > gpurun_out/$tool.log 2>&1
  echo "exit $?" >> gpurun_out/$tool.log
done
