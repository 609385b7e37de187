cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 600 --timeout-method thread -rf -x -k "wide or layer_bf16" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q --timeout 900 --timeout-method thread -rf -x > gpurun_out/pytest_full.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_full.log
for i in 1 2; do
for m in 0 58 63; do
FMOE_TC_WIDE=$m timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_w$m.$i.json 2> gpurun_out/bench_w$m.$i.err
done
done
