cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 --timeout-method thread -rf -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --workload cfg5 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
bash tools/gpu_ncu_cublas.sh
