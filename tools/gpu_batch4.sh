cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_ep.py tests/test_gpu_ep_procs.py tests/test_gpu_train.py -v -x --timeout 200 --timeout-method thread > gpurun_out/ep.log 2>&1
echo "exit $?" >> gpurun_out/ep.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
