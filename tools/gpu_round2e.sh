cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ep_procs.py tests/test_gpu_ep.py tests/test_gpu_bench.py -q --timeout 600 --timeout-method thread -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --shared-gpu --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_shared2.json 2> gpurun_out/bench_shared2.err
SKIP=69 COUNT=23 bash tools/gpu_profile.sh
