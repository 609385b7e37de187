cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ep_procs.py tests/test_gpu_ep.py tests/test_gpu_parity.py tests/test_gpu_bench.py -q --timeout 600 --timeout-method thread -rf -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --shared-gpu --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_shared2.json 2> gpurun_out/bench_shared2.err
timeout 1200 ncu --set full --clock-control none --nvtx --nvtx-include "cublas/" -c 3 \
  -o gpurun_out/prof_cublas -f python tools/ncu_vs_cublas.py > gpurun_out/ncu_cublas.log 2>&1
echo "cublas exit $?" >> gpurun_out/ncu_cublas.log
