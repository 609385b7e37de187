# One GPU call: new multi-process EP test, full gpu suite, bench, cfg4, ncu of fc1/fc2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_ep_procs.py -v -x --timeout 250 --timeout-method thread > gpurun_out/procs.log 2>&1
echo "exit $?" >> gpurun_out/procs.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method thread --deselect tests/test_gpu_ep_procs.py::test_ep_two_processes_peer_memory > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload cfg4 --steps 10 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
TAG=fc12 bash tools/gpu_ncu_gemm.sh
