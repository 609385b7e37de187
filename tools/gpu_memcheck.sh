# compute-sanitizer memcheck over the GPU suite (minus the multi-GB cfg5 case)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1300 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest \
  tests/test_gpu_ep.py tests/test_gpu_workloads.py tests/test_gpu_edges.py tests/test_gpu_train.py \
  tests/test_gpu_parity.py tests/test_checkpoint.py tests/test_gpu_graph.py -q -k "not cfg5_full" \
  > gpurun_out/memcheck.log 2>&1
echo "exit $?" >> gpurun_out/memcheck.log
