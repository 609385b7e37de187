cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_checkpoint.py tests/test_gpu_cli.py tests/test_dropin.py -v --timeout 250 --timeout-method thread > gpurun_out/new.log 2>&1
echo "exit $?" >> gpurun_out/new.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --timeout-method thread -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
bash tools/gpu_profile.sh
