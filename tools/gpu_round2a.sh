# Round-2 first look: GPU suite, smoke, default bench, GEMM-vs-cuBLAS calibration.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 --timeout-method thread -rf -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/gemm_calib.py > gpurun_out/gemm_calib.jsonl 2> gpurun_out/gemm_calib.err
