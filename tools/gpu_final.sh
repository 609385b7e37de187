# Round evidence on one B200: gpu tests, smoke, ncu launch list + GEMM capture,
# bench (default, with the CPU baseline), the reference arm, cfg1 / cfg3 / cfg4 / cfg5 lines
# (+ the reference arm at the full cfg1).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 --timeout-method thread -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
bash tools/gpu_profile.sh
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for w in cfg5 cfg4 cfg3 cfg1; do
timeout 900 python bench.py --workload $w --steps 10 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 900 python bench.py --impl reference --workload cfg1 --steps 3 --warmup 1 > gpurun_out/bench_ref_cfg1.json 2> gpurun_out/bench_ref_cfg1.err
