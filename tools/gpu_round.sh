# Full round check on one B200: gpu tests, smoke, default bench (with cpu_baseline),
# reference arm, and the extra BASELINE workloads (WORKLOADS="cfg4 cfg5").
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -rf ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
for w in ${WORKLOADS}; do
timeout 900 python bench.py --workload $w --steps ${WL_STEPS:-10} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
echo "bench $w exit $?" >> gpurun_out/bench_$w.err
done
if [ -z "$NO_REF" ]; then
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref exit $?" >> gpurun_out/bench_ref.err
fi
