cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in ${REPEAT:-1}; do
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -rf ${PYTEST_ARGS} > gpurun_out/pytest_gpu$i.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu$i.log
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
