# round 2g: FMOE_F32 on the tensor cores (bf16x3) -- GPU suite, cfg2 / cfg1 bench lines, reference arm at cfg1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -rf -x -k "f32" > gpurun_out/pytest_f32.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_f32.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 900 python bench.py --workload cfg1 --steps 20 --warmup 5 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
FMOE_F32_SIMT=1 timeout 900 python bench.py --workload cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1_simt.json 2> gpurun_out/bench_cfg1_simt.err
timeout 900 python bench.py --impl reference --workload cfg1 --steps 20 --warmup 5 > gpurun_out/bench_cfg1_ref.json 2> gpurun_out/bench_cfg1_ref.err
