# round 2h: FMOE_F32 bf16x6 parity, drop-in tests, cfg1 lines (C-ABI fp32, reference C++ API f64 via the drop-in)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -rf -k "f32" > gpurun_out/pytest_f32.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_f32.log
timeout 900 python -m pytest tests/test_dropin.py tests/test_gpu_train.py tests/test_gpu_cli.py -q --timeout 600 -rf > gpurun_out/pytest_dropin.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_dropin.log
timeout 900 python bench.py --workload cfg1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err
FMOE_F32_SIMT=1 timeout 900 python bench.py --workload cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1_simt.json 2> gpurun_out/bench_cfg1_simt.err
timeout 900 paper_2103_13262_b200/fmoe_bench bench-local --api reference --n-b 8192 --d-m 1024 --d-h 4096 --k 2 --n-e 16 --reps 3 --warmup 1 > gpurun_out/cli_cfg1_refapi.csv 2> gpurun_out/cli_cfg1_refapi.err
timeout 900 paper_2103_13262_b200/fmoe_bench bench-local --dtype f64 --n-b 8192 --d-m 1024 --d-h 4096 --k 2 --n-e 16 --reps 3 --warmup 1 > gpurun_out/cli_cfg1_f64.csv 2> gpurun_out/cli_cfg1_f64.err
timeout 900 paper_2103_13262_b200/fmoe_bench bench-local --dtype f32 --n-b 8192 --d-m 1024 --d-h 4096 --k 2 --n-e 16 --reps 10 --warmup 2 > gpurun_out/cli_cfg1_f32.csv 2> gpurun_out/cli_cfg1_f32.err
