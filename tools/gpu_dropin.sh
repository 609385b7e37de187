# drop-in: the reference's unit tests (device route), route-vs-composition tests, reference-API bench at cfg1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_dropin.py tests/test_gpu_parity.py -q --timeout 600 -rf -k "dropin or reference_unit or f32 or layer_f64" > gpurun_out/pytest_dropin.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_dropin.log
B=paper_2103_13262_b200/fmoe_bench
A="bench-local --api reference --n-b 8192 --d-m 1024 --d-h 4096 --k 2 --n-e 16 --reps 8 --warmup 2"
timeout 600 $B $A > gpurun_out/refapi_f64.csv 2>&1
FMOE_DROPIN_DTYPE=f32 timeout 600 $B $A > gpurun_out/refapi_f32.csv 2>&1
FMOE_DROPIN_DTYPE=bf16 timeout 600 $B $A > gpurun_out/refapi_bf16.csv 2>&1
FMOE_DROPIN_PATH=ops timeout 600 $B $A --reps 2 > gpurun_out/refapi_ops.csv 2>&1
