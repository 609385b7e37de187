# ncu --set full of the cfg4 weight-gradient GEMMs (128 experts on one GPU, ~256 rows each):
# the two wgrad launches of the first layer of the timed step (3 warm-up steps x 12 layers x 2 skipped)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:tc_gemm_kernel<.int.256, .bool.1, .bool.1, .int.[12], .int.2" -s 72 -c 1 \
  -o gpurun_out/prof_cfg4 -f python bench.py --workload cfg4 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/ncu_cfg4.log 2>&1
echo "exit $?" >> gpurun_out/ncu_cfg4.log
