# ncu --set full (+ source) of the latency-bound small kernels of one cfg2 step:
# the gate GEMM (first tc_gemm launch of a step), gate d_wg (9th) and the d_b2 column sums.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 27 -c 1 \
  -o gpurun_out/prof_gate -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_gate.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 35 -c 1 \
  -o gpurun_out/prof_dwg -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_dwg.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_colsum -s 3 -c 1 \
  -o gpurun_out/prof_colsum -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_colsum.log 2>&1
