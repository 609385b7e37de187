# ncu --set full of the cfg5 (Zipf) weight-gradient GEMMs (6 tc_gemm launches per routed step; the 4th step)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:tc_gemm -s 18 -c 6 \
  -o gpurun_out/prof_cfg5 -f python bench.py --workload cfg5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cfg5.log 2>&1
echo "exit $?" >> gpurun_out/ncu_cfg5.log
