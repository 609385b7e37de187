# ncu evidence for profiles/: launch list of one bench step + full capture of the grouped GEMMs.
# One bf16 step = 21 launches of ours (9 of them tc_gemm); bench runs 3 warm-up steps first
# (torch's input-generation kernels are filtered out by the namespace).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=${NCU:-ncu}
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --kernel-name-base demangled -k regex:fmoe_b200 -s ${SKIP:-63} -c ${COUNT:-21} --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_bench.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch_bench.log
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:tc_gemm -s ${TC_SKIP:-27} -c ${TC_COUNT:-9} \
  -o gpurun_out/prof_tc -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_full.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full.log
