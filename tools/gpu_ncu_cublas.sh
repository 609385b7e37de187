# ncu --set full of our expert GEMMs (fc2, wgrad_fc1 of the 2nd step) next to
# cuBLAS kernels of the same shapes and the 8192^3 peak shape.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 9 -c 9 \
  -o gpurun_out/prof_ours -f python tools/ncu_vs_cublas.py > gpurun_out/ncu_ours.log 2>&1
echo "ours exit $?" >> gpurun_out/ncu_ours.log
timeout 1200 ncu --set full --clock-control none --nvtx --nvtx-include "cublas/" -c 3 \
  -o gpurun_out/prof_cublas -f python tools/ncu_vs_cublas.py > gpurun_out/ncu_cublas.log 2>&1
echo "cublas exit $?" >> gpurun_out/ncu_cublas.log
