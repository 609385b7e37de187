# bench.py's N>1 code path on a one-GPU box: W ranks under torchrun, all on
# cuda:0 (--shared-gpu: gloo plumbing, fused peer exchange over CUDA IPC).
# Checks the multi-rank bench (barrier, max over ranks, EP step, e2e) runs and
# prints its line; the numbers are W ranks sharing one GPU, not scaling.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
port=29611
for spec in "2 cfg2" "4 cfg2" "2 cfg3" "2 cfg4" "2 cfg5"; do
  set -- $spec
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $1 --workload $2 --steps 5 --warmup 3 --shared-gpu \
    > gpurun_out/shared_w$1_$2.json 2> gpurun_out/shared_w$1_$2.err
  echo "w=$1 $2 exit $?" >> gpurun_out/shared.log
  port=$((port + 1))
done
