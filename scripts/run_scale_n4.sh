# Multi-GPU check on a 4-GPU box: the NCCL multi-rank parity tests, then the driver's scaling
# commands for C2 at N=1, 2, 4 (same flags as the driver: --steps 20 --warmup 5).
T=${T:-r02s}
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q -p no:cacheprovider -k nccl_parity > gpurun_out/${T}_mr.log 2>&1
echo "multirank=$?"; tail -1 gpurun_out/${T}_mr.log
P=29700
for n in 1 2 4; do
  P=$((P+1))
  if [ $n = 1 ]; then
    timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_n$n.log 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $P bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/${T}_n$n.log 2>&1
  fi
  echo "n$n=$?"; python scripts/bench_summary.py gpurun_out/${T}_n$n.log
done
