# 4-GPU evidence run (gpurun --gpus 4): multi-rank parity over NCCL across GPUs, bench lines
# for C2/C3/C4 at N=4, and the isolated exchange bandwidth at N=4.
T=${T:-r02}
timeout 1200 python -m pytest tests/test_gpu_multirank.py -x -q -s -p no:cacheprovider -k nccl_parity > gpurun_out/${T}_mr_4gpu.log 2>&1
echo "mr4=$?"; grep -E "passed|failed" gpurun_out/${T}_mr_4gpu.log
P=29600
for c in c2 c3 c4; do
  P=$((P+1))
  E=""; [ $c != c2 ] && E="--no-e2e"
  S=20; [ $c != c2 ] && S=3
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P \
    bench.py --gpus 4 --steps $S --config $c $E > gpurun_out/${T}_bench_${c}_n4.log 2>&1
  echo "$c=$?"; python scripts/bench_summary.py gpurun_out/${T}_bench_${c}_n4.log
done
for c in c3 c4; do
  P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P \
    scripts/nvlink_exchange.py --config $c --reps 10 > gpurun_out/${T}_nvlink_${c}_n4.log 2>&1
  echo "nv_$c=$?"
done
