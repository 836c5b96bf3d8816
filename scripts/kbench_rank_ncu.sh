# kbench_rank.py for C2 at N=1/2/4 (rank 0), event times then ncu cycles (elapsed max vs active
# average = the launch tail).   bash scripts/kbench_rank_ncu.sh TAG
TAG=${1:-kr}
M=sm__cycles_elapsed.max,sm__cycles_active.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for n in 1 2 4; do
  timeout 300 python scripts/kbench_rank.py --world $n --rank 0 > gpurun_out/${TAG}_n${n}_time.json 2>&1
  tail -1 gpurun_out/${TAG}_n${n}_time.json
  timeout 600 ncu --metrics $M -k regex:"attn_(fwd|bwd|dqg|dq)_kernel" --csv python scripts/kbench_rank.py --world $n --rank 0 --reps 2 \
    > gpurun_out/${TAG}_n${n}_ncu.csv 2>&1
  python scripts/ncu_cycles.py gpurun_out/${TAG}_n${n}_ncu.csv | tail -1
done
