# 4-GPU run: received-group A/B on C2 at N=2 and N=4, cross-GPU multi-rank parity, and the
# NVLink counter capture of the K5 pulls (scripts/nvlink_ncu_probe.py, one process, 2 GPUs).
T=${T:-r02g}
timeout 1200 python -m pytest tests/test_gpu_multirank.py -x -q -s -p no:cacheprovider -k nccl_parity > gpurun_out/${T}_mr_4gpu.log 2>&1
echo "mr4=$?"; grep -E "passed|failed" gpurun_out/${T}_mr_4gpu.log
for n in 2 4; do
  N=$n CFG=c2 STEPS=30 bash scripts/ab_multi.sh ${T}_n$n "grp=FCPB_RECV_GROUPS=1 nogrp=FCPB_RECV_GROUPS=0"
done
timeout 300 python scripts/nvlink_ncu_probe.py --config c3 --world 2 > gpurun_out/${T}_nvprobe_plain.log 2>&1
echo "probe=$?"; tail -2 gpurun_out/${T}_nvprobe_plain.log
M=nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum
timeout 900 ncu --replay-mode range --profile-from-start off --metrics $M --csv \
  python scripts/nvlink_ncu_probe.py --config c3 --world 2 --reps 1 > gpurun_out/${T}_nvprobe_ncu_range.log 2>&1
echo "ncu_range=$?"; tail -8 gpurun_out/${T}_nvprobe_ncu_range.log
timeout 900 ncu --replay-mode app-range --profile-from-start off --metrics $M --csv \
  python scripts/nvlink_ncu_probe.py --config c3 --world 2 --reps 1 > gpurun_out/${T}_nvprobe_ncu_apprange.log 2>&1
echo "ncu_apprange=$?"; tail -8 gpurun_out/${T}_nvprobe_ncu_apprange.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 \
  scripts/nvlink_exchange.py --config c2 --reps 20 > gpurun_out/${T}_nvlink_c2_n4.log 2>&1
echo "nv_c2=$?"; tail -1 gpurun_out/${T}_nvlink_c2_n4.log | cut -c1-600
