# 4-GPU run: K5 pull kernel vs copy-engine pulls (C2 at N=2/4), parity of the pull kernel and
# of the executor at N>1 (shared-GPU and cross-GPU), and NVLink counters under ncu.
T=${T:-r02p}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -p no:cacheprovider -k gather > gpurun_out/${T}_gather_test.log 2>&1
echo "gather_test=$?"; tail -1 gpurun_out/${T}_gather_test.log
timeout 1500 python -m pytest tests/test_gpu_multirank.py -x -q -s -p no:cacheprovider > gpurun_out/${T}_mr.log 2>&1
echo "mr=$?"; grep -E "passed|failed" gpurun_out/${T}_mr.log
for n in 2 4; do
  N=$n CFG=c2 STEPS=30 bash scripts/ab_multi.sh ${T}_n$n "sm=FCPB_PULL=sm ce=FCPB_PULL=ce"
done
for m in ce sm; do
  timeout 300 python scripts/nvlink_ncu_probe.py --config c3 --world 2 --mode $m > gpurun_out/${T}_nvprobe_$m.log 2>&1
  echo "probe_$m=$?"; tail -1 gpurun_out/${T}_nvprobe_$m.log
  timeout 300 python scripts/nvlink_ncu_probe.py --config c2 --world 4 --mode $m > gpurun_out/${T}_nvprobe_c2_$m.log 2>&1
  echo "probe_c2_$m=$?"; tail -1 gpurun_out/${T}_nvprobe_c2_$m.log
done
M=nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum
timeout 900 ncu --replay-mode range --metrics $M --csv \
  python scripts/nvlink_ncu_probe.py --config c3 --world 2 --reps 1 --mode ce > gpurun_out/${T}_nvprobe_ncu_range_ce.log 2>&1
echo "ncu_range_ce=$?"; tail -6 gpurun_out/${T}_nvprobe_ncu_range_ce.log
timeout 900 ncu --kernel-name regex:gather --metrics $M,dram__bytes_write.sum --csv \
  python scripts/nvlink_ncu_probe.py --config c3 --world 2 --reps 1 --mode sm > gpurun_out/${T}_nvprobe_ncu_kernel_sm.log 2>&1
echo "ncu_kernel_sm=$?"; grep -v "^==PROF==" gpurun_out/${T}_nvprobe_ncu_kernel_sm.log | tail -8
