# 2-GPU run: NVLink counters of the K5 pulls (copy engine under ncu range replay, the pull
# kernel under ncu kernel replay), plain GB/s of both, and C3/C4 at N=2 with each transport.
T=${T:-r02q}
for m in ce sm; do
  for c in "c3 2" "c2 4"; do
    set -- $c
    timeout 300 python scripts/nvlink_ncu_probe.py --config $1 --world $2 --mode $m > gpurun_out/${T}_nvprobe_$1_$m.log 2>&1
    echo "probe_$1_$m=$?"; tail -1 gpurun_out/${T}_nvprobe_$1_$m.log | cut -c1-400
  done
done
M=nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum
timeout 900 ncu --replay-mode range --metrics $M --csv \
  python scripts/nvlink_ncu_probe.py --config c3 --world 2 --reps 1 --mode ce > gpurun_out/${T}_nvprobe_ncu_range_ce.log 2>&1
echo "ncu_range_ce=$?"; grep -v "^==PROF==" gpurun_out/${T}_nvprobe_ncu_range_ce.log | tail -8
timeout 900 ncu --kernel-name regex:gather --launch-skip 1 --launch-count 1 --metrics $M,dram__bytes_write.sum --csv \
  python scripts/nvlink_ncu_probe.py --config c3 --world 2 --reps 1 --mode sm > gpurun_out/${T}_nvprobe_ncu_kernel_sm.log 2>&1
echo "ncu_kernel_sm=$?"; grep -v "^==PROF==" gpurun_out/${T}_nvprobe_ncu_kernel_sm.log | tail -8
for c in c3 c4; do
  N=2 CFG=$c STEPS=3 bash scripts/ab_multi.sh ${T}_${c}_n2 "sm=FCPB_PULL=sm ce=FCPB_PULL=ce"
done
