# A/B of kernel cycles (clock-independent) and event times for library variants on one GPU.
# usage: bash scripts/ab_cycles.sh TAG "label1=libpath1 label2=libpath2 ..." [extra env]
TAG=$1; VARIANTS=$2
for kv in $VARIANTS; do
  name=${kv%%=*}; lib=${kv#*=}
  [ "$lib" = default ] && lib=""
  FCPB_LIB=$lib timeout 300 python scripts/kbench.py --reps 10 --kernels ${KERNELS:-fwd,bwd,dq} > gpurun_out/${TAG}_${name}_time.json 2>&1
  FCPB_LIB=$lib timeout 600 ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed \
    -k regex:"attn_(fwd|bwd|dqg|dq)_kernel" --csv python scripts/kbench.py --reps 3 --kernels ${KERNELS:-fwd,bwd,dq} > gpurun_out/${TAG}_${name}_ncu.csv 2>&1
done
