# 2-GPU: copy-engine pulls alone vs beside a GEMM that fills every SM (can the forward's
# local tiles hide copy-engine pulls?).
T=${T:-r02c}
for c in "c2 4 5" "c3 2 2"; do
  set -- $c
  for b in "" "--busy"; do
    timeout 300 python scripts/nvlink_ncu_probe.py --config $1 --world $2 --reps $3 --mode ce $b > gpurun_out/${T}_$1_ce$b.log 2>&1
    echo "$1 ce $b rc=$?"; tail -1 gpurun_out/${T}_$1_ce$b.log | cut -c1-420
  done
done
