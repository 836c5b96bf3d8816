# One `ncu --set full --import-source on` capture of one attention kernel on C2 N=1
# (scripts/kbench.py), with its raw metrics and per-SASS-line source page (stall reasons).
# usage: bash scripts/ncu_kernel_full.sh TAG KERNEL(fwd|bwd|dq) [lib]
TAG=$1; K=$2; LIB=${3:-}
case $K in fwd) RX=attn_fwd_kernel;; bwd) RX=attn_bwd_kernel;; dq) RX="attn_dqg?_kernel";; esac
FCPB_LIB=$LIB timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$RX" -s 1 -c 1 \
  -o gpurun_out/${TAG}_${K} python scripts/kbench.py --kernels $K --reps 1 > gpurun_out/${TAG}_${K}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}_${K}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${K}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_${K}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${K}_source.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_${K}.ncu-rep --page details --csv > gpurun_out/${TAG}_${K}_details.csv 2>/dev/null
ls -la gpurun_out/${TAG}_${K}*
