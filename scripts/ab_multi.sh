# Multi-GPU A/B of an env knob on bench.py (torchrun, N = number of visible GPUs).
# usage: N=4 CFG=c2 STEPS=20 bash scripts/ab_multi.sh TAG "name1=ENV=val ..." 
TAG=$1; VARIANTS=$2; N=${N:-2}; CFG=${CFG:-c2}; STEPS=${STEPS:-20}
P=29700
for rep in 1 2; do
for kv in $VARIANTS; do
  name=${kv%%=*}; envs=${kv#*=}
  P=$((P+1))
  env ${envs//,/ } timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $P bench.py --gpus $N --steps $STEPS --config $CFG --no-e2e > gpurun_out/${TAG}_${name}_${rep}.log 2>&1
  python scripts/bench_summary.py gpurun_out/${TAG}_${name}_${rep}.log
done
done
