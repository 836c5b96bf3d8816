# C2 bench A/B of environment variants at N=2 and N=4 on a 4-GPU box, interleaved twice.
#   bash scripts/ab_multi_env.sh TAG "name=ENV=VAL;ENV2=VAL ..."  (";" separates variables)
TAG=$1; VARIANTS=$2
P=29800
for r in 1 2; do
  for n in 2 4; do
    for kv in $VARIANTS; do
      name=${kv%%=*}; envs=${kv#*=}; [ "$envs" = base ] && envs=""
      P=$((P+1))
      env $(echo $envs | tr ";" " ") timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
        --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --steps 20 --warmup 5 --no-cpu --no-e2e \
        > gpurun_out/${TAG}_${name}_n${n}_$r.log 2>&1
      echo "$name n$n r$r $(python scripts/bench_summary.py gpurun_out/${TAG}_${name}_n${n}_$r.log | cut -d: -f2-)"
    done
  done
done
