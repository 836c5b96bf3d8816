# One bench line per (config, N) for simulator validation -> gpurun_out/configs.jsonl
out=${OUT:-gpurun_out/configs.jsonl}; : > $out
run() {  # config n steps [block]
  if [ "$2" = 1 ]; then cmd="python bench.py"; else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $2"; fi
  extra=""; [ -n "$4" ] && extra="--block $4"
  timeout 900 $cmd --config $1 --steps $3 --no-cpu --no-e2e $extra 2>/dev/null | tail -1 >> $out
}
for n in 1 2 4; do run c2 $n 30; done
for n in 1 2 4; do run c4 $n 4; done
for b in 1024 2048 4096 6144; do run c5 1 10 $b; done
for n in 1 2 4; do run c3 $n 4; done
wc -l $out
