# N=1 bench lines for C3/C4/C5 (block sweep) on one B200.
T=${T:-r02}
for c in c3 c4; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_${c}_n1.log 2>&1
  python scripts/bench_summary.py gpurun_out/${T}_bench_${c}_n1.log
done
for b in 1024 2048 4096 6144; do
  timeout 600 python bench.py --config c5 --block $b --steps 10 --no-cpu --no-e2e > gpurun_out/${T}_bench_c5_b${b}_n1.log 2>&1
  python scripts/bench_summary.py gpurun_out/${T}_bench_c5_b${b}_n1.log
done
