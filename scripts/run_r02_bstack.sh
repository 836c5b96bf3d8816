# 4-GPU A/B of the backward stacked tails (FCPB_BWD_STACK) on C2 at N=2 and N=4, plus N=1.
T=${T:-r02b}
for n in 2 4; do
  N=$n CFG=c2 STEPS=30 bash scripts/ab_multi.sh ${T}_n$n "st=FCPB_BWD_STACK=1 nost=FCPB_BWD_STACK=0"
done
for v in 1 0; do
  FCPB_BWD_STACK=$v FCPB_FWD_STACK=$v timeout 600 python bench.py --steps 30 --no-cpu --no-e2e > gpurun_out/${T}_n1_$v.log 2>&1
  python scripts/bench_summary.py gpurun_out/${T}_n1_$v.log
done
