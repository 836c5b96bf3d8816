# 4-GPU A/B of K1 stacked tails (FCPB_FWD_STACK) on C2 at N=2 and N=4.
T=${T:-r02s}
for n in 2 4; do
  N=$n CFG=c2 STEPS=30 bash scripts/ab_multi.sh ${T}_n$n "st=FCPB_FWD_STACK=1 nost=FCPB_FWD_STACK=0"
done
