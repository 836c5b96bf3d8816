# 4-GPU: parity of the resumed forward (simulated ranks + 3 processes on one GPU), then the
# C2 A/B of FCPB_FUSE_REMOTE=resume (local wave || copy-engine pulls, remote wave continues
# the partials) against the default (one wave after the pull kernel) at N=2 and N=4.
T=${T:-r02r}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k resume > gpurun_out/${T}_parity.log 2>&1
echo "parity=$?"; tail -1 gpurun_out/${T}_parity.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q -p no:cacheprovider -k resumed > gpurun_out/${T}_mr.log 2>&1
echo "mr=$?"; tail -1 gpurun_out/${T}_mr.log
for n in 2 4; do
  N=$n CFG=c2 STEPS=30 bash scripts/ab_multi.sh ${T}_n$n "res=FCPB_FUSE_REMOTE=resume all=FCPB_FUSE_REMOTE=all"
done
