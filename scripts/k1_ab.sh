# K1 A/B on one GPU: forward parity subset, MUFU-per-warp micro, per-kernel event times and
# ncu cycles of the in-tree library against dbg/libfcpb_old.so.   bash scripts/k1_ab.sh TAG
TAG=${1:-k1}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "forward or full_mask or c1_lengths or resume or simulated_ranks_ragged or c2_llama8b" > gpurun_out/${TAG}_pt.log 2>&1; tail -2 gpurun_out/${TAG}_pt.log
[ -x scripts/micro/mufu_warps ] && timeout 120 scripts/micro/mufu_warps > gpurun_out/${TAG}_mufu.log 2>&1; cat gpurun_out/${TAG}_mufu.log
KERNELS=fwd bash scripts/ab_cycles.sh ${TAG} "new=default old=dbg/libfcpb_old.so"
for v in new old; do cat gpurun_out/${TAG}_${v}_time.json; grep -E "attn_fwd" gpurun_out/${TAG}_${v}_ncu.csv | grep -E "cycles_elapsed|tensor|xu" | awk -F'","' '{print $(NF-2), $NF}' | sort -u; done
