# Forward kernel A/B against the same-box library yardstick (CuTe-DSL sm100 FA4-style flash
# attention in vllm), C2 N=1: CUDA-event times back to back, then ncu clock-independent cycles,
# tensor-pipe and XU (MUFU) activity of both forward kernels on the same inputs.
#   bash scripts/fwd_vs_fa4_cycles.sh TAG
TAG=${1:-fa4cmp}
M=sm__cycles_elapsed.max,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,smsp__cycles_active.avg
timeout 300 python scripts/kbench.py --reps 10 --kernels fwd > gpurun_out/${TAG}_ours_time.json 2>&1
timeout 300 python scripts/yardstick_fa4.py --steps 10 > gpurun_out/${TAG}_fa4_time.json 2>&1
timeout 600 ncu --metrics $M -k regex:"attn_fwd_kernel" -c 3 --csv python scripts/kbench.py --reps 2 --kernels fwd \
  > gpurun_out/${TAG}_ours_ncu.csv 2>&1
timeout 600 ncu --metrics $M -k regex:"[Ff]wd|Forward" -c 3 --csv python scripts/yardstick_fa4.py --steps 1 \
  > gpurun_out/${TAG}_fa4_ncu.csv 2>&1
python - "$TAG" <<'EOF'
import csv, sys, io, collections
tag = sys.argv[1]
for who in ("ours", "fa4"):
    txt = open(f"gpurun_out/{tag}_{who}_ncu.csv").read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:]))) if i >= 0 else []
    agg = collections.defaultdict(dict)
    for r in rows:
        agg[(r["ID"], r["Kernel Name"][:60])][r["Metric Name"]] = r["Metric Value"]
    for (i_, k), m in agg.items():
        print(who, i_, k, {a.split("__")[1][:28]: b for a, b in m.items()})
EOF
