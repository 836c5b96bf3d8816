# Round profile capture (1 GPU): bench lines, ncu launch list, ncu --set full of the attention kernels.
#   R=r02 bash scripts/profile_round.sh
set -x
R=${R:-r02}
timeout 900 python bench.py > gpurun_out/${R}_bench_c2_n1.json 2> gpurun_out/${R}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_reference_c2_n1.json 2> gpurun_out/${R}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_c2_n1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${R}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"attn_(fwd|bwd|dq|dqg)_kernel" -s 3 -c 3 \
  -o gpurun_out/${R}_full python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/${R}_ncu_full.log 2>&1
ncu -i gpurun_out/${R}_full.ncu-rep --page raw --csv > gpurun_out/${R}_ncu_full_raw_c2_n1.csv 2>/dev/null
tail -c 600 gpurun_out/${R}_bench_c2_n1.json
