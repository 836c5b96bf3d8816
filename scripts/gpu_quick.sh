# quick GPU check: parity, cycle-level trace medians, 3 short bench runs
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
NPRINT=${NPRINT:-0} NPRINT2=${NPRINT2:-0} NPRINT3=${NPRINT3:-0} timeout 300 python scripts/trace_bwd.py > gpurun_out/tr.log 2>&1; grep -E "median|step" gpurun_out/tr.log
for i in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e 2>gpurun_out/b$i.err | tail -1 > gpurun_out/b$i.json
  python -c "import json,sys; d=json.load(open('gpurun_out/b$i.json')); print(round(d['ms_per_step'],2), int(d['value']), {k:round(v['ms'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
