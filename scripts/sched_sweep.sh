for cfg in "0,0,0 lpt" "0,1,0 lpt" "1,1,1 lpt" "0,1,1 lpt" "0,1,0 seq" "0,0,0 seq"; do
  set -- $cfg
  FCPB_SCHED=$1 FCPB_ORDER=$2 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 > gpurun_out/s.json
  python -c "import json; d=json.load(open('gpurun_out/s.json')); print('$1 $2', round(d['ms_per_step'],2), {k:round(v['ms'],3) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done
