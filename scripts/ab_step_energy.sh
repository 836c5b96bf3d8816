# Whole-step A/B under the power cap: bench.py with library variants (FCPB_LIB), interleaved,
# reporting ms/step, SM clock and NVML energy per step.   bash scripts/ab_step_energy.sh TAG "a=lib b=lib" [reps]
TAG=$1; VARIANTS=$2; REPS=${3:-2}
for r in $(seq 1 $REPS); do
  for kv in $VARIANTS; do
    name=${kv%%=*}; lib=${kv#*=}; [ "$lib" = default ] && lib=""
    FCPB_LIB=$lib timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/${TAG}_${name}_$r.json 2>/dev/null
    python -c "
import json,sys; d=json.load(open('gpurun_out/${TAG}_${name}_$r.json'))
print('$name', '$r', round(d['ms_per_step'],3), int(d['value']), d['clocks']['sm_mhz'], d['energy']['j_per_step'], d['energy']['power_w_avg'], {k: round(v['ms'],3) for k,v in d['kernels'].items()})"
  done
done
