# A/B: per-kernel duration / cycles / tensor-active for several builds of libfcpb (FCPB_LIB)
for lib in "$@"; do
  FCPB_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:attn_ -s 3 -c 3 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null \
    | python -c "
import csv,sys
lines=sys.stdin.read().split('\n'); s=[i for i,l in enumerate(lines) if l.startswith('\"ID\"')][0]
rows=list(csv.reader(lines[s:])); h=rows[0]
out={}
for r in rows[1:]:
    if len(r)<len(h): continue
    out.setdefault(r[h.index('Kernel Name')].split('(')[0], {})[r[h.index('Metric Name')].split('.')[0]]=r[h.index('Metric Value')]
print('$lib', {k:(round(float(v['gpu__time_duration'])/1e6,3), int(v['sm__cycles_elapsed'])//1000, v['sm__pipe_tensor_cycles_active']) for k,v in out.items()})
"
done
