# A/B over environment settings (e.g. FCPB_SCHED=f,b,q): per-kernel ms / kcycles / tensor% / DRAM GB
for envs in "$@"; do
  env $envs timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:attn_ -s 3 -c 3 --csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e 2>/dev/null \
    | python -c "
import csv,sys
lines=sys.stdin.read().split('\n'); s=[i for i,l in enumerate(lines) if l.startswith('\"ID\"')][0]
rows=list(csv.reader(lines[s:])); h=rows[0]
U={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9,'nsecond':1e-9,'usecond':1e-6,'msecond':1e-3,'ns':1e-9,'us':1e-6,'ms':1e-3}
out={}
for r in rows[1:]:
    if len(r)<len(h): continue
    v=float(r[h.index('Metric Value')].replace(',',''))*U.get(r[h.index('Metric Unit')],1)
    out.setdefault(r[h.index('Kernel Name')].split('(')[0].split('::')[-1], {})[r[h.index('Metric Name')].split('.')[0]]=v
print('$envs', {k:(round(v['gpu__time_duration']*1e3,3), int(v['sm__cycles_elapsed'])//1000, round(v['sm__pipe_tensor_cycles_active'],1), round(v['dram__bytes_read']/1e9,2)) for k,v in out.items()})
"
done
