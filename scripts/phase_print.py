import json,sys
d=json.loads(sys.stdin.read()); ph=d["phases_ms_rank0"]
print(sys.argv[1], round(d["ms_per_step"],3), {k.split(':')[1]:v for k,v in ph.items() if "stage_done" not in k and "wave" not in k})
