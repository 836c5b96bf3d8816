"""Debug driver: one small fwd+bwd case with error report."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_08524_b200.costmodel import ModelConfig
from tests.gpu_harness import schedule, make_inputs, run_plan_on_gpu, oracle, compare
from oracle.simworkers import global_offsets

lengths = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "256").split(",")]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
model = ModelConfig(q_heads=8, kv_heads=2, head_dim=128)
r = schedule(lengths, n, 512, model)
_, T = global_offsets(r)
q, k, v, do = make_inputs(T, model)
gpu = run_plan_on_gpu(r, model, q, k, v, do, backward=True)
ref, idx = oracle(r, model, q, k, v, do)
print(compare(gpu, ref, idx), flush=True)
