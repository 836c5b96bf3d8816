"""Debug driver: run one forward case and print errors / device messages."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_08524_b200.costmodel import ModelConfig
from tests.gpu_harness import schedule, make_inputs, run_plan_on_gpu, oracle, compare
from oracle.simworkers import global_offsets

cases = {
    "two_tiles": ([256], 1, 512),         # one pack chunk of 256 rows: 2 mblocks, diag tiles
    "two_chunks": ([512], 1, 512),        # zigzag k=1: 2 chunks of 256: chunk1 sees 2 kv chunks
    "ragged": ([1, 127, 129, 300, 513], 1, 256),
}
model = ModelConfig(q_heads=8, kv_heads=2, head_dim=128)
for name in sys.argv[1:]:
    lengths, n, block = cases[name]
    r = schedule(lengths, n, block, model)
    _, T = global_offsets(r)
    q, k, v, do = make_inputs(T, model)
    print("case", name, flush=True)
    gpu = run_plan_on_gpu(r, model, q, k, v, do, backward=False)
    ref, idx = oracle(r, model, q, k, v, do)
    print(name, compare(gpu, ref, idx, ("o", "lse")), flush=True)
