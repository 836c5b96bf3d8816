"""Multi-rank executor check, run under torchrun: the FcpExecutor's fwd+bwd with the real
exchange (IPC peer regions, copy-engine pulls, flag barriers) vs the fp64 oracle.

One process per GPU over NVLink (NCCL group), or -- when the box has fewer GPUs than ranks,
or FCPB_SHARED_GPU=1 -- every rank a separate process on GPU 0 (gloo group): the same
product code path (IPC regions opened by another process, stream-memory-op flags, 2-D
copy-engine pulls), time-sliced on one device.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P tests/mp_gpu_check.py [lengths] [block]
"""
import json
import math
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.attention_ref import mono_bwd, mono_fwd  # noqa: E402
from oracle.simworkers import gather_rank, global_offsets, global_sequence_rows  # noqa: E402
from paper_2605_08524_b200.costmodel import ModelConfig  # noqa: E402
from paper_2605_08524_b200.executor import FcpExecutor  # noqa: E402
from tests.gpu_harness import err, make_inputs, schedule, within_fixed_caps  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    shared = os.environ.get("FCPB_SHARED_GPU") == "1" or torch.cuda.device_count() < world
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if shared:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    lengths = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "3523,2702,2219,1292,1438,413,544,319").split(",")]
    block = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    hq, hk = (int(x) for x in os.environ.get("FCPB_CHECK_HEADS", "8,2").split(","))
    dim = int(os.environ.get("FCPB_CHECK_DIM", "128"))
    model = ModelConfig(q_heads=hq, kv_heads=hk, head_dim=dim)
    sched = os.environ.get("FCPB_CHECK_SCHED", "fcp")
    if sched == "fcp":
        r = schedule(lengths, world, block, model)
    else:                            # the reference's ring plan (relays) on the same executor
        from paper_2605_08524_b200.baselines import ring_schedule
        from paper_2605_08524_b200.workload import Batch, Sequence
        r = ring_schedule(Batch(tuple(Sequence(i, l) for i, l in enumerate(lengths)), world,
                                -(-sum(lengths) // world)), world, model)
    goff, T = global_offsets(r)
    q, k, v, do = make_inputs(T, model)
    ex = FcpExecutor(r, rank, model, dev)
    lay = ex.layout
    loc = [gather_rank(x, lay, goff, r.deps).to(dev) for x in (q, k, v, do)]
    for _ in range(2):   # twice: the executor is reused across layers
        o, lse, dq, dk, dv = ex.step(*loc)
    torch.cuda.synchronize()
    rows = global_sequence_rows(r)
    scale = 1 / math.sqrt(model.head_dim)
    qf, kf, vf, dof = (x.to(dev, torch.float64) for x in (q, k, v, do))   # fp64 checker on the GPU
    ro, rl = mono_fwd(qf, kf, vf, rows, scale)
    rdq, rdk, rdv = mono_bwd(qf, kf, vf, ro, rl, dof, rows, scale)
    ro, rl, rdq, rdk, rdv = (x.cpu() for x in (ro, rl, rdq, rdk, rdv))
    del qf, kf, vf, dof
    rep = {}
    for name, got, ref in (("o", o, ro), ("lse", lse, rl), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        rep[name] = err(got.cpu(), gather_rank(ref, lay, goff, r.deps))
    ok = within_fixed_caps(rep)
    # the same step through torch.autograd (fcp_attention over the executor, N ranks)
    qg, kg, vg = (x.clone().requires_grad_(True) for x in loc[:3])
    og = ex.attention(qg, kg, vg)
    (og.float() * loc[3].float()).sum().backward()
    autograd_same = (torch.equal(og.detach(), o) and torch.equal(qg.grad, dq) and torch.equal(kg.grad, dk)
                     and torch.equal(vg.grad, dv))
    ok = ok and autograd_same
    # transparent reshuffler (§8f): user layout -> FCP layout equals the executor's inputs
    # exactly, and the round trip is the identity (symmetric-memory copy-engine pulls)
    from paper_2605_08524_b200.reshuffle import Reshuffler, user_layouts
    ul = user_layouts(r)[rank]
    usr = [torch.cat([x[goff[c]:goff[c] + r.deps.chunk_tokens[c]] for c in ul.chunks]).to(dev)
           if ul.chunks else x.new_zeros((0,) + tuple(x.shape[1:])).to(dev) for x in (q, k, v, do)]
    rs = Reshuffler(r, rank, model, dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    fcp_in = rs.to_fcp(*usr)
    t1.record()
    back = rs.from_fcp(*fcp_in)
    torch.cuda.synchronize()
    reshuffle_ok = all(torch.equal(a, b) for a, b in zip(fcp_in, loc)) and \
        all(torch.equal(a, b) for a, b in zip(back, usr))
    ok = ok and reshuffle_ok
    # forward from the user layout: remote reshuffle pulls overlapped with the PRE_WAVE tiles
    # of the rows that stay here (an executor built with the reshuffler's resident chunks)
    ex_u = FcpExecutor(r, rank, model, dev, resident=rs.resident_chunks())
    usr3 = [x.clone() for x in usr[:3]]
    user_fwd_ok = True
    for overlap in (True, False):       # PRE_WAVE beside copy-engine pulls / move, then forward
        (qf, kf, vf), (o_u, lse_u) = ex_u.forward_user(rs, *usr3, overlap=overlap)
        torch.cuda.synchronize()
        user_fwd_ok = user_fwd_ok and torch.equal(qf, loc[0]) and torch.equal(kf, loc[1]) \
            and torch.equal(vf, loc[2])
        rep_u = {"o": err(o_u.cpu(), gather_rank(ro, lay, goff, r.deps)),
                 "lse": err(lse_u.cpu(), gather_rank(rl, lay, goff, r.deps))}
        user_fwd_ok = user_fwd_ok and within_fixed_caps(rep_u)
    ok = ok and user_fwd_ok
    # measured SimReport-shaped record (collective): one WorkerStats per rank, one record per stage
    mr = ex.measured_report(*loc, reps=2)
    ok = ok and len(mr.per_worker) == world and len(mr.stages) == len(ex.stages) \
        and mr.total_time > 0 and all(w.compute_time > 0 for w in mr.per_worker) and mr.total_flops > 0
    print(json.dumps({"rank": rank, "world": world, "shared_gpu": shared, "autograd_same": autograd_same, "user_fwd_ok": user_fwd_ok,
                      "pre_wave": any(w.stage == -2 for w in ex_u.work.fwd.waves), "recv_tokens": lay.recv_tokens,
                      "stages": len(ex.stages), "ok": ok, "errors": rep,
                      "measured_total_ms": mr.total_time * 1e3,
                      "reshuffle_ok": reshuffle_ok, "reshuffle_to_fcp_ms": t0.elapsed_time(t1),
                      "measured_eta": [round(w.eta, 3) for w in mr.per_worker]}), flush=True)
    # collective release of every peer-memory region (a new executor per batch must not leak)
    for obj in (ex_u, ex, rs):
        obj.close()
    flag = torch.tensor([1 if ok else 0], device="cpu" if shared else dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
