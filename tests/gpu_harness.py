"""Shared GPU-test harness: run the real kernels for every rank of a plan on one
device (simulated workers), compare against the CPU oracle.

Inputs follow BASELINE.md: Q, K, V, dO ~ N(0,1) drawn in fp32 on the CPU from a
seeded generator and rounded to bf16; the oracle consumes the same bf16 values
upcast, so the reported error is kernel arithmetic only.
"""

from __future__ import annotations

import math

import torch

from oracle.attention_ref import mono_bwd, mono_fwd
from oracle.simworkers import gather_rank, global_offsets, global_sequence_rows
from paper_2605_08524_b200.attention import BlockAttention
from paper_2605_08524_b200.costmodel import DEFAULT_EFFICIENCY, ModelConfig
from paper_2605_08524_b200.distributor import chunk_placement
from paper_2605_08524_b200.pipeline import fcp_schedule
from paper_2605_08524_b200.sharding import ShardingConfig
from paper_2605_08524_b200.workload import Batch, Sequence
from paper_2605_08524_b200.worklist import build_rank_work

# Stated tolerance (bf16 inputs/outputs, fp32 accumulation), GPU vs fp64 oracle:
#   relative L2 error  ||gpu - ref|| / ||ref||   <= REL_L2   for O, dQ, dK, dV
#   LSE max-abs error                             <= LSE_ABS  (natural-log units)
REL_L2 = 2e-2
LSE_ABS = 2e-2


def schedule(lengths, n, block, model, mask="causal", tpw=None):
    tpw = tpw or -(-sum(lengths) // n)
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(lengths)), n, tpw)
    return fcp_schedule(batch, n, ShardingConfig(block, mask), model, DEFAULT_EFFICIENCY)


def make_inputs(T, model: ModelConfig, seed=1234):
    g = torch.Generator().manual_seed(seed)
    H, Hk, D = model.q_heads, model.kv_heads, model.head_dim
    mk = lambda h: torch.randn((T, h, D), generator=g).to(torch.bfloat16)
    return mk(H), mk(Hk), mk(Hk), mk(H)


def err(a, b):
    a = a.double().cpu()
    b = b.double().cpu()
    d = (a - b)
    return {"max_abs": d.abs().max().item(), "rel_l2": (d.norm() / b.norm().clamp_min(1e-30)).item(),
            "ref_max": b.abs().max().item()}


def run_plan_on_gpu(result, model, q, k, v, do, device="cuda", backward=True, fuse_remote=False):
    """Execute every rank's work list with the CUDA kernels; the exchange is an
    on-device gather of the owners' K/V, the dKV return uses the K4 kernel."""
    n = result.assignment.n_workers
    deps = result.deps
    goff, T = global_offsets(result)
    owner = chunk_placement(result.assignment, result.units)
    works = [build_rank_work(result, w, fuse_remote=fuse_remote) for w in range(n)]
    ops = [BlockAttention(w, model, device) for w in works]
    o = torch.zeros((T, model.q_heads, model.head_dim), dtype=torch.bfloat16)
    lse = torch.zeros((T, model.q_heads), dtype=torch.float32)
    loc = []
    for w, (work, op) in enumerate(zip(works, ops)):
        lay = work.layout
        t = {name: gather_rank(x, lay, goff, deps).to(device) for name, x in
             (("q", q), ("k", k), ("v", v), ("do", do))}
        t["kr"] = gather_rank(k, lay, goff, deps, recv=True).to(device) if lay.recv_tokens else None
        t["vr"] = gather_rank(v, lay, goff, deps, recv=True).to(device) if lay.recv_tokens else None
        ow, lw = op.forward(t["q"], t["k"], t["v"], t["kr"], t["vr"])
        t["o"], t["lse"] = ow, lw
        loc.append(t)
    torch.cuda.synchronize()
    out = {"o": o, "lse": lse}
    for w, work in enumerate(works):
        lay = work.layout
        for c in lay.chunks:
            a, m = lay.offset[c], deps.chunk_tokens[c]
            o[goff[c]:goff[c] + m] = loc[w]["o"][a:a + m].cpu()
            lse[goff[c]:goff[c] + m] = loc[w]["lse"][a:a + m].cpu()
    if not backward:
        return out
    dq = torch.zeros((T, model.q_heads, model.head_dim), dtype=torch.bfloat16)
    dk = torch.zeros((T, model.kv_heads, model.head_dim), dtype=torch.float32)
    dv = torch.zeros_like(dk)
    acc = []
    for w, op in enumerate(ops):
        t = loc[w]
        prep = op.backward_prepare(t["o"], t["lse"], t["do"])
        dka, dva = op.alloc_dkv(False)
        dkr, dvr = op.alloc_dkv(True)
        op.backward_launch(True, t["q"], t["k"], t["v"], t["kr"], t["vr"], prep, t["do"],
                           dka, dva, dkr, dvr)
        op.backward_launch(False, t["q"], t["k"], t["v"], t["kr"], t["vr"], prep, t["do"],
                           dka, dva, dkr, dvr)
        dqa = op.backward_dq(t["q"], t["k"], t["v"], t["kr"], t["vr"], prep, t["do"])
        acc.append((dqa, dka, dva, dkr, dvr))
    # dKV return to the owner from every consuming rank + K4 reduce at the owner
    for w, work in enumerate(works):
        lay = work.layout
        dkr, dvr = acc[w][3], acc[w][4]
        for c in lay.recv_chunks:
            if c not in lay.consumed:       # relayed only (ring / ByteScale plans)
                continue
            o_rank = owner[c]
            m = deps.chunk_tokens[c]
            a = lay.recv_offset[c]
            b = works[o_rank].layout.offset[c]
            rows = torch.arange(b, b + m, dtype=torch.int32, device=device)
            ops[o_rank].reduce_dkv(acc[o_rank][1], dkr[a:a + m].contiguous(), rows)
            ops[o_rank].reduce_dkv(acc[o_rank][2], dvr[a:a + m].contiguous(), rows)
    for w, (work, op) in enumerate(zip(works, ops)):
        lay = work.layout
        dq_b = acc[w][0]
        for c in lay.chunks:
            a, m = lay.offset[c], deps.chunk_tokens[c]
            dq[goff[c]:goff[c] + m] = dq_b[a:a + m].cpu()
            dk[goff[c]:goff[c] + m] = acc[w][1][a:a + m].cpu()
            dv[goff[c]:goff[c] + m] = acc[w][2][a:a + m].cpu()
    torch.cuda.synchronize()
    out.update(dq=dq, dk=dk.to(torch.bfloat16), dv=dv.to(torch.bfloat16))
    return out


def oracle(result, model, q, k, v, do, seq_ids=None, dtype=torch.float64):
    """fp64 oracle on (a subset of) sequences; returns dict + the row index used."""
    rows = global_sequence_rows(result)
    if seq_ids is not None:
        rows = {s: rows[s] for s in seq_ids}
    scale = 1.0 / math.sqrt(model.head_dim)
    qf, kf, vf, dof = (x.to(dtype) for x in (q, k, v, do))
    causal = result.deps.mask == "causal"
    o, lse = mono_fwd(qf, kf, vf, rows, scale, causal, dtype)
    dq, dk, dv = mono_bwd(qf, kf, vf, o, lse, dof, rows, scale, causal, dtype)
    idx = torch.cat(list(rows.values()))
    return {"o": o, "lse": lse, "dq": dq, "dk": dk, "dv": dv}, idx


def compare(gpu, ref, idx, keys=("o", "lse", "dq", "dk", "dv")):
    rep = {}
    for key in keys:
        if key in gpu:
            rep[key] = err(gpu[key][idx], ref[key][idx])
    return rep


def assert_within_tolerance(rep):
    for key, e in rep.items():
        if key == "lse":
            assert e["max_abs"] <= LSE_ABS, (key, e)
        else:
            assert e["rel_l2"] <= REL_L2, (key, e)
