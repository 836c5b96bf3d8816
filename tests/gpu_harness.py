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

# Stated tolerance (bf16 inputs/outputs, fp32 accumulation), GPU vs fp64 oracle, per tensor
# and per case (the FlashAttention convention):
#   max-abs(gpu - oracle) <= 2 * max-abs(bf16 torch reference - oracle) + ATOL_FRAC * max|oracle|
#   rel-L2 (gpu - oracle) <= 2 * rel-L2 (bf16 torch reference - oracle) + REL_FLOOR
# for O, LSE, dQ, dK, dV, where the bf16 torch reference (``bf16_reference``) evaluates the
# same attention with bf16 operands and bf16-rounded intermediates (cuBLAS, fp32 accumulate).
# On top of that, fixed ceilings that hold for every case:
#   relative L2 error  ||gpu - ref|| / ||ref||   <= REL_L2   for O, dQ, dK, dV
#   LSE max-abs error                             <= LSE_ABS * max(1, max|LSE|)  (natural log)
REL_L2 = 1e-2
LSE_ABS = 1e-4
ATOL_FRAC = 2.0 ** -10
REL_FLOOR = 1e-4


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


def oracle(result, model, q, k, v, do, seq_ids=None, dtype=torch.float64, device=None):
    """fp64 oracle on (a subset of) sequences; returns dict + the row index used.  device:
    where the checker's fp64 arithmetic runs (default: the GPU when there is one)."""
    rows = global_sequence_rows(result)
    if seq_ids is not None:
        rows = {s: rows[s] for s in seq_ids}
    scale = 1.0 / math.sqrt(model.head_dim)
    # fp64 on the GPU when there is one (the checker's arithmetic is the same; minutes -> seconds)
    odev = torch.device(device) if device is not None else (
        torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu"))
    qf, kf, vf, dof = (x.to(odev, dtype) for x in (q, k, v, do))
    causal = result.deps.mask == "causal"
    o, lse = mono_fwd(qf, kf, vf, rows, scale, causal, dtype)
    dq, dk, dv = mono_bwd(qf, kf, vf, o, lse, dof, rows, scale, causal, dtype)
    idx = torch.cat(list(rows.values()))
    ref = {"o": o, "lse": lse, "dq": dq, "dk": dk, "dv": dv}
    return {k_: v_.cpu() for k_, v_ in ref.items()}, idx


def compare(gpu, ref, idx, keys=("o", "lse", "dq", "dk", "dv")):
    rep = {}
    for key in keys:
        if key in gpu:
            rep[key] = err(gpu[key][idx], ref[key][idx])
    return rep


# ---------------------------------------------------------------------------- bf16 reference
def bf16_chunk_reference(q, k, v, do, q_rows, kv_rows, diag_from, scale, device="cuda"):
    """The bf16 torch reference of one Q-row block against its KV rows (test infrastructure,
    FlashAttention's ``attention_ref(upcast=False)`` convention): S = Q K^T with bf16 operands
    (cuBLAS, fp32 accumulate, bf16 result), softmax in fp32 from the bf16 scores, P rounded to
    bf16, O = P V (bf16); backward dP = dO V^T (bf16), delta = rowsum(dO * O) in fp32,
    dS = P (dP - delta) rounded to bf16, dQ = dS K, dK = dS^T Q, dV = P^T dO (bf16 per head,
    summed over the GQA group in fp32).  KV rows from ``diag_from`` on form the diagonal chunk
    (inclusive causal ``j <= i``); the ones before it are fully visible.
    Returns fp64 CPU tensors (o, lse, dq, dk, dv) for those rows."""
    H, Hk, D = q.shape[1], k.shape[1], q.shape[2]
    G = H // Hk
    qn, kn = q_rows.numel(), kv_rows.numel()
    dev = torch.device(device)
    keep = torch.ones(qn, kn, dtype=torch.bool, device=dev)
    keep[:, diag_from:] = torch.ones(qn, kn - diag_from, dtype=torch.bool, device=dev).tril()
    out = {"o": torch.empty((qn, H, D), dtype=torch.float64), "lse": torch.empty((qn, H), dtype=torch.float64),
           "dq": torch.empty((qn, H, D), dtype=torch.float64),
           "dk": torch.zeros((kn, Hk, D), dtype=torch.float64), "dv": torch.zeros((kn, Hk, D), dtype=torch.float64)}
    qr, kr = q_rows.to(torch.long), kv_rows.to(torch.long)
    for kh in range(Hk):
        ks = k[kr, kh].to(dev, torch.bfloat16)
        vs = v[kr, kh].to(dev, torch.bfloat16)
        dk32 = torch.zeros((kn, D), dtype=torch.float32, device=dev)
        dv32 = torch.zeros((kn, D), dtype=torch.float32, device=dev)
        for h in range(kh * G, (kh + 1) * G):
            qs = q[qr, h].to(dev, torch.bfloat16)
            dos = do[qr, h].to(dev, torch.bfloat16)
            s = torch.matmul(qs, ks.T).float() * scale
            s = s.masked_fill(~keep, -math.inf)
            lse = torch.logsumexp(s, dim=-1)
            p = torch.exp(s - lse.unsqueeze(1)).to(torch.bfloat16)
            del s
            o = torch.matmul(p, vs)
            dp = torch.matmul(dos, vs.T)
            delta = (dos.float() * o.float()).sum(-1, keepdim=True)
            ds = (p.float() * (dp.float() - delta)).to(torch.bfloat16)
            del dp
            dq = torch.matmul(ds, ks).float() * scale
            dk32 += (torch.matmul(ds.T, qs).float() * scale).to(torch.bfloat16).float()
            dv32 += torch.matmul(p.T, dos).float()
            out["o"][:, h] = o.double().cpu()
            out["lse"][:, h] = lse.double().cpu()
            out["dq"][:, h] = dq.to(torch.bfloat16).double().cpu()
            del p, ds
        out["dk"][:, kh] = dk32.to(torch.bfloat16).double().cpu()
        out["dv"][:, kh] = dv32.to(torch.bfloat16).double().cpu()
    return out


def bf16_reference(result, model, q, k, v, do, seq_ids=None, device="cuda"):
    """``bf16_chunk_reference`` over whole sequences, laid out like ``oracle``."""
    rows = global_sequence_rows(result)
    if seq_ids is not None:
        rows = {sid: rows[sid] for sid in seq_ids}
    scale = 1.0 / math.sqrt(model.head_dim)
    causal = result.deps.mask == "causal"
    T = q.shape[0]
    H, Hk, D = model.q_heads, model.kv_heads, model.head_dim
    out = {"o": torch.zeros((T, H, D), dtype=torch.float64), "lse": torch.zeros((T, H), dtype=torch.float64),
           "dq": torch.zeros((T, H, D), dtype=torch.float64), "dk": torch.zeros((T, Hk, D), dtype=torch.float64),
           "dv": torch.zeros((T, Hk, D), dtype=torch.float64)}
    for idx in rows.values():
        r = bf16_chunk_reference(q, k, v, do, idx, idx, 0 if causal else idx.numel(), scale, device)
        for key in ("o", "lse", "dq"):
            out[key][idx] = r[key]
        out["dk"][idx] = r["dk"]
        out["dv"][idx] = r["dv"]
    return out


def tolerance_report(rep, brep):
    """Per tensor: the GPU error, the bf16 torch reference's error and the derived bounds."""
    out = {}
    for key, e in rep.items():
        b = brep[key]
        out[key] = dict(e, bf16_max_abs=b["max_abs"], bf16_rel_l2=b["rel_l2"],
                        bound_max_abs=2 * b["max_abs"] + ATOL_FRAC * e["ref_max"],
                        bound_rel_l2=2 * b["rel_l2"] + REL_FLOOR)
    return out


def within_fixed_caps(rep) -> bool:
    """The fixed ceilings of ``assert_within_tolerance`` as a predicate (multi-process checks)."""
    return all((e["max_abs"] <= LSE_ABS * max(1.0, e["ref_max"])) if key == "lse" else
               (e["rel_l2"] <= REL_L2) for key, e in rep.items())


def assert_within_tolerance(rep, brep=None, fixed_caps=True):
    """The fixed ceilings (N(0,1) inputs; ``fixed_caps=False`` for deliberately
    ill-conditioned inputs) and the per-case FlashAttention-convention bounds when the bf16
    torch reference's errors ``brep`` are given."""
    for key, e in rep.items():
        if not fixed_caps:
            break
        if key == "lse":
            assert e["max_abs"] <= LSE_ABS * max(1.0, e["ref_max"]), (key, e)
        else:
            assert e["rel_l2"] <= REL_L2, (key, e)
    if brep is not None:
        for key, t in tolerance_report(rep, brep).items():
            assert t["max_abs"] <= t["bound_max_abs"], (key, t)
            assert t["rel_l2"] <= t["bound_rel_l2"], (key, t)
