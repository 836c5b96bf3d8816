"""GPU parity: sm_100a kernels (through the C ABI) vs the CPU fp64 oracle.

Tolerance (stated in tests/gpu_harness.py): rel-L2 <= 2e-2 for O, dQ, dK, dV and
LSE max-abs <= 2e-2; every test prints max-abs and rel-L2 per tensor.
"""

import json

import pytest
import torch

from paper_2605_08524_b200 import configs
from paper_2605_08524_b200.costmodel import ModelConfig
from tests.gpu_harness import (assert_within_tolerance, compare, make_inputs, oracle,
                               run_plan_on_gpu, schedule)

pytestmark = pytest.mark.gpu

GQA_SMALL = ModelConfig(q_heads=8, kv_heads=2, head_dim=128)
LLAMA = configs.LLAMA3_8B


def _report(name, rep):
    print(f"\n[parity] {name}: " + json.dumps(rep))


def _full_check(lengths, n, block, model, mask="causal", seq_ids=None, backward=True,
                fuse_remote=False):
    r = schedule(lengths, n, block, model, mask)
    from oracle.simworkers import global_offsets
    _, T = global_offsets(r)
    q, k, v, do = make_inputs(T, model)
    gpu = run_plan_on_gpu(r, model, q, k, v, do, backward=backward, fuse_remote=fuse_remote)
    ref, idx = oracle(r, model, q, k, v, do, seq_ids)
    keys = ("o", "lse", "dq", "dk", "dv") if backward else ("o", "lse")
    rep = compare(gpu, ref, idx, keys)
    return rep


def test_forward_single_tile():
    rep = _full_check([128], 1, 256, GQA_SMALL, backward=False)
    _report("fwd 128 tokens", rep)
    assert_within_tolerance(rep)


def test_forward_ragged_small():
    rep = _full_check([1, 127, 129, 300, 513], 1, 256, GQA_SMALL, backward=False)
    _report("fwd ragged", rep)
    assert_within_tolerance(rep)


def test_fwd_bwd_c1_lengths_single_rank():
    w = configs.c1_tiny(2)
    rep = _full_check(list(w.lengths), 1, 512, GQA_SMALL)
    _report("C1 lengths N=1", rep)
    assert_within_tolerance(rep)


def test_fwd_bwd_c1_two_simulated_ranks():
    w = configs.c1_tiny(2)
    rep = _full_check(list(w.lengths), 2, 512, GQA_SMALL)
    _report("C1 lengths N=2 (merge + dKV return)", rep)
    assert_within_tolerance(rep)


def test_fwd_bwd_four_simulated_ranks_ragged():
    rep = _full_check([4000, 2100, 1000, 700, 129, 128, 5], 4, 1024, GQA_SMALL)
    _report("ragged N=4", rep)
    assert_within_tolerance(rep)


def test_full_mask():
    rep = _full_check([700, 300, 64], 2, 256, GQA_SMALL, mask="full")
    _report("full mask N=2", rep)
    assert_within_tolerance(rep)


def test_c2_llama8b_n1_sampled():
    """C2 (Llama-3-8B GQA 32/8, 64K packed, block 2K) at N=1; the oracle checks a
    sample of sequences including the longest (bounded CPU time)."""
    w = configs.c2_llama8b_64k(1)
    lengths = list(w.lengths)
    # a 3-pair zigzag sequence (5487), a 2-pair one (2091) and a varlen-pack member (1520)
    pick = [lengths.index(5487), lengths.index(2091), lengths.index(1520)]
    rep = _full_check(lengths, 1, 2048, LLAMA, seq_ids=pick)
    _report("C2 N=1 sampled", rep)
    assert_within_tolerance(rep)


def test_measured_report_single_rank():
    """The executor's measured SimReport-shaped record (the counterpart of the reference's
    analytic simulate()) at N=1: one worker, no stages, FLOPs from the reference accounting."""
    from paper_2605_08524_b200.costmodel import batch_token_pairs
    from paper_2605_08524_b200.executor import FcpExecutor
    lengths = [1500, 700, 300]
    r = schedule(lengths, 1, 512, GQA_SMALL)
    from oracle.simworkers import global_offsets, gather_rank
    goff, T = global_offsets(r)
    ex = FcpExecutor(r, 0, GQA_SMALL, torch.device("cuda", 0))
    loc = [gather_rank(x, ex.layout, goff, r.deps).cuda() for x in make_inputs(T, GQA_SMALL)]
    rep = ex.measured_report(*loc, reps=2)
    _report("measured report N=1", {"total_ms": rep.total_time * 1e3,
                                    "compute_ms": rep.per_worker[0].compute_time * 1e3})
    assert len(rep.per_worker) == 1 and rep.stages == []
    # compute = the sum of CUDA-event spans around each launch (about ten launches of a
    # ~0.1 ms step here), so per-span event resolution alone can add several percent
    assert 0 < rep.per_worker[0].compute_time <= rep.total_time * 1.25
    assert rep.total_flops == 3.5 * GQA_SMALL.flops_per_token_pair * batch_token_pairs(lengths, "causal")


def test_executor_single_rank_parity():
    """FcpExecutor at N=1 (the bench path): no partials come back, so the dK/dV kernel
    writes the final bf16 gradients directly; checked against the fp64 oracle."""
    import math
    from oracle.attention_ref import mono_bwd, mono_fwd
    from oracle.simworkers import gather_rank, global_offsets, global_sequence_rows
    from paper_2605_08524_b200.executor import FcpExecutor
    from tests.gpu_harness import err, REL_L2, LSE_ABS
    model = GQA_SMALL
    r = schedule([1500, 700, 300, 129, 40], 1, 512, model)
    goff, T = global_offsets(r)
    q, k, v, do = make_inputs(T, model)
    ex = FcpExecutor(r, 0, model, torch.device("cuda", 0))
    assert ex.ret_tokens == 0
    loc = [gather_rank(x, ex.layout, goff, r.deps).cuda() for x in (q, k, v, do)]
    o, lse, dq, dk, dv = ex.step(*loc)
    assert dk.dtype == torch.bfloat16 and dv.dtype == torch.bfloat16
    rows = global_sequence_rows(r)
    scale = 1 / math.sqrt(model.head_dim)
    qf, kf, vf, dof = (x.double() for x in (q, k, v, do))
    ro, rl = mono_fwd(qf, kf, vf, rows, scale)
    rdq, rdk, rdv = mono_bwd(qf, kf, vf, ro, rl, dof, rows, scale)
    rep = {n: err(g.cpu(), gather_rank(ref, ex.layout, goff, r.deps))
           for n, g, ref in (("o", o, ro), ("lse", lse, rl), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv))}
    _report("executor N=1", rep)
    for n, e in rep.items():
        assert (e["max_abs"] <= LSE_ABS) if n == "lse" else (e["rel_l2"] <= REL_L2), (n, e)


def test_fwd_bwd_eight_simulated_ranks():
    """N=8 plan structures on one GPU (simulated workers): many stages, chunks with several
    receivers (race-free K4 rounds), merges of multi-stage partials."""
    rep = _full_check([4000, 3100, 2100, 1500, 1000, 700, 520, 300, 129, 128, 64, 5], 8, 512, GQA_SMALL)
    _report("ragged N=8", rep)
    assert_within_tolerance(rep)


def test_fwd_bwd_four_simulated_ranks_fused_remote_wave():
    """All received KV of a rank in one forward wave (the executor's fused-remote policy)."""
    rep = _full_check([4000, 2100, 1000, 700, 129, 128, 5], 4, 512, GQA_SMALL, fuse_remote=True)
    _report("ragged N=4 fused remote wave", rep)
    assert_within_tolerance(rep)


def test_fwd_bwd_recompute_dq(monkeypatch):
    """The recompute dQ kernel (K2b), used when dS does not fit in HBM (C3, C4): forced
    here on a case the default would run with materialised dS."""
    monkeypatch.setenv("FCPB_DS", "0")
    rep = _full_check([4000, 2100, 1000, 700, 129, 128, 5], 2, 512, GQA_SMALL)
    _report("recompute dQ N=2", rep)
    assert_within_tolerance(rep)


def test_materialised_ds_is_default_when_it_fits():
    from paper_2605_08524_b200.attention import BlockAttention
    from paper_2605_08524_b200.worklist import build_rank_work
    r = schedule([1000, 300], 1, 512, GQA_SMALL)
    op = BlockAttention(build_rank_work(r, 0), GQA_SMALL, torch.device("cuda", 0))
    assert op.ds_mode


@pytest.mark.gpu
def test_dkv_finalize_matches_ordered_fp32_sum():
    """K4 fused finalize through the C ABI: bf16(local + staged partials in CSR order), against
    the same fp32 sum in the same order on the host side (bit-exact)."""
    from paper_2605_08524_b200.attention import BlockAttention  # noqa: F401  (loads the lib)
    from paper_2605_08524_b200 import native
    lib = native.load()
    g = torch.Generator().manual_seed(7)
    T, R, row = 37, 50, 8 * 128
    local_k, local_v = (torch.randn(T, row, generator=g) for _ in range(2))
    st_k, st_v = (torch.randn(R, row, generator=g) for _ in range(2))
    counts = torch.randint(0, 4, (T,), generator=g)
    row_ptr = torch.zeros(T + 1, dtype=torch.int32)
    row_ptr[1:] = torch.cumsum(counts, 0).to(torch.int32)
    src = torch.randint(0, R, (int(row_ptr[-1]),), generator=g, dtype=torch.int32)
    ref_k, ref_v = local_k.clone(), local_v.clone()
    for r in range(T):
        for j in range(int(row_ptr[r]), int(row_ptr[r + 1])):
            ref_k[r] += st_k[src[j]]
            ref_v[r] += st_v[src[j]]
    dev = torch.device("cuda", 0)
    d = [x.to(dev) for x in (local_k, local_v, st_k, st_v, row_ptr, src)]
    out_k = torch.empty(T, row, dtype=torch.bfloat16, device=dev)
    out_v = torch.empty_like(out_k)
    native.check(lib.fcpb_dkv_finalize(*(x.data_ptr() for x in d), T, row, out_k.data_ptr(),
                                       out_v.data_ptr(), 0))
    torch.cuda.synchronize()
    assert torch.equal(out_k.cpu(), ref_k.to(torch.bfloat16))
    assert torch.equal(out_v.cpu(), ref_v.to(torch.bfloat16))
