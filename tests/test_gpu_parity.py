"""GPU parity: sm_100a kernels (through the C ABI) vs the CPU fp64 oracle.

Tolerance (stated in tests/gpu_harness.py), per tensor and per case: max-abs and rel-L2 of
the GPU result against the oracle at most twice those of a bf16 torch reference of the same
attention plus a small floor (the FlashAttention convention), and under fixed
ceilings (rel-L2 <= 1e-2 for O, dQ, dK, dV; LSE max-abs <= 1e-4 * max(1, |LSE|)).  Every test
prints the GPU and bf16-reference errors and the bounds per tensor.
"""

import json

import pytest
import torch

from paper_2605_08524_b200 import configs
from paper_2605_08524_b200.costmodel import ModelConfig
from tests.gpu_harness import (assert_within_tolerance, bf16_chunk_reference, bf16_reference,
                               compare, err, make_inputs, oracle, run_plan_on_gpu, schedule,
                               tolerance_report)

pytestmark = pytest.mark.gpu

GQA_SMALL = ModelConfig(q_heads=8, kv_heads=2, head_dim=128)
LLAMA = configs.LLAMA3_8B


def _report(name, rep):
    print(f"\n[parity] {name}: " + json.dumps(rep))


def _full_check(lengths, n, block, model, mask="causal", seq_ids=None, backward=True,
                fuse_remote=False, inputs=None, name="case", fixed_caps=True):
    """GPU (simulated ranks on one device) vs the fp64 oracle, with the bf16 torch reference's
    errors beside it; asserts the stated tolerance and returns the report."""
    r = schedule(lengths, n, block, model, mask)
    from oracle.simworkers import global_offsets
    _, T = global_offsets(r)
    q, k, v, do = inputs(T, model, r) if inputs else make_inputs(T, model)
    gpu = run_plan_on_gpu(r, model, q, k, v, do, backward=backward, fuse_remote=fuse_remote)
    ref, idx = oracle(r, model, q, k, v, do, seq_ids)
    keys = ("o", "lse", "dq", "dk", "dv") if backward else ("o", "lse")
    rep = compare(gpu, ref, idx, keys)
    brep = compare(bf16_reference(r, model, q, k, v, do, seq_ids), ref, idx, keys)
    _report(name, tolerance_report(rep, brep))
    assert_within_tolerance(rep, brep, fixed_caps)
    return rep


def test_forward_single_tile():
    _full_check([128], 1, 256, GQA_SMALL, backward=False, name="fwd 128 tokens")


def test_forward_ragged_small():
    _full_check([1, 127, 129, 300, 513], 1, 256, GQA_SMALL, backward=False, name="fwd ragged")


def test_fwd_bwd_c1_lengths_single_rank():
    w = configs.c1_tiny(2)
    _full_check(list(w.lengths), 1, 512, GQA_SMALL, name="C1 lengths N=1")


def test_fwd_bwd_c1_two_simulated_ranks():
    w = configs.c1_tiny(2)
    _full_check(list(w.lengths), 2, 512, GQA_SMALL, name="C1 lengths N=2 (merge + dKV return)")


def test_fwd_bwd_four_simulated_ranks_ragged():
    _full_check([4000, 2100, 1000, 700, 129, 128, 5], 4, 1024, GQA_SMALL, name="ragged N=4")


def test_full_mask():
    _full_check([700, 300, 64], 2, 256, GQA_SMALL, mask="full", name="full mask N=2")


def test_many_q_heads_405b_shape():
    """Llama-3.1-405B-shaped heads (128 q / 8 kv, GQA group 16): more q-heads than one block of
    the backward preprocess covers (64 per gridDim.y slice), 2 simulated ranks."""
    _full_check([900, 300, 129], 2, 512, ModelConfig(q_heads=128, kv_heads=8, head_dim=128),
                name="128/8 heads N=2")


def test_c2_llama8b_n1_every_sequence():
    """C2 (Llama-3-8B GQA 32/8, 62,956-token packed batch, block 2K) at N=1, every sequence
    against the fp64 oracle, including the 16,561-token one whose last Q chunk has an
    18-chunk KV list (materialised-dS backward, the bench path)."""
    w = configs.c2_llama8b_64k(1)
    _full_check(list(w.lengths), 1, 2048, LLAMA, name="C2 N=1 all 15 sequences")


def _planted_max_inputs(T, model, r):
    """Scores that climb by ~80 raw units (> the 62.7-unit lazy-rescale threshold,
    8 / (scale * log2 e)) from one 128-key tile to the next along every sequence: every
    query gets +8 u and key j of a sequence +10 * (j // 128) u, u a unit vector."""
    from oracle.simworkers import global_sequence_rows
    g = torch.Generator().manual_seed(99)
    H, Hk, D = model.q_heads, model.kv_heads, model.head_dim
    q, k, v, do = (torch.randn((T, h, D), generator=g) for h in (H, Hk, Hk, H))
    u = torch.randn(D, generator=g)
    u = u / u.norm()
    q += 8.0 * u
    for idx in global_sequence_rows(r).values():
        k[idx] += (10.0 * (torch.arange(idx.numel()) // 128)).float()[:, None, None] * u
    return tuple(x.to(torch.bfloat16) for x in (q, k, v, do))


def test_forward_lazy_rescale_path():
    """K1 rescales O in TMEM only when a row max grows by > 2^8 in the exp2 domain; N(0,1)
    inputs never trigger it.  Planted scores force it on every KV tile step, and the kernel's
    rescale counter proves the branch ran (fcpb_debug_counters)."""
    from paper_2605_08524_b200 import native
    native.fwd_rescale_events(reset=True)
    # scores of ~100 nats and |K| up to ~110 make dQ ill-conditioned (the bf16 reference is
    # off by 5% rel-L2 there), so only the bf16-relative bound applies
    _full_check([1500, 700, 300], 1, 512, GQA_SMALL, inputs=_planted_max_inputs,
                name="fwd+bwd forced lazy O rescale", fixed_caps=False)
    torch.cuda.synchronize()
    n = native.fwd_rescale_events(reset=True)
    _report("lazy rescale events (warp level)", {"events": n})
    assert n > 0
    # and N(0,1) inputs do not take the branch (it stays off the hot path)
    _full_check([1500, 700], 1, 512, GQA_SMALL, backward=False, name="fwd N(0,1)")
    torch.cuda.synchronize()
    assert native.fwd_rescale_events(reset=True) == 0


def _last_chunk_check(lengths, block, model, name, env=None, monkeypatch=None, expect_ds=None):
    """A long sequence's last Q chunk (the longest KV list of the batch) at N=1 against the
    fp64 oracle of that chunk: O, LSE and dQ of its rows, and dK/dV of its rows -- complete
    there, since under the causal mask only the last Q chunk attends to the last KV chunk."""
    import math
    from oracle.attention_ref import chunk_fwd_bwd
    from oracle.simworkers import global_offsets, global_sequence_rows
    from paper_2605_08524_b200.attention import BlockAttention
    from paper_2605_08524_b200.worklist import build_rank_work
    for key, val in (env or {}).items():
        monkeypatch.setenv(key, val)
    r = schedule(lengths, 1, block, model)
    goff, T = global_offsets(r)
    if expect_ds is not None:
        assert BlockAttention(build_rank_work(r, 0), model, torch.device("cuda", 0)).ds_mode == expect_ds
    q, k, v, do = make_inputs(T, model)
    gpu = run_plan_on_gpu(r, model, q, k, v, do)
    sid = max(range(len(lengths)), key=lambda i: lengths[i])
    idx = global_sequence_rows(r)[sid]
    last = max(c for (s_, c) in r.deps.chunk_tokens if s_ == sid)
    m = r.deps.chunk_tokens[(sid, last)]
    L = idx.numel()
    q_rows, kv_rows = idx[L - m:], idx
    scale = 1.0 / math.sqrt(model.head_dim)
    o, lse, dq, dk, dv = (x.cpu() for x in chunk_fwd_bwd(q.cuda(), k.cuda(), v.cuda(), do.cuda(), q_rows,
                                                         kv_rows, L - m, scale, torch.float64))
    ref = {"o": o, "lse": lse, "dq": dq, "dk": dk[L - m:], "dv": dv[L - m:]}
    b = bf16_chunk_reference(q, k, v, do, q_rows, kv_rows, L - m, scale)
    b["dk"], b["dv"] = b["dk"][L - m:], b["dv"][L - m:]
    rep = {key: err(gpu[key][q_rows], ref[key]) for key in ref}
    brep = {key: err(b[key], ref[key]) for key in ref}
    _report(f"{name} (last chunk: {m} q rows x {L} kv rows)", tolerance_report(rep, brep))
    assert_within_tolerance(rep, brep)


def test_c3_shape_long_sequence_recompute_dq(monkeypatch):
    """C3's 256K sequence at Llama-3-8B 32/8, block 2K: its last Q chunk has a 256-entry KV
    list.  dS (about 1 TB) does not fit, so dQ runs the recompute kernel K2b."""
    _last_chunk_check([262144], 2048, LLAMA, "C3 256K seq, K2b recompute dQ", monkeypatch=monkeypatch,
                      expect_ds=False)


def test_c4_shape_block_4k(monkeypatch):
    """C4's 128K sequence, block 4K (2,048-token chunks), 32/8 heads (recompute dQ)."""
    _last_chunk_check([131072], 4096, LLAMA, "C4 128K seq, block 4K", monkeypatch=monkeypatch,
                      expect_ds=False)


def test_c5_shape_block_6k_both_dq_modes(monkeypatch):
    """C5's largest block (6K: 3,072-token chunks) with a varlen pack beside it, 32/8 heads,
    with materialised dS (default here) and with the recompute kernel forced."""
    _full_check([30000, 5000, 700], 1, 6144, LLAMA, seq_ids=[1, 2], name="C5 block 6K packed seqs")
    _last_chunk_check([30000, 5000, 700], 6144, LLAMA, "C5 block 6K, materialised dS", expect_ds=True)
    _last_chunk_check([30000, 5000, 700], 6144, LLAMA, "C5 block 6K, K2b recompute dQ",
                      env={"FCPB_DS": "0"}, monkeypatch=monkeypatch, expect_ds=False)


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
    b = bf16_reference(r, model, q, k, v, do)
    brep = {n: err(gather_rank(b[n], ex.layout, goff, r.deps), gather_rank(ref, ex.layout, goff, r.deps))
            for n, ref in (("o", ro), ("lse", rl), ("dq", rdq), ("dk", rdk), ("dv", rdv))}
    _report("executor N=1", tolerance_report(rep, brep))
    assert_within_tolerance(rep, brep)


def test_fwd_bwd_eight_simulated_ranks():
    """N=8 plan structures on one GPU (simulated workers): many stages, chunks with several
    receivers (race-free K4 rounds), merges of multi-stage partials."""
    _full_check([4000, 3100, 2100, 1500, 1000, 700, 520, 300, 129, 128, 64, 5], 8, 512, GQA_SMALL,
                name="ragged N=8")


def test_fwd_bwd_four_simulated_ranks_fused_remote_wave():
    """All received KV of a rank in one forward wave (the executor's fused-remote policy)."""
    _full_check([4000, 2100, 1000, 700, 129, 128, 5], 4, 512, GQA_SMALL, fuse_remote=True,
                name="ragged N=4 fused remote wave")


@pytest.mark.parametrize("n", [4, 8])
def test_fwd_resume_chained_partials(n):
    """fuse_remote="resume": the remote wave continues each Q run from the local wave's fp32
    (O, LSE) partial in the forward kernel (FcpbSegment.in_row), no K3 merge."""
    _full_check([4000, 3100, 2100, 1000, 700, 129, 128, 5], n, 512, GQA_SMALL, fuse_remote="resume",
                name=f"ragged N={n} resumed remote wave")


def test_fwd_bwd_recompute_dq(monkeypatch):
    """The recompute dQ kernel (K2b), used when dS does not fit in HBM (C3, C4): forced
    here on a case the default would run with materialised dS."""
    monkeypatch.setenv("FCPB_DS", "0")
    _full_check([4000, 2100, 1000, 700, 129, 128, 5], 2, 512, GQA_SMALL, name="recompute dQ N=2")

    
def test_fwd_bwd_llama_heads_four_simulated_ranks():
    """The Llama-3-8B head shape (32/8) through the multi-rank path (partials, merge, dKV
    return) on simulated ranks."""
    _full_check([9000, 4100, 3000, 2100, 1500, 700, 129], 4, 2048, LLAMA, name="Llama 32/8 N=4")


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


@pytest.mark.parametrize("runner", ["executor", "block_attention"])
def test_autograd_fcp_attention(runner):
    """``fcp_attention`` under ``loss.backward()`` (torch.autograd.Function over the executor
    and over a single-rank BlockAttention) against the fp64 oracle, same tolerance."""
    import math
    from oracle.attention_ref import mono_bwd, mono_fwd
    from oracle.simworkers import gather_rank, global_offsets, global_sequence_rows
    from paper_2605_08524_b200.attention import BlockAttention, fcp_attention
    from paper_2605_08524_b200.executor import FcpExecutor
    from paper_2605_08524_b200.worklist import build_rank_work
    model = GQA_SMALL
    r = schedule([1500, 700, 300, 129, 40], 1, 512, model)
    goff, T = global_offsets(r)
    q, k, v, do = make_inputs(T, model)
    dev = torch.device("cuda", 0)
    if runner == "executor":
        run = FcpExecutor(r, 0, model, dev)
        lay = run.layout
    else:
        work = build_rank_work(r, 0)
        run, lay = BlockAttention(work, model, dev), work.layout
    ql, kl, vl, dol = (gather_rank(x, lay, goff, r.deps).to(dev) for x in (q, k, v, do))
    ql.requires_grad_(True)
    kl.requires_grad_(True)
    vl.requires_grad_(True)
    o, lse = fcp_attention(ql, kl, vl, run, return_lse=True)
    (o.float() * dol.float()).sum().backward()
    rows = global_sequence_rows(r)
    scale = 1 / math.sqrt(model.head_dim)
    qf, kf, vf, dof = (x.double() for x in (q, k, v, do))
    ro, rl = mono_fwd(qf, kf, vf, rows, scale)
    rdq, rdk, rdv = mono_bwd(qf, kf, vf, ro, rl, dof, rows, scale)
    g = lambda x: gather_rank(x, lay, goff, r.deps)
    rep = {n: err(t.detach().cpu(), g(ref)) for n, t, ref in
           (("o", o, ro), ("lse", lse, rl), ("dq", ql.grad, rdq), ("dk", kl.grad, rdk), ("dv", vl.grad, rdv))}
    b = bf16_reference(r, model, q, k, v, do)
    brep = {n: err(g(b[n]), g(ref)) for n, ref in (("o", ro), ("lse", rl), ("dq", rdq), ("dk", rdk), ("dv", rdv))}
    _report(f"autograd through {runner}", tolerance_report(rep, brep))
    assert_within_tolerance(rep, brep)


def test_c1_tiny_model_through_the_executor():
    """The C1 tiny model itself (Hq = Hkv = 4, D = 64, run in bf16 on the GPU):
    the executor maps it onto the D=128, even-group kernels (executor.kernel_config: zero
    padding, q-heads run twice with a zero dO for the copy) -- C1 lengths, block 512, fwd+bwd
    and autograd against the fp64 oracle at scale 1/sqrt(64)."""
    import math
    from oracle.attention_ref import mono_bwd, mono_fwd
    from oracle.simworkers import gather_rank, global_offsets, global_sequence_rows
    from paper_2605_08524_b200.executor import FcpExecutor
    w = configs.c1_tiny(1)
    model = configs.TINY_MODEL
    r = schedule(list(w.lengths), 1, 512, model)
    goff, T = global_offsets(r)
    q, k, v, do = make_inputs(T, model)
    ex = FcpExecutor(r, 0, model, torch.device("cuda", 0))
    assert ex.adapt and ex.q_rep == 2
    loc = [gather_rank(x, ex.layout, goff, r.deps).cuda() for x in (q, k, v, do)]
    o, lse, dq, dk, dv = ex.step(*loc)
    assert o.shape == loc[0].shape and dk.shape == loc[1].shape and lse.shape == (T, 4)
    rows = global_sequence_rows(r)
    scale = 1 / math.sqrt(model.head_dim)
    qf, kf, vf, dof = (x.double() for x in (q, k, v, do))
    ro, rl = mono_fwd(qf, kf, vf, rows, scale)
    rdq, rdk, rdv = mono_bwd(qf, kf, vf, ro, rl, dof, rows, scale)
    g = lambda x: gather_rank(x, ex.layout, goff, r.deps)
    rep = {n: err(t.cpu(), g(ref)) for n, t, ref in
           (("o", o, ro), ("lse", lse, rl), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv))}
    b = bf16_reference(r, model, q, k, v, do)
    brep = {n: err(g(b[n]), g(ref)) for n, ref in (("o", ro), ("lse", rl), ("dq", rdq), ("dk", rdk), ("dv", rdv))}
    _report("C1 tiny model (4/4 heads, D=64) through the executor", tolerance_report(rep, brep))
    assert_within_tolerance(rep, brep)
    # and through autograd
    qg, kg, vg = (x.clone().requires_grad_(True) for x in loc[:3])
    og = ex.attention(qg, kg, vg)
    (og.float() * loc[3].float()).sum().backward()
    assert torch.equal(og.detach(), o) and torch.equal(qg.grad, dq) and torch.equal(kg.grad, dk)


def test_gather_copy_pull_kernel_is_exact():
    """K5 pull kernel (fcpb_gather_copy): byte-exact ranges, 16-byte granularity, full and
    partial 64 KB segments, and nothing written outside the ranges."""
    from paper_2605_08524_b200 import native
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(7)
    src = torch.randint(-2**31, 2**31 - 1, (1 << 22,), dtype=torch.int32, generator=g).to(dev)
    dst = torch.zeros(1 << 22, dtype=torch.int32, device=dev)
    step = native.gather_seg_bytes()
    assert step % 16 == 0
    # (src byte offset, dst byte offset, bytes): 16-byte aligned, sizes around the segment size
    ranges = [(0, 1 << 20, 16), (4096, 0, step), (2 * step, 3 << 20, step - 16),
              (5 << 20, 6 << 20, 3 * step + 48), (160, 8 << 20, 2048 * 7)]
    segs = []
    for so, do_, n in ranges:
        for o in range(0, n, step):
            segs.append((dst.data_ptr() + do_ + o, src.data_ptr() + so + o, min(step, n - o)))
    tab = torch.tensor(segs, dtype=torch.int64, device=dev)
    native.gather_copy(tab, 7, torch.cuda.current_stream(dev))
    torch.cuda.synchronize(dev)
    want = torch.zeros_like(dst)
    for so, do_, n in ranges:
        want[do_ // 4:(do_ + n) // 4] = src[so // 4:(so + n) // 4]
    assert torch.equal(dst, want)


def test_gather_copy_based_is_exact():
    """fcpb_gather_copy_based: base-relative segments resolve against the bases passed by
    value (two sources, two destinations), byte-exact, nothing written outside the ranges,
    and the same table reused with other bases."""
    from paper_2605_08524_b200 import native
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(11)
    srcs = [torch.randint(-2**31, 2**31 - 1, (1 << 20,), dtype=torch.int32, generator=g).to(dev) for _ in range(2)]
    step = native.gather_seg_bytes()
    # (dst base, dst off, src base, src off, bytes); bases 0/1 destinations, 2/3 sources
    ranges = [(0, 0, 2, 4096, 16), (1, 64, 3, 0, step + 32), (0, 1 << 16, 3, 1 << 18, 2 * step),
              (1, 1 << 19, 2, 160, 2048 * 3)]
    segs = []
    for db, do_, sb, so, n in ranges:
        for o in range(0, n, step):
            segs.append(((db << 56) | (do_ + o), (sb << 56) | (so + o), min(step, n - o)))
    tab = torch.tensor(segs, dtype=torch.int64, device=dev)
    for _ in range(2):                        # the same table against fresh destinations
        dsts = [torch.zeros(1 << 20, dtype=torch.int32, device=dev) for _ in range(2)]
        bases = [d.data_ptr() for d in dsts] + [s.data_ptr() for s in srcs]
        native.gather_copy_based(tab, bases, 5, torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        want = [torch.zeros_like(d) for d in dsts]
        for db, do_, sb, so, n in ranges:
            want[db][do_ // 4:(do_ + n) // 4] = srcs[sb - 2][so // 4:(so + n) // 4]
        assert all(torch.equal(a, b) for a, b in zip(dsts, want))
