"""CPU oracle ladder: SDPA pin -> dense -> tiled -> work-list emulation (N=1, 2, 3).

Level 3 interprets the exact device work lists the kernels consume, with
in-process copies standing in for the NVLink exchange, so the host side of the
data plane (layout, waves, partial rows, merge groups, KV-keyed backward, dKV
return) is verified here without a GPU.
"""

import math

import pytest
import torch

from oracle.attention_ref import (chunk_fwd_bwd, emulate_backward, emulate_forward, mono_bwd,
                                  mono_fwd, sequence_rows, tiled_fwd)
from oracle.simworkers import (gather_rank, global_offsets, global_sequence_rows,
                               return_partials, scatter_rank)
from paper_2605_08524_b200.costmodel import DEFAULT_EFFICIENCY, ModelConfig
from paper_2605_08524_b200.distributor import chunk_placement
from paper_2605_08524_b200.pipeline import fcp_schedule
from paper_2605_08524_b200.sharding import ShardingConfig
from paper_2605_08524_b200.workload import Batch, Sequence
from paper_2605_08524_b200.worklist import build_rank_work

MODEL = ModelConfig(q_heads=4, kv_heads=2, head_dim=32, dtype_bytes=2)


def _schedule(lengths, n, block, mask="causal", coalesce=16, scheduler="fcp"):
    tpw = -(-sum(lengths) // n)
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(lengths)), n, tpw)
    if scheduler == "ring":
        from paper_2605_08524_b200.baselines import ring_schedule
        return ring_schedule(batch, n, MODEL, mask)
    if scheduler == "bytescale":
        from paper_2605_08524_b200.baselines import bytescale_schedule
        return bytescale_schedule(batch, n, tpw, MODEL, mask)
    return fcp_schedule(batch, n, ShardingConfig(block, mask), MODEL, DEFAULT_EFFICIENCY,
                        coalesce_degree=coalesce)


def _inputs(T, seed=0):
    g = torch.Generator().manual_seed(seed)
    H, Hk, D = MODEL.q_heads, MODEL.kv_heads, MODEL.head_dim
    mk = lambda h: torch.randn((T, h, D), generator=g, dtype=torch.float64)
    return mk(H), mk(Hk), mk(Hk), mk(H)


def test_dense_matches_torch_sdpa():
    lengths = [300, 77, 1]
    T = sum(lengths)
    q, k, v, _ = _inputs(T)
    rows, pos = {}, 0
    for i, l in enumerate(lengths):
        rows[i] = torch.arange(pos, pos + l)
        pos += l
    scale = 1 / math.sqrt(MODEL.head_dim)
    o, _ = mono_fwd(q, k, v, rows, scale)
    for idx in rows.values():
        qq = q[idx].transpose(0, 1)
        kk = k[idx].repeat_interleave(2, 1).transpose(0, 1)
        vv = v[idx].repeat_interleave(2, 1).transpose(0, 1)
        ref = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
        assert torch.allclose(o[idx].transpose(0, 1), ref, atol=1e-12)


def test_dense_backward_matches_autograd():
    lengths = [200, 31]
    T = sum(lengths)
    q, k, v, do = _inputs(T, 1)
    rows = {0: torch.arange(0, 200), 1: torch.arange(200, 231)}
    scale = 1 / math.sqrt(MODEL.head_dim)
    qa, ka, va = (x.clone().requires_grad_() for x in (q, k, v))
    o, lse = mono_fwd(q, k, v, rows, scale)
    dq, dk, dv = mono_bwd(q, k, v, o, lse, do, rows, scale)
    outs = []
    for idx in rows.values():
        qq = qa[idx].transpose(0, 1)
        kk = ka[idx].repeat_interleave(2, 1).transpose(0, 1)
        vv = va[idx].repeat_interleave(2, 1).transpose(0, 1)
        outs.append((idx, torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=True)))
    loss = sum((y.transpose(0, 1) * do[idx]).sum() for idx, y in outs)
    loss.backward()
    for a, b in ((dq, qa.grad), (dk, ka.grad), (dv, va.grad)):
        assert torch.allclose(a, b, atol=1e-10)


def test_chunk_fwd_bwd_equals_dense():
    """The per-Q-chunk evaluator (bench CPU sample, GPU last-chunk checks) against the dense
    sequence: O/LSE/dQ of the chunk rows; dK/dV of the last chunk's rows are complete."""
    L, m = 700, 170
    q, k, v, do = _inputs(L, 3)
    rows = {0: torch.arange(L)}
    scale = 1 / math.sqrt(MODEL.head_dim)
    o, lse = mono_fwd(q, k, v, rows, scale)
    dq, dk, dv = mono_bwd(q, k, v, o, lse, do, rows, scale)
    for start in (0, 230, L - m):
        qr = torch.arange(start, start + m)
        co, cl, cdq, cdk, cdv = chunk_fwd_bwd(q, k, v, do, qr, torch.arange(start + m), start, scale,
                                              torch.float64)
        assert torch.allclose(co, o[qr], atol=1e-12) and torch.allclose(cl, lse[qr], atol=1e-12)
        assert torch.allclose(cdq, dq[qr], atol=1e-12)
    assert torch.allclose(cdk[L - m:], dk[L - m:], atol=1e-12)
    assert torch.allclose(cdv[L - m:], dv[L - m:], atol=1e-12)


@pytest.mark.parametrize("mask", ["causal", "full"])
def test_tiled_equals_dense(mask):
    r = _schedule([1000, 333, 200, 90, 45], 1, 256, mask)
    lay = build_rank_work(r, 0).layout
    q, k, v, _ = _inputs(lay.tokens, 2)
    scale = 1 / math.sqrt(MODEL.head_dim)
    rows = sequence_rows(r.deps, lay.offset)
    o1, l1 = mono_fwd(q, k, v, rows, scale, causal=(mask == "causal"))
    o2, l2 = tiled_fwd(q, k, v, r.deps, lay.offset, scale)
    assert torch.allclose(o1, o2, atol=1e-10)
    assert torch.allclose(l1, l2, atol=1e-10)


@pytest.mark.parametrize("fuse", [False, True, "all", "resume"])
@pytest.mark.parametrize("n,lengths,block,coalesce,sched", [
    (1, [700, 260, 130, 100, 50, 9], 256, 16, "fcp"),
    (2, [700, 260, 130, 100, 50, 9], 256, 16, "fcp"),
    (3, [1100, 513, 300, 129, 128, 127, 40, 1], 256, 16, "fcp"),
    (3, [1100, 513, 300, 129, 128, 127, 40, 1], 256, 1, "fcp"),     # many stages: fusion matters
    (4, [1100, 513, 300, 129, 128, 127, 40, 9], 256, 1, "ring"),     # relays, unconsumed chunks
    (4, [1100, 513, 300, 129, 128, 127, 40, 9], 256, 1, "bytescale"),
    (8, [1500, 900, 513, 300, 129, 128, 127, 40, 9], 256, 16, "fcp"),  # the driver's N=8 run
    (2, [3000, 1100, 513], 256, 16, "fcp"),     # received groups seen by prefixes (kv_limit)
])
def test_worklist_emulation_matches_dense(n, lengths, block, coalesce, sched, fuse):
    """Simulated workers: per-rank work lists + in-process exchange == dense attention,
    with one forward wave per arrival stage or all remote KV fused into one wave, for FCP
    plans and for the ring / ByteScale plans (relay edges) of baselines.py."""
    r = _schedule(lengths, n, block, coalesce=coalesce, scheduler=sched)
    works = [build_rank_work(r, w, fuse_remote=fuse) for w in range(n)]
    if fuse:
        assert all(sum(1 for wv in wk.fwd.waves if wv.stage >= 0) <= 1 for wk in works)
    if fuse == "all":        # one wave per rank: no partials, no merge
        assert all(len(wk.fwd.waves) == 1 and wk.fwd.partial_rows == 0 for wk in works)
    if fuse == "resume":     # chained partials: no merge groups; some segment continues one
        assert all(len(wk.fwd.merge_groups) == 0 for wk in works)
        if n > 1:
            assert any((wv.segments[:, 5] > 0).any() for wk in works for wv in wk.fwd.waves)
    if lengths[0] == 3000:   # multi-chunk received groups, visited by prefix-limited Q refs
        assert any(k[0] == "recv" and k[3] != k[2] for wk in works for b in wk.bwd for k in b.kv_keys)
        assert any((b.qrefs[:, 3] > 0).any() for wk in works for b in wk.bwd)
    goff, T = global_offsets(r)
    q, k, v, do = _inputs(T, 3)
    scale = 1 / math.sqrt(MODEL.head_dim)
    rows = global_sequence_rows(r)
    o_ref, l_ref = mono_fwd(q, k, v, rows, scale)
    dq_ref, dk_ref, dv_ref = mono_bwd(q, k, v, o_ref, l_ref, do, rows, scale)

    deps = r.deps
    owner = chunk_placement(r.assignment, r.units)
    o = torch.zeros_like(q)
    lse = torch.zeros_like(l_ref)
    dq = torch.zeros_like(q)
    dk_loc, dv_loc, dk_recv, dv_recv = [], [], [], []
    for w, work in enumerate(works):
        lay = work.layout
        ql, kl, vl, dol = (gather_rank(x, lay, goff, deps) for x in (q, k, v, do))
        kr, vr = (gather_rank(x, lay, goff, deps, recv=True) for x in (k, v))
        ow, lw = emulate_forward(work, ql, kl, vl, kr, vr, scale)
        scatter_rank(ow, o, lay, goff, deps)
        scatter_rank(lw, lse, lay, goff, deps)
        dqw, dkw, dvw, dkrw, dvrw = emulate_backward(work, ql, kl, vl, kr, vr, ow, lw, dol, scale)
        scatter_rank(dqw, dq, lay, goff, deps)
        dk_loc.append(dkw)
        dv_loc.append(dvw)
        dk_recv.append(dkrw)
        dv_recv.append(dvrw)
    layouts = [wk.layout for wk in works]
    return_partials(dk_recv, dk_loc, layouts, deps, owner)
    return_partials(dv_recv, dv_loc, layouts, deps, owner)
    dk = torch.zeros_like(k)
    dv = torch.zeros_like(v)
    for w, work in enumerate(works):
        scatter_rank(dk_loc[w], dk, work.layout, goff, deps)
        scatter_rank(dv_loc[w], dv, work.layout, goff, deps)
    for a, b in ((o, o_ref), (lse, l_ref), (dq, dq_ref), (dk, dk_ref), (dv, dv_ref)):
        assert torch.allclose(a, b, atol=1e-9), (a - b).abs().max()
    if n > 1 and fuse not in ("all", "resume"):
        assert any(wk.fwd.partial_rows for wk in works)   # the merge path was exercised


@pytest.mark.parametrize("n", [1, 2, 3])
def test_prewave_for_reshuffle_matches_dense(n):
    """Forward with a PRE_WAVE (the tiles whose chunks stay on their user-layout rank, run
    while the reshuffle into the FCP layout is in flight): emulated == dense, and the pre
    wave is non-empty, so its partials and the extra merge are exercised."""
    from paper_2605_08524_b200.reshuffle import user_layouts
    from paper_2605_08524_b200.worklist import PRE_WAVE
    r = _schedule([1100, 513, 300, 129, 128, 127, 40, 1], n, 256)
    owner = chunk_placement(r.assignment, r.units)
    users = user_layouts(r)
    goff, T = global_offsets(r)
    q, k, v, _ = _inputs(T, 5)
    scale = 1 / math.sqrt(MODEL.head_dim)
    o_ref, l_ref = mono_fwd(q, k, v, global_sequence_rows(r), scale)
    o = torch.zeros_like(q)
    lse = torch.zeros_like(l_ref)
    pre = 0
    for w in range(n):
        resident = {c for c in users[w].chunks if owner[c] == w}
        work = build_rank_work(r, w, resident=resident)
        pre += sum(1 for wv in work.fwd.waves if wv.stage == PRE_WAVE)
        lay = work.layout
        ql, kl, vl = (gather_rank(x, lay, goff, r.deps) for x in (q, k, v))
        kr, vr = (gather_rank(x, lay, goff, r.deps, recv=True) for x in (k, v))
        ow, lw = emulate_forward(work, ql, kl, vl, kr, vr, scale)
        scatter_rank(ow, o, lay, goff, r.deps)
        scatter_rank(lw, lse, lay, goff, r.deps)
        assert work.pairs == build_rank_work(r, w).pairs       # same tiles, regrouped
    assert pre > 0
    assert torch.allclose(o, o_ref, atol=1e-9) and torch.allclose(lse, l_ref, atol=1e-9)


def test_worklist_pairs_match_reference_accounting():
    """Visible pairs of all tiles == batch_token_pairs (reference costmodel.py:196-200)."""
    from paper_2605_08524_b200.costmodel import batch_token_pairs
    lengths = [5000, 2049, 2048, 2047, 300, 1]
    for n in (1, 2, 4):
        r = _schedule(lengths, n, 2048)
        tot = sum(build_rank_work(r, w).pairs for w in range(n))
        assert tot == batch_token_pairs(lengths, "causal")
        tot_b = sum(b.pairs for w in range(n) for b in build_rank_work(r, w).bwd)
        assert tot_b == tot


@pytest.mark.parametrize("curve", ["reference", "b200"])
def test_bench_c2_plans_at_eight_ranks(curve):
    """The driver's scaling run goes to N=8: bench's C2 plan and every rank's work list
    build, and the ranks' tokens partition the batch."""
    import bench
    w, r = bench.build_workload("c2", 8, None, "fcp", curve)
    works = [build_rank_work(r, k) for k in range(8)]
    assert sum(wk.layout.tokens for wk in works) == sum(s.length for s in w.batch().sequences)


def test_kernel_shape_adapter_is_exact():
    """The executor's adapter for shapes the kernels are not compiled for (C1: Hq = Hkv = 4,
    D = 64): head dim zero-padded to 128, every q-head run twice with a zero dO for the copy.
    Through the work-list emulator on the padded shapes at the user's softmax scale, then
    un-padded: equal to dense attention on the original shapes (fp64)."""
    from paper_2605_08524_b200.costmodel import ModelConfig
    from paper_2605_08524_b200.executor import (kernel_config, pad_head_dim, replicate_q_heads,
                                                unreplicate_q)
    tiny = ModelConfig(q_heads=4, kv_heads=4, head_dim=64, dtype_bytes=4)
    kcfg, rep = kernel_config(tiny)
    assert (kcfg.q_heads, kcfg.kv_heads, kcfg.head_dim, rep) == (8, 4, 128, 2)
    tpw = -(-sum([700, 300, 129]) // 2)
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate([700, 300, 129])), 2, tpw)
    r = fcp_schedule(batch, 2, ShardingConfig(256), tiny, DEFAULT_EFFICIENCY)
    goff, T = global_offsets(r)
    g = torch.Generator().manual_seed(11)
    q, k, v, do = (torch.randn((T, 4, 64), generator=g, dtype=torch.float64) for _ in range(4))
    scale = 1 / math.sqrt(64)
    rows = global_sequence_rows(r)
    o_ref, l_ref = mono_fwd(q, k, v, rows, scale)
    dq_ref, dk_ref, dv_ref = mono_bwd(q, k, v, o_ref, l_ref, do, rows, scale)
    owner = chunk_placement(r.assignment, r.units)
    works = [build_rank_work(r, w) for w in range(2)]
    o = torch.zeros_like(q)
    lse = torch.zeros_like(l_ref)
    dq = torch.zeros_like(q)
    dk_loc, dv_loc, dk_recv, dv_recv = [], [], [], []
    for w, work in enumerate(works):
        lay = work.layout
        ql, kl, vl, dol = (gather_rank(x, lay, goff, r.deps) for x in (q, k, v, do))
        kr, vr = (gather_rank(x, lay, goff, r.deps, recv=True) for x in (k, v))
        qa, doa = replicate_q_heads(pad_head_dim(ql), rep), replicate_q_heads(pad_head_dim(dol), rep, True)
        ka, va, kra, vra = (pad_head_dim(x) for x in (kl, vl, kr, vr))
        oa, la = emulate_forward(work, qa, ka, va, kra, vra, scale)
        scatter_rank(unreplicate_q(oa, rep, 64), o, lay, goff, r.deps)
        scatter_rank(unreplicate_q(la, rep, 64), lse, lay, goff, r.deps)
        # the kernels see O of the duplicates as zero too (only dO*O matters: delta = 0)
        oa_in = replicate_q_heads(pad_head_dim(unreplicate_q(oa, rep, 64)), rep, True)
        dqa, dka, dva, dkra, dvra = emulate_backward(work, qa, ka, va, kra, vra, oa_in, la, doa, scale)
        scatter_rank(unreplicate_q(dqa, rep, 64), dq, lay, goff, r.deps)
        dk_loc.append(dka[..., :64])
        dv_loc.append(dva[..., :64])
        dk_recv.append(dkra[..., :64])
        dv_recv.append(dvra[..., :64])
    layouts = [wk.layout for wk in works]
    return_partials(dk_recv, dk_loc, layouts, r.deps, owner)
    return_partials(dv_recv, dv_loc, layouts, r.deps, owner)
    dk = torch.zeros_like(k)
    dv = torch.zeros_like(v)
    for w, work in enumerate(works):
        scatter_rank(dk_loc[w], dk, work.layout, goff, r.deps)
        scatter_rank(dv_loc[w], dv, work.layout, goff, r.deps)
    for a, b in ((o, o_ref), (lse, l_ref), (dq, dq_ref), (dk, dk_ref), (dv, dv_ref)):
        assert torch.allclose(a, b, atol=1e-9), (a - b).abs().max()
