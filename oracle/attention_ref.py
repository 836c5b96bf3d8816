"""TEST INFRASTRUCTURE ONLY: CPU restatement of FCP block attention (the oracle).

The reference package contains no attention arithmetic (its data
plane is the analytic ``simulate``), so this oracle restates the math of the
paper on the reference's data model:

* formula: O = softmax(Q K^T * scale (+ causal mask)) V, scale = 1/sqrt(D)
  (``PAPER.md:172-187``); LSE = log sum exp of the scaled scores (natural log);
* chunk geometry: chunks are contiguous token ranges of a sequence with sizes
  ``chunk_token_counts`` (reference ``sharding.py:91-111``); packed short
  sequences are whole sequences (``sharding.py:114-140``);
* tile set: the (Q chunk, KV chunk) pairs of ``kv_dependencies``
  (``sharding.py:172-201``); a causal diagonal tile keeps j <= i
  (``costmodel.py:141-149``);
* GQA: q-head h reads kv-head h // (Hq/Hkv) (convention; the reference is silent).

Three levels, each checked against the previous one in ``tests/``:
  1. ``mono_*``      per-sequence dense attention (float64 or float32, torch; it runs on
                     the device its inputs live on -- the GPU suites feed it CUDA fp64
                     tensors so the fp64 checker takes seconds, not minutes);
  2. ``tiled_fwd``   the same computed tile by tile with an LSE merge;
  3. ``emulate_*``   an interpreter of the device work lists (``worklist.py``)
                     that walks segments / KV refs / 128-row items exactly as the
                     kernels do, with in-process copies standing in for the
                     NVLink exchange ("simulated workers", like the reference's
                     integer workers).

Parity status: the control plane is pinned bit-for-bit by the reference; the
attention *values* are unpinned by any reference fixture (none exist) and are
pinned here against torch's own SDPA (``tests/test_oracle.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may use it.
"""

from __future__ import annotations

import math

import torch

TILE = 128


# ---------------------------------------------------------------------------- layout helpers
def chunk_starts(deps) -> dict:
    """(seq, chunk) -> first position of the chunk inside its sequence."""
    by_seq: dict[int, list] = {}
    for key in deps.chunk_tokens:
        by_seq.setdefault(key[0], []).append(key)
    starts = {}
    for keys in by_seq.values():
        pos = 0
        for key in sorted(keys, key=lambda k: k[1]):
            starts[key] = pos
            pos += deps.chunk_tokens[key]
    return starts


def sequence_rows(deps, offset: dict) -> dict[int, torch.Tensor]:
    """seq id -> packed-buffer row index of every position, in position order,
    for a packed layout ``offset`` (chunk -> first row)."""
    by_seq: dict[int, list] = {}
    for key in deps.chunk_tokens:
        if key in offset:
            by_seq.setdefault(key[0], []).append(key)
    rows = {}
    for sid, keys in by_seq.items():
        parts = [torch.arange(offset[k], offset[k] + deps.chunk_tokens[k])
                 for k in sorted(keys, key=lambda k: k[1])]
        rows[sid] = torch.cat(parts)
    return rows


# ---------------------------------------------------------------------------- level 1: dense
def _expand_kv(x, group):
    return x.repeat_interleave(group, dim=1) if group > 1 else x


def mono_fwd(q, k, v, rows, scale, causal=True, dtype=torch.float64):
    """Dense per-sequence attention over packed buffers.  Returns (O, LSE).

    One (sequence, head) at a time so the L x L score matrix stays bounded."""
    T, H, D = q.shape
    group = H // k.shape[1]
    dev = q.device        # the oracle's arithmetic runs wherever its inputs live (fp64 either way)
    o = torch.zeros((T, H, D), dtype=dtype, device=dev)
    lse = torch.full((T, H), -math.inf, dtype=dtype, device=dev)
    for idx in rows.values():
        idx = idx.to(dev)
        L = idx.numel()
        keep = torch.ones(L, L, dtype=torch.bool, device=dev).tril() if causal else None
        for h in range(H):
            qs = q[idx, h].to(dtype)
            ks = k[idx, h // group].to(dtype)
            vs = v[idx, h // group].to(dtype)
            s = torch.matmul(qs, ks.T) * scale
            if keep is not None:
                s = s.masked_fill(~keep, -math.inf)
            m = s.amax(dim=-1, keepdim=True)
            p = torch.exp(s - m)
            l = p.sum(dim=-1, keepdim=True)
            o[idx, h] = torch.matmul(p, vs) / l
            lse[idx, h] = (m + torch.log(l)).squeeze(-1)
    return o, lse


def mono_bwd(q, k, v, o, lse, do, rows, scale, causal=True, dtype=torch.float64):
    """Dense per-sequence backward.  Returns (dQ, dK, dV) in ``dtype``."""
    T, H, D = q.shape
    Hk = k.shape[1]
    group = H // Hk
    dev = q.device
    dq = torch.zeros((T, H, D), dtype=dtype, device=dev)
    dk = torch.zeros((T, Hk, D), dtype=dtype, device=dev)
    dv = torch.zeros((T, Hk, D), dtype=dtype, device=dev)
    for idx in rows.values():
        idx = idx.to(dev)
        L = idx.numel()
        keep = torch.ones(L, L, dtype=torch.bool, device=dev).tril() if causal else None
        for h in range(H):
            kh = h // group
            qs = q[idx, h].to(dtype)
            ks = k[idx, kh].to(dtype)
            vs = v[idx, kh].to(dtype)
            dos = do[idx, h].to(dtype)
            p = torch.exp(torch.matmul(qs, ks.T) * scale - lse[idx, h].to(dtype).unsqueeze(1))
            if keep is not None:
                p = p.masked_fill(~keep, 0.0)
            delta = (dos * o[idx, h].to(dtype)).sum(-1, keepdim=True)
            ds = p * (torch.matmul(dos, vs.T) - delta)
            dq[idx, h] = torch.matmul(ds, ks) * scale
            dk[idx, kh] += torch.matmul(ds.T, qs) * scale
            dv[idx, kh] += torch.matmul(p.T, dos)
    return dq, dk, dv


def chunk_fwd_bwd(q, k, v, do, q_rows, kv_rows, diag_from, scale, dtype=torch.float32):
    """One Q chunk's whole fwd+bwd against its concatenated KV list, head by head (the CPU
    timing sample of ``bench.py``; the reference's unit of work is a Q chunk with its
    ``q_to_kv`` list, ``sharding.py:172-201``).  ``q_rows``/``kv_rows``: row indices into the
    packed buffers; the last ``len(kv_rows) - diag_from`` KV rows are the diagonal chunk
    (inclusive causal mask ``j <= i``, ``costmodel.py:141-149``), the ones before it are fully
    visible.  Returns (O, LSE, dQ, dK_part, dV_part) for those rows."""
    H, Hk = q.shape[1], k.shape[1]
    group = H // Hk
    qn, kn = q_rows.numel(), kv_rows.numel()
    dev = q.device
    q_rows, kv_rows = q_rows.to(dev), kv_rows.to(dev)
    keep = torch.ones(qn, kn, dtype=torch.bool, device=dev)
    keep[:, diag_from:] = torch.ones(qn, kn - diag_from, dtype=torch.bool, device=dev).tril()
    D = q.shape[2]
    o = torch.empty((qn, H, D), dtype=dtype, device=dev)
    lse = torch.empty((qn, H), dtype=dtype, device=dev)
    dq = torch.empty((qn, H, D), dtype=dtype, device=dev)
    dk = torch.zeros((kn, Hk, D), dtype=dtype, device=dev)
    dv = torch.zeros((kn, Hk, D), dtype=dtype, device=dev)
    for h in range(H):
        kh = h // group
        qs, dos = q[q_rows, h].to(dtype), do[q_rows, h].to(dtype)
        ks, vs = k[kv_rows, kh].to(dtype), v[kv_rows, kh].to(dtype)
        s = (torch.matmul(qs, ks.T) * scale).masked_fill(~keep, -math.inf)
        m = s.amax(dim=-1, keepdim=True)
        p = torch.exp(s - m)
        l = p.sum(dim=-1, keepdim=True)
        p = p / l
        oh = torch.matmul(p, vs)
        o[:, h], lse[:, h] = oh, (m + torch.log(l)).squeeze(-1)
        ds = p * (torch.matmul(dos, vs.T) - (dos * oh).sum(-1, keepdim=True))
        dq[:, h] = torch.matmul(ds, ks) * scale
        dk[:, kh] += torch.matmul(ds.T, qs) * scale
        dv[:, kh] += torch.matmul(p.T, dos)
    return o, lse, dq, dk, dv


# ---------------------------------------------------------------------------- level 2: tiles
def tiled_fwd(q, k, v, deps, offset, scale, dtype=torch.float64):
    """Attention evaluated tile by tile over ``deps.q_to_kv`` with an LSE merge."""
    T, H, D = q.shape
    group = H // k.shape[1]
    causal = deps.mask == "causal"
    o = torch.zeros((T, H, D), dtype=dtype)
    lse = torch.full((T, H), -math.inf, dtype=dtype)
    for qk, kvs in deps.q_to_kv.items():
        if qk not in offset:
            continue
        qa, qn = offset[qk], deps.chunk_tokens[qk]
        qs = q[qa:qa + qn].to(dtype).transpose(0, 1)
        parts = []
        for kv in kvs:
            ka, kn = offset[kv], deps.chunk_tokens[kv]
            ks = _expand_kv(k[ka:ka + kn].to(dtype), group).transpose(0, 1)
            vs = _expand_kv(v[ka:ka + kn].to(dtype), group).transpose(0, 1)
            s = torch.matmul(qs, ks.transpose(1, 2)) * scale
            if causal and kv == qk:
                s = s.masked_fill(~torch.ones(qn, kn, dtype=torch.bool).tril(), -math.inf)
            m = s.amax(-1, keepdim=True)
            p = torch.exp(s - m)
            l = p.sum(-1, keepdim=True)
            parts.append((torch.matmul(p, vs) / l, (m + torch.log(l))))
        lses = torch.stack([pl for _, pl in parts])                   # [n, H, qn, 1]
        tot = torch.logsumexp(lses, dim=0)
        acc = sum(torch.exp(pl - tot) * po for po, pl in parts)
        o[qa:qa + qn] = acc.transpose(0, 1)
        lse[qa:qa + qn] = tot.squeeze(-1).transpose(0, 1)
    return o, lse


# ---------------------------------------------------------------------------- level 3: work lists
def _tile_scores(qs, ks, scale, row0, col0, q_len, kv_len, diag):
    """Scores of a 128x128 block with the kernel's masking rules."""
    s = torch.matmul(qs, ks.transpose(-1, -2)) * scale
    r = torch.arange(qs.shape[-2]).unsqueeze(1) + row0
    c = torch.arange(ks.shape[-2]).unsqueeze(0) + col0
    vis = (c < kv_len) & (r < q_len)
    if diag:
        vis = vis & (c <= r)
    return s.masked_fill(~vis, -math.inf), vis


def emulate_forward(work, q, k, v, k_recv, v_recv, scale, dtype=torch.float64):
    """Interpret ``work.fwd`` (waves -> segments -> kv refs -> 128-row items) on
    the CPU, producing exactly what the kernels are specified to produce:
    final (O, LSE) for single-wave chunks, fp32 partials + K3 merge otherwise."""
    T, H, D = q.shape
    group = H // k.shape[1]
    f = work.fwd
    o = torch.zeros((T, H, D), dtype=dtype)
    lse = torch.full((T, H), -math.inf, dtype=dtype)
    op = torch.zeros((f.partial_rows, H, D), dtype=dtype)
    lp = torch.full((f.partial_rows, H), -math.inf, dtype=dtype)
    for wave in f.waves:
        for seg_idx, mb in wave.items.tolist():
            q_off, q_len, kb, ke, out_row, in_row = wave.segments[seg_idx].tolist()
            r0 = mb * TILE
            nrow = min(TILE, q_len - r0)
            qs = q[q_off + r0:q_off + r0 + nrow].to(dtype).transpose(0, 1)     # [H, n, D]
            s_all, v_all = [], []
            for ref in wave.kvrefs[kb:ke].tolist():
                off, kn, flags, _ = ref
                src_k, src_v = (k_recv, v_recv) if flags & 2 else (k, v)
                diag = bool(flags & 1)
                ntile = -(-kn // TILE)
                if diag:
                    ntile = min(ntile, mb + 1)
                for t in range(ntile):
                    c0 = t * TILE
                    cn = min(TILE, kn - c0)
                    ks = _expand_kv(src_k[off + c0:off + c0 + cn].to(dtype), group).transpose(0, 1)
                    vs = _expand_kv(src_v[off + c0:off + c0 + cn].to(dtype), group).transpose(0, 1)
                    s, _ = _tile_scores(qs, ks, scale, r0, c0, q_len, kn, diag)
                    s_all.append(s)
                    v_all.append(vs)
            s = torch.cat(s_all, dim=-1)
            vv = torch.cat(v_all, dim=-2)
            m = s.amax(-1, keepdim=True)
            p = torch.exp(s - m)
            l = p.sum(-1, keepdim=True)
            out = (torch.matmul(p, vv) / l).transpose(0, 1)
            ls = (m + torch.log(l)).squeeze(-1).transpose(0, 1)
            if in_row > 0:     # continue an earlier wave's partial (worklist fuse_remote="resume")
                pr = slice(in_row - 1 + r0, in_row - 1 + r0 + nrow)
                l0, o0 = lp[pr], op[pr]
                tot = torch.logaddexp(l0, ls)
                out = torch.exp(l0 - tot).unsqueeze(-1) * o0 + torch.exp(ls - tot).unsqueeze(-1) * out
                ls = tot
            if out_row < 0:
                o[q_off + r0:q_off + r0 + nrow] = out
                lse[q_off + r0:q_off + r0 + nrow] = ls
            else:
                op[out_row + r0:out_row + r0 + nrow] = out
                lp[out_row + r0:out_row + r0 + nrow] = ls
    for q_off, q_len, pb, pe, _, _ in f.merge_groups.tolist():
        rows = f.merge_part_rows[pb:pe].tolist()
        lses = torch.stack([lp[r:r + q_len] for r in rows])
        tot = torch.logsumexp(lses, dim=0)
        acc = sum(torch.exp(lses[i] - tot).unsqueeze(-1) * op[r:r + q_len] for i, r in enumerate(rows))
        o[q_off:q_off + q_len] = acc
        lse[q_off:q_off + q_len] = tot
    return o, lse


def emulate_backward(work, q, k, v, k_recv, v_recv, o, lse, do, scale, dtype=torch.float64):
    """Interpret the backward work lists on the CPU: ``work.bwd`` (KV-keyed dK/dV
    launches) and ``work.dq`` (query-stationary dQ).  Returns local (dQ, dK, dV)
    and the received chunks' (dK, dV) partials."""
    T, H, D = q.shape
    Hk = k.shape[1]
    group = H // Hk
    R = 0 if k_recv is None else k_recv.shape[0]
    delta = (do.to(dtype) * o.to(dtype)).sum(-1)                          # [T, H]
    dq = torch.zeros((T, H, D), dtype=dtype)
    dk = torch.zeros((T, Hk, D), dtype=dtype)
    dv = torch.zeros((T, Hk, D), dtype=dtype)
    dkr = torch.zeros((R, Hk, D), dtype=dtype)
    dvr = torch.zeros((R, Hk, D), dtype=dtype)
    for launch in work.bwd:
        for kidx, nb in launch.items.tolist():
            kv_off, kv_len, flags, qb, qe, _ = launch.kvsegs[kidx].tolist()
            src_k, src_v = (k_recv, v_recv) if flags & 2 else (k, v)
            c0 = nb * TILE
            cn = min(TILE, kv_len - c0)
            kk = src_k[kv_off + c0:kv_off + c0 + cn].to(dtype)                 # [cn, Hk, D]
            vv = src_v[kv_off + c0:kv_off + c0 + cn].to(dtype)
            gk = torch.zeros((cn, Hk, D), dtype=dtype)
            gv = torch.zeros((cn, Hk, D), dtype=dtype)
            for q_off, q_len, diag, kv_limit in launch.qrefs[qb:qe].tolist():
                if kv_limit and c0 >= kv_limit:   # a received group's prefix (worklist._group_received)
                    continue
                kv_end = min(kv_len, kv_limit) if kv_limit else kv_len
                first = nb if diag else 0
                for mb in range(first, -(-q_len // TILE)):
                    r0 = mb * TILE
                    nrow = min(TILE, q_len - r0)
                    sl = slice(q_off + r0, q_off + r0 + nrow)
                    for h in range(H):
                        kh = h // group
                        qs = q[sl, h].to(dtype)
                        s, vis = _tile_scores(qs, kk[:, kh], scale, r0, c0, q_len, kv_end, bool(diag))
                        p = torch.exp(s - lse[sl, h].to(dtype).unsqueeze(1)).masked_fill(~vis, 0.0)
                        dp = torch.matmul(do[sl, h].to(dtype), vv[:, kh].transpose(0, 1))
                        ds = p * (dp - delta[sl, h].unsqueeze(1))
                        gk[:, kh] += torch.matmul(ds.transpose(0, 1), qs) * scale
                        gv[:, kh] += torch.matmul(p.transpose(0, 1), do[sl, h].to(dtype))
            dst_k, dst_v = (dkr, dvr) if flags & 2 else (dk, dv)
            dst_k[kv_off + c0:kv_off + c0 + cn] = gk
            dst_v[kv_off + c0:kv_off + c0 + cn] = gv
    # dQ: query-stationary tables (work.dq) -- one 128-row item per Q chunk block
    d = work.dq
    for seg_idx, mb in d.items.tolist():
        q_off, q_len, kb, ke, _, _ = d.segments[seg_idx].tolist()
        r0 = mb * TILE
        nrow = min(TILE, q_len - r0)
        sl = slice(q_off + r0, q_off + r0 + nrow)
        for ref in d.kvrefs[kb:ke].tolist():
            off, kn, flags, _ = ref
            src_k, src_v = (k_recv, v_recv) if flags & 2 else (k, v)
            diag = bool(flags & 1)
            ntile = -(-kn // TILE)
            if diag:
                ntile = min(ntile, mb + 1)
            for t in range(ntile):
                c0 = t * TILE
                cn = min(TILE, kn - c0)
                for h in range(H):
                    kh = h // group
                    kk = src_k[off + c0:off + c0 + cn, kh].to(dtype)
                    vv = src_v[off + c0:off + c0 + cn, kh].to(dtype)
                    s, vis = _tile_scores(q[sl, h].to(dtype), kk, scale, r0, c0, q_len, kn, diag)
                    p = torch.exp(s - lse[sl, h].to(dtype).unsqueeze(1)).masked_fill(~vis, 0.0)
                    dp = torch.matmul(do[sl, h].to(dtype), vv.transpose(0, 1))
                    ds = p * (dp - delta[sl, h].unsqueeze(1))
                    dq[sl, h] += torch.matmul(ds, kk) * scale
    return dq, dk, dv, dkr, dvr
