"""TEST INFRASTRUCTURE ONLY: "simulated workers" for the FCP data plane.

Mirrors the reference's testing style (workers are integers in one process):
a global batch laid out sequence by sequence is scattered into each rank's
packed layout, the plan's edges are executed as in-process copies into the
receive arenas, and dK/dV partials travel back along the reversed edges.
Used by the CPU tests (with the work-list emulator) and by the GPU tests
(with the real kernels, several ranks on one device).
"""

from __future__ import annotations

import torch

from oracle.attention_ref import chunk_starts


def global_offsets(result) -> tuple[dict, int]:
    """Canonical order: sequences in batch (unit) order of first appearance,
    positions ascending.  Returns chunk -> first global row, total tokens."""
    deps = result.deps
    starts = chunk_starts(deps)
    seq_len: dict[int, int] = {}
    order: list[int] = []
    for u in result.units:
        for c in u.members:
            if c.seq_id not in seq_len:
                order.append(c.seq_id)
                seq_len[c.seq_id] = 0
            seq_len[c.seq_id] += c.token_count
    seq_base, pos = {}, 0
    for sid in sorted(order):
        seq_base[sid] = pos
        pos += seq_len[sid]
    return {key: seq_base[key[0]] + starts[key] for key in deps.chunk_tokens}, pos


def global_sequence_rows(result) -> dict[int, torch.Tensor]:
    goff, _ = global_offsets(result)
    deps = result.deps
    out: dict[int, list] = {}
    for key in sorted(deps.chunk_tokens):
        out.setdefault(key[0], []).append(
            torch.arange(goff[key], goff[key] + deps.chunk_tokens[key]))
    return {sid: torch.cat(parts) for sid, parts in out.items()}


def gather_rank(x_global, layout, goff, deps, recv=False):
    """Rows of a global [T, ...] tensor in one rank's local (or receive) layout."""
    chunks = layout.recv_chunks if recv else layout.chunks
    if not chunks:
        return x_global.new_zeros((0,) + tuple(x_global.shape[1:]))
    parts = [x_global[goff[c]:goff[c] + deps.chunk_tokens[c]] for c in chunks]
    return torch.cat(parts).contiguous()


def scatter_rank(y_local, x_global, layout, goff, deps):
    """Write a rank's local rows back into the global tensor (in place)."""
    for c in layout.chunks:
        a = layout.offset[c]
        n = deps.chunk_tokens[c]
        x_global[goff[c]:goff[c] + n] = y_local[a:a + n].to(x_global.dtype)


def return_partials(dkv_recv_by_rank, dkv_local_by_rank, layouts, deps, owner):
    """dK/dV return + reduce (K6 + K4, in-process): every received chunk's
    partial is added into its owner's local accumulator."""
    for r, lay in enumerate(layouts):
        part = dkv_recv_by_rank[r]
        if part is None:
            continue
        for c in lay.recv_chunks:
            if c not in lay.consumed:       # relayed only: no partial exists
                continue
            o = owner[c]
            a = lay.recv_offset[c]
            n = deps.chunk_tokens[c]
            b = layouts[o].offset[c]
            dkv_local_by_rank[o][b:b + n] += part[a:a + n].to(dkv_local_by_rank[o].dtype)
