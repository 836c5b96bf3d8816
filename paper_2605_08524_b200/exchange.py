"""K5/K6 plan bookkeeping: which rows the coalesced Delta-matching plan moves.

Each coalesced stage of ``ScheduleResult.plan`` (reference ``planner.py:234-248``) moves
every KV chunk on an edge ``dst == rank`` into that chunk's receive-arena slot
(``worklist.rank_layout``).  Every round of a stage is a matching, so within a stage each
GPU sends at most ``degree`` and receives at most ``degree`` chunks -- over NVSwitch
(uniform 900 GB/s per direction to every peer) this is the congestion-free schedule the
reference models with its flat full-duplex NIC (``simulator.py:136-151``).

The backward return (K6) walks the same edges reversed: the consumer's dK/dV partial of a
chunk goes back to the owner, which adds it with K4.  ``owner_returns`` and
``return_staging_layout`` describe that traffic; ``p2p.py`` turns both directions into
copy-engine pulls.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from .pipeline import ScheduleResult
from .worklist import RankLayout


@dataclass
class Transfer:
    peer: int
    row: int          # first token row (local buffer for sends, receive arena for recvs)
    tokens: int
    chunk: tuple[int, int]
    from_recv: bool = False   # a relay send (ring / ByteScale): the rows sit in the receive arena


@dataclass
class StageOps:
    sends: list[Transfer] = field(default_factory=list)
    recvs: list[Transfer] = field(default_factory=list)

    @property
    def empty(self) -> bool:
        return not self.sends and not self.recvs


def build_stage_ops(result: ScheduleResult, lay: RankLayout, all_layouts=None) -> list[StageOps]:
    """Per coalesced stage, this rank's sends (from its local rows) and receives
    (into its receive arena), in plan edge order."""
    rank = lay.rank
    out = []
    for s, stage in enumerate(result.plan.stages):
        ops = StageOps()
        for e in stage:
            for c in e.chunks:
                n = lay.chunk_tokens[c]
                if e.src == rank:
                    if c in lay.offset:
                        ops.sends.append(Transfer(e.dst, lay.offset[c], n, c))
                    else:                   # relay: forwarded from the receive arena
                        ops.sends.append(Transfer(e.dst, lay.recv_offset[c], n, c, True))
                if e.dst == rank and lay.recv_stage.get(c) == s:
                    ops.recvs.append(Transfer(e.src, lay.recv_offset[c], n, c))
        out.append(ops)
    return out


def owner_returns(layouts, owner, rank: int) -> list[Transfer]:
    """K6, owner side: one transfer per (my chunk, rank that consumed it), in consumer rank
    order then that rank's receive order.  ``row`` is the chunk's row in my local buffer,
    ``peer`` the consumer.  Owner-centric, so relay plans (where the edge sender is not
    the owner) return every partial to the right rank."""
    out = []
    for q, lay in enumerate(layouts):
        if q == rank:
            continue
        for c in lay.recv_chunks:
            if c in lay.consumed and owner[c] == rank:
                out.append(Transfer(q, layouts[rank].offset[c], lay.chunk_tokens[c], c))
    return out


def return_staging_layout(returns: list[Transfer]):
    """Owner-side staging for returned dK/dV partials (``returns`` from ``owner_returns``).

    Returns (rows, rounds, total): ``rows[(chunk, peer)]`` is the first staging row of
    that peer's partial; ``rounds`` is a list of (src_rows, dst_rows) pairs where round
    k holds the k-th consumer of every chunk, so within a round every destination row
    appears once (K4 launches per round are race-free and sum in a fixed order).
    """
    rows, pos = {}, 0
    per_chunk: dict = {}
    for t in returns:
        rows[(t.chunk, t.peer)] = pos
        per_chunk.setdefault(t.chunk, []).append((t.row, pos, t.tokens))
        pos += t.tokens
    rounds: list[tuple[list[int], list[int]]] = []
    for parts in per_chunk.values():
        for k, (dst0, src0, n) in enumerate(parts):
            while len(rounds) <= k:
                rounds.append(([], []))
            rounds[k][0].extend(range(src0, src0 + n))
            rounds[k][1].extend(range(dst0, dst0 + n))
    return rows, rounds, pos


def exchange_bytes(stages: list[StageOps], bytes_per_token: int) -> tuple[int, int]:
    sent = sum(t.tokens for st in stages for t in st.sends) * bytes_per_token
    got = sum(t.tokens for st in stages for t in st.recvs) * bytes_per_token
    return sent, got


def sync_plan_digest(digest: str, group=None) -> None:
    """All ranks must hold the same plan: all-gather its hash (cheap, once per batch)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    mine = torch.tensor([int(digest, 16) & ((1 << 62) - 1)], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        mine = mine.cuda()
    got = [torch.zeros_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(got, mine, group=group)
    if any(int(x.item()) != int(mine.item()) for x in got):
        from .errors import ConsistencyError
        raise ConsistencyError("ranks disagree on the FCP plan (hash mismatch)")
