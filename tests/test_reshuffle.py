"""§8f(1) transparent reshuffler, host logic on CPU: the pull plans move every chunk
between the user layout (reference ``default_contiguous_layout``, simulator.py:279-291)
and the FCP layout in both directions, and the bytes they move across ranks equal the
reference accounting of ``reshuffle_cost`` (simulator.py:294-342)."""

import pytest
import torch

from oracle.simworkers import gather_rank, global_offsets
from paper_2605_08524_b200 import configs
from paper_2605_08524_b200.costmodel import B200_HARDWARE, DEFAULT_EFFICIENCY, qkv_bytes_per_token
from paper_2605_08524_b200.pipeline import fcp_schedule
from paper_2605_08524_b200.reshuffle import apply_pulls, moved_bytes, reshuffle_plans, user_layouts
from paper_2605_08524_b200.sharding import ShardingConfig
from paper_2605_08524_b200.simmodel import default_contiguous_layout, reshuffle_cost
from paper_2605_08524_b200.workload import Batch, Sequence
from paper_2605_08524_b200.worklist import rank_layout


def _gather_user(x, lay, goff, deps):
    parts = [x[goff[c]:goff[c] + deps.chunk_tokens[c]] for c in lay.chunks]
    return torch.cat(parts) if parts else x.new_zeros((0,) + tuple(x.shape[1:]))


@pytest.mark.parametrize("name,n,custom", [("c1", 2, False), ("c2", 4, False), ("c2", 8, False),
                                           ("c5", 4, False), ("c2", 4, True)])
def test_round_trip_and_bytes(name, n, custom):
    w = configs.by_name(name, n)
    batch = Batch(tuple(Sequence(i, l) for i, l in enumerate(w.lengths)), n, w.tokens_per_worker)
    r = fcp_schedule(batch, n, ShardingConfig(w.block_size), w.model, DEFAULT_EFFICIENCY)
    init = None
    if custom:   # a scattered user layout: chunk i of the unit order on rank i % n
        keys = [c.key for u in r.units for c in u.members]
        init = {k: i % n for i, k in enumerate(keys)}
    goff, T = global_offsets(r)
    x = torch.arange(T, dtype=torch.float64).unsqueeze(1) * 10 + torch.arange(3)
    users = user_layouts(r, init)
    assert sum(u.tokens for u in users) == T
    fcps = [rank_layout(r, k) for k in range(n)]
    plans = reshuffle_plans(r, init)
    user_x = [_gather_user(x, u, goff, r.deps) for u in users]
    fcp_x = [gather_rank(x, lay, goff, r.deps) for lay in fcps]
    for k, p in enumerate(plans):
        got = apply_pulls(p.to_fcp, user_x, torch.full_like(fcp_x[k], -1))
        assert torch.equal(got, fcp_x[k])
        back = apply_pulls(p.from_fcp, fcp_x, torch.full_like(user_x[k], -1))
        assert torch.equal(back, user_x[k])
    ref = reshuffle_cost(init if init is not None else default_contiguous_layout(r.units, n),
                         r.assignment, r.units, r.deps, B200_HARDWARE, w.model, DEFAULT_EFFICIENCY)
    out_b, in_b = moved_bytes(plans, qkv_bytes_per_token(w.model))
    assert out_b == list(ref.out_bytes) and in_b == list(ref.in_bytes)
