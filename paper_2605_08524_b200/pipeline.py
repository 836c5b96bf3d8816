"""``fcp_schedule``: the control-plane entry point (reference ``pipeline.py:31-60``).

shard -> dependency map -> efficiency-weighted loads -> LPT placement (on
``InfeasibleError`` the memory slack doubles, ``delta = max(2*delta, 0.01)``,
up to ``delta_retries`` times) -> transfer multigraph -> Delta matchings ->
density ordering -> coalescing into stages of ``coalesce_degree`` rounds.

The returned ``ScheduleResult`` is what ``worklist.build_rank_worklists`` turns
into device tile tables and what ``exchange`` executes; it is computed once
per batch and shared by every attention layer.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, replace

from .costmodel import EfficiencyCurve, ModelConfig, unit_costs
from .distributor import AssignParams, Assignment, assign, effective_unit_loads
from .errors import InfeasibleError
from .errors import ConsistencyError, ParameterError
from .planner import (CoalescedPlan, CommPlan, Edge, build_comm_graph, coalesce,
                      decompose_matchings, stage_ordering)
from .sharding import Chunk, DependencyMap, ScheduleUnit, ShardingConfig, kv_dependencies, shard_batch
from .workload import Batch

DEFAULT_COALESCE_DEGREE = 16

SCHEDULE_FORMAT = "blocksched.schedule/1"
PLAN_FORMAT = "blocksched.plan/1"


@dataclass
class ScheduleResult:
    label: str
    units: list[ScheduleUnit]
    deps: DependencyMap
    assignment: Assignment
    sub_stage_plan: CommPlan
    plan: CoalescedPlan
    params: AssignParams | None = None


def fcp_schedule(batch: Batch, n_workers: int, sharding: ShardingConfig,
                 cfg: ModelConfig, curve: EfficiencyCurve,
                 params: AssignParams | None = None,
                 coalesce_degree: int = DEFAULT_COALESCE_DEGREE,
                 delta_retries: int = 3) -> ScheduleResult:
    if params is None:
        params = AssignParams(mem_limit=float(batch.tokens_per_worker))
    units = shard_batch(batch, sharding)
    deps = kv_dependencies(units, sharding.mask)
    loads = effective_unit_loads(units, deps, cfg, curve)
    tried = params
    attempt = 0
    while True:
        try:
            placement = assign(loads, n_workers, tried)
            break
        except InfeasibleError:
            if attempt == delta_retries:
                raise
            attempt += 1
            tried = replace(tried, delta=max(tried.delta * 2, 0.01))
    graph = build_comm_graph(placement, deps, units, cfg)
    rounds = stage_ordering(decompose_matchings(graph))
    return ScheduleResult("fcp", units, deps, placement, rounds,
                          coalesce(rounds, coalesce_degree), tried)


# ---------------------------------------------------------------------------
# Wire formats (reference cli.py:214-250): the canonical serialisation used to
# prove plan parity and to hand precomputed plans to the executor.

def schedule_payload(result: ScheduleResult, cfg: ModelConfig) -> dict:
    units = [{"unit_id": u.unit_id, "kind": u.kind,
              "members": [[c.seq_id, c.chunk_index, c.token_count] for c in u.members]}
             for u in result.units]
    rows = []
    for u in result.units:
        cost = unit_costs(u, result.deps, cfg)
        rows.append([u.unit_id, result.assignment.worker_of(u.unit_id),
                     cost.memory, cost.compute])
    return {"format": SCHEDULE_FORMAT, "scheduler": result.label,
            "n_workers": result.assignment.n_workers, "mask": result.deps.mask,
            "units": units, "assignment": rows}


def plan_payload(plan: CommPlan, degree: int) -> dict:
    return {"format": PLAN_FORMAT, "n_workers": plan.n, "coalesce_degree": degree,
            "sub_stages": [[[e.src, e.dst, e.nbytes, [list(c) for c in e.chunks]]
                            for e in rnd] for rnd in plan.sub_stages]}


def plan_digest(result: ScheduleResult, cfg: ModelConfig) -> str:
    """sha256[:16] of the canonical schedule+plan JSON."""
    blob = json.dumps([schedule_payload(result, cfg),
                       plan_payload(result.sub_stage_plan, result.plan.degree)],
                      sort_keys=True)
    return hashlib.sha256(blob.encode()).hexdigest()[:16]


def result_from_payloads(schedule: dict, plan: dict) -> ScheduleResult:
    """Inverse of the wire formats (reference ``cli.py:226-258``,
    ``load_schedule``/``load_plan``): rebuild a ScheduleResult the executor runs directly
    from a precomputed schedule and plan, e.g. the reference CLI's ``schedule.json`` and
    ``plan.json``.  Dependencies are rederived from the units and mask
    (``kv_dependencies``); the coalesced stages from the stored degree."""
    if schedule.get("format") != SCHEDULE_FORMAT:
        raise ParameterError("not a blocksched.schedule/1 payload")
    if plan.get("format") != PLAN_FORMAT:
        raise ParameterError("not a blocksched.plan/1 payload")
    n = schedule["n_workers"]
    if plan["n_workers"] != n:
        raise ConsistencyError(f"schedule has {n} workers, plan {plan['n_workers']}")
    units = [ScheduleUnit(u["unit_id"], u["kind"], tuple(Chunk(*m) for m in u["members"]))
             for u in schedule["units"]]
    deps = kv_dependencies(units, schedule["mask"])
    mapping: dict[int, int] = {}
    memory, compute = [0.0] * n, [0.0] * n
    for unit_id, worker, mem, comp in schedule["assignment"]:
        mapping[unit_id] = worker
        memory[worker] += mem
        compute[worker] += comp
    if set(mapping) != {u.unit_id for u in units}:
        raise ConsistencyError("assignment does not cover exactly the schedule's units")
    rounds = CommPlan(n, [[Edge(src, dst, tuple(tuple(c) for c in chunks), nbytes)
                           for src, dst, nbytes, chunks in rnd] for rnd in plan["sub_stages"]])
    return ScheduleResult(schedule.get("scheduler", "fcp"), units, deps,
                          Assignment(n, mapping, memory, compute), rounds,
                          coalesce(rounds, plan["coalesce_degree"]), None)


def load_schedule_result(schedule_path, plan_path) -> ScheduleResult:
    """``result_from_payloads`` on the reference CLI's artifact files."""
    with open(schedule_path, "r", encoding="utf-8") as fh:
        sched = json.load(fh)
    with open(plan_path, "r", encoding="utf-8") as fh:
        pl = json.load(fh)
    return result_from_payloads(sched, pl)
