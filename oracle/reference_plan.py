"""TEST INFRASTRUCTURE ONLY: load the *unmodified* reference ``blocksched``.

The reference package (``/root/reference/pkg/src/blocksched``) is pure Python;
it is imported here under the alias ``blocksched_ref`` (its modules use
relative imports, so a renamed copy behaves identically) to act as the
control-plane oracle: the FCP plan (units, placement, Delta-matching rounds)
must be bit-identical to what it emits.  Available only in the build
container -- the GPU box has no ``/root/reference``; there the committed
golden fixtures under ``tests/golden/`` stand in for it.
"""

from __future__ import annotations

import hashlib
import importlib
import json
import os
import shutil
import sys
import tempfile

REFERENCE_SRC = "/root/reference/pkg/src/blocksched"
ALIAS = "blocksched_ref"


def available() -> bool:
    return os.path.isdir(REFERENCE_SRC)


def load():
    """Import the reference package as ``blocksched_ref`` (cached)."""
    if ALIAS in sys.modules:
        return sys.modules[ALIAS]
    if not available():
        raise ImportError("reference package not present (GPU box?)")
    root = tempfile.mkdtemp(prefix="refpkg_")
    shutil.copytree(REFERENCE_SRC, os.path.join(root, ALIAS))
    sys.path.insert(0, root)
    try:
        pkg = importlib.import_module(ALIAS)
        for sub in ("cli", "pipeline", "simulator", "metrics", "planner",
                    "distributor", "sharding", "costmodel", "workload"):
            importlib.import_module(f"{ALIAS}.{sub}")
    finally:
        sys.path.remove(root)
    return pkg


def reference_digest(lengths, n, tpw, block, model_kw, mask="causal", coalesce_degree=16,
                     curve_anchors=None):
    """sha256[:16] of the reference's canonical schedule+plan JSON.  curve_anchors: an
    efficiency curve for the reference's EfficiencyCurve (default: its DEFAULT_EFFICIENCY)."""
    ref = load()
    cli = sys.modules[f"{ALIAS}.cli"]
    model = ref.ModelConfig(**model_kw)
    batch = ref.Batch(tuple(ref.Sequence(i, l) for i, l in enumerate(lengths)), n, tpw)
    curve = ref.DEFAULT_EFFICIENCY if curve_anchors is None else \
        sys.modules[f"{ALIAS}.costmodel"].EfficiencyCurve(tuple(tuple(a) for a in curve_anchors))
    r = ref.fcp_schedule(batch, n, ref.ShardingConfig(block_size=block, mask=mask), model,
                         curve, coalesce_degree=coalesce_degree)
    blob = json.dumps([cli.schedule_payload(r, model),
                       cli.plan_payload(r.sub_stage_plan, r.plan.degree)], sort_keys=True)
    return hashlib.sha256(blob.encode()).hexdigest()[:16], r
