"""Drop-in alias: ``import blocksched`` resolves to the B200-native package.

The reference API (``pkg/src/blocksched/__init__.py:4-20``) is served by
``paper_2605_08524_b200``; each reference submodule name is bound to the
corresponding module here so ``from blocksched.planner import ...`` and the
reference's own tests run unchanged against this implementation.
"""

import importlib
import sys

_IMPL = "paper_2605_08524_b200"
_SUBMODULES = {
    "errors": "errors", "workload": "workload", "sharding": "sharding",
    "costmodel": "costmodel", "distributor": "distributor", "planner": "planner",
    "pipeline": "pipeline", "simulator": "simmodel", "metrics": "metrics",
    "baselines": "baselines",
}
for _name, _target in _SUBMODULES.items():
    _mod = importlib.import_module(f"{_IMPL}.{_target}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

from paper_2605_08524_b200.api import *  # noqa: E402,F401,F403

__version__ = "0.1.0+b200"
