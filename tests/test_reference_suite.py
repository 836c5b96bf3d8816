"""Run the reference's own hot-path tests, unchanged, against the drop-in.

``pkg/tests/test_{sharding,costmodel,distributor,planner,pipeline,simulator,baselines}.py``
import ``blocksched``; with the repo root first on ``PYTHONPATH`` that name is
the alias package ``blocksched/`` over ``paper_2605_08524_b200``.  Skipped
where the reference checkout is absent (the GPU box).
"""

import os
import shutil
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOT_PATH = ["test_sharding.py", "test_costmodel.py", "test_distributor.py",
            "test_planner.py", "test_pipeline.py", "test_simulator.py",
            "test_baselines.py"]                        # §8f-2: competitor plans


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference checkout absent")
def test_reference_hot_path_suite_passes(tmp_path):
    dst = tmp_path / "reftests"
    shutil.copytree(REF_TESTS, dst)
    env = dict(os.environ, PYTHONPATH=ROOT)
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                           *HOT_PATH], cwd=dst, env=env, capture_output=True, text=True,
                          timeout=900)
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-2000:]
    probe = subprocess.run([sys.executable, "-c",
                            "import blocksched.planner as p; print(p.__name__)"],
                           cwd=dst, env=env, capture_output=True, text=True)
    assert probe.stdout.strip() == "paper_2605_08524_b200.planner"
