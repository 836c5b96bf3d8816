"""Multi-GPU executor parity (NCCL over NVLink): runs tests/mp_gpu_check.py under
torchrun on 2 GPUs (and 4 if present).  Skipped on boxes with fewer GPUs."""

import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,sched", [(2, "fcp"), (4, "fcp"), (4, "ring")])
def test_executor_nccl_parity(n, sched):
    """FCP plans, and the ring plan of baselines.py (relay edges, relayed-only chunks)."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_gpu_check.py")]
    proc = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600,
                          env=dict(os.environ, FCPB_CHECK_SCHED=sched))
    print(proc.stdout[-4000:])
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]
