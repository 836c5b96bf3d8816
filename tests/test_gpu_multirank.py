"""Multi-rank executor parity: runs tests/mp_gpu_check.py under torchrun.

* one process per GPU (NVLink, NCCL group) on 2 and 4 GPUs when the box has them;
* two or three processes sharing GPU 0 (gloo group) on any box: the product transport --
  IPC peer regions opened by another process, flag barriers, 2-D copy-engine pulls, the
  dK/dV return and K4 -- runs exactly as across GPUs, time-sliced on one device.  This is
  the case a one-GPU box runs."""

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


def _run(n, sched="fcp", shared=False, args=(), heads="8,2", dim=128, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "mp_gpu_check.py"), *args]
    env = dict(os.environ, FCPB_CHECK_SCHED=sched, FCPB_CHECK_HEADS=heads, FCPB_CHECK_DIM=str(dim),
               FCPB_SHARED_GPU="1" if shared else "0", **(env or {}))
    proc = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    print(proc.stdout[-4000:])
    assert proc.returncode == 0, proc.stdout[-3000:] + proc.stderr[-3000:]


@pytest.mark.parametrize("n,sched", [(2, "fcp"), (4, "fcp"), (4, "ring")])
def test_executor_nccl_parity(n, sched):
    """FCP plans, and the ring plan of baselines.py (relay edges, relayed-only chunks)."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    _run(n, sched)


@pytest.mark.parametrize("n,sched,args,heads", [
    (2, "fcp", (), "4,4:64"),                   # the C1 tiny model (Hq = Hkv = 4, D = 64)
    (2, "fcp", (), "8,2"),
    (3, "fcp", (), "8,2"),
    (3, "ring", (), "8,2"),
    # ranks none of whose chunks is consumed remotely (no dK/dV comes back)
    (4, "fcp", ("2048,2048,4096", "2048"), "8,2"),
    (2, "fcp", ("9000,4100,3000,2100,1500,700,129", "2048"), "32,8"),   # Llama-3-8B heads
    (8, "fcp", (), "8,2"),                      # the driver's N=8 path: 7 peers per rank
])
def test_executor_shared_gpu_parity(n, sched, args, heads):
    """N ranks as N processes on GPU 0: the multi-rank product path on a one-GPU box."""
    heads, _, dim = heads.partition(":")
    _run(n, sched, shared=True, args=args, heads=heads, dim=int(dim or 128))


def test_executor_shared_gpu_resumed_forward():
    """The executor with the local wave overlapped with copy-engine pulls and the remote wave
    continuing its partials (FCPB_FUSE_REMOTE=resume), 3 ranks on GPU 0."""
    _run(3, shared=True, env={"FCPB_FUSE_REMOTE": "resume"})
