"""Multi-GPU pipeline parity: torchrun, one stage per GPU over NCCL,
in lockstep with the oracle pipeline of the same P (tests/mp_pipeline_worker.py).
Skipped when the box has fewer GPUs than the case needs."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("P,shape", [(2, "tiny"), (2, "small"), (2, "smallq"), (4, "small:4"), (4, "smallq:4")])
def test_nccl_pipeline_lockstep(P, shape):
    if _gpus() < P:
        pytest.skip(f"needs {P} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_pipeline_worker.py"), shape]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
