"""Multi-GPU parity over NCCL (torchrun, one process per GPU): every rank's output, payload
and residual bit-identical to the oracle and to the other ranks (tests/dist_check.py).
Needs >= 2 GPUs (gpurun --gpus 2 / 4); skipped otherwise."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def torchrun(nproc, *args, port=29533, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "dist_check.py"),
           *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "DIST OK" in r.stdout
    return r.stdout


@pytest.mark.parametrize("nproc,G", [(2, 1), (2, 2), (4, 1), (4, 2), (4, 4), (8, 1), (8, 4)])
def test_nccl_parity(nproc, G):
    if ngpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    from paper_2205_09470_b200 import build
    build.build()
    torchrun(nproc, f"--gpus-per-cluster={G}", port=29500 + 10 * nproc + G)
