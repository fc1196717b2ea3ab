"""Distributed parity on >= 2 GPUs of one box (skipped with fewer): torchrun launches
tests/dist_worker.py, one rank per GPU; Y(P) must match the oracle within 1e-12.  Every exchange
mode: the device-initiated peer pulls (default), the direct remote reads
of the off-diagonal kernels (H2_EXCHANGE=p2p-direct) and the NCCL groups (H2_EXCHANGE=nccl)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("exchange", ["p2p", "p2p-direct", "nccl"])
@pytest.mark.parametrize("P", [2, 4])
def test_distributed_parity(P, exchange):
    if _ngpu() < P:
        pytest.skip(f"needs {P} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "dist_worker.py")]
    env = dict(os.environ, H2_EXCHANGE=exchange)
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
