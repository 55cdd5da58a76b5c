"""NCCL multi-GPU parity of the C ABI (C1/C2/C3 inside the library), run with torchrun
when the box has >= 2 GPUs (tools/mgpu_parity.py); skipped on a single GPU."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("p2p", ["1", "0"])
@pytest.mark.parametrize("n", [2, 4])
def test_nccl_multigpu_parity(n, p2p):
    """The loss statistics reduced in-kernel over NVLink peer memory (RLVLA_P2P=1, the
    default) and through NCCL (RLVLA_P2P=0) both match the oracle."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tools", "mgpu_parity.py")]
    env = dict(os.environ, RLVLA_P2P=p2p)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MGPU PARITY OK" in r.stdout
    if p2p == "0":
        assert "in-kernel-p2p=False" in r.stdout
