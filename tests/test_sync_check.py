"""RLVLA_SYNC_CHECK=1 (SURVEY §5 failure detection): the device error counters become return
codes — a call whose data carries an error returns RLVLA_ERR_DATA (5), a clean call OK. Run in
a subprocess because the library reads the variable once."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import torch, numpy as np
import paper_2602_05765_b200 as P
from paper_2602_05765_b200 import _abi as A
out = []
E, T, A_ = 4, 8, 3
buf = P.TrajectoryBuffer.allocate(E, T, A_)
def batch(env):
    n = len(env)
    i = lambda *s: torch.zeros(*s, dtype=torch.int32, device="cuda")
    f = lambda *s: torch.zeros(*s, dtype=torch.float32, device="cuda")
    return P.StepBatch(torch.tensor(env, dtype=torch.int32, device="cuda"), i(n), i(n), f(n),
                       torch.zeros(n, dtype=torch.uint8, device="cuda"), f(n), i(n, A_), f(n, A_))
cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
out.append(P.rlvla_scatter_steps(buf, batch([0, 1]), 5, 1, cnt, check=False))
out.append(P.rlvla_scatter_steps(buf, batch([0, 9]), 5, 3, cnt, check=False))      # OOB env
x = torch.randn(6, 64, device="cuda")
lp = torch.empty(6, device="cuda")
st = torch.zeros(24, dtype=torch.float64, device="cuda")
ws = P.workspace(1)
out.append(P.rlvla_logprob_fwd_bwd(x, torch.tensor([1, 2, 3, 4, 5, 6], dtype=torch.int32, device="cuda"),
                                   logp=lp, stats=st, ws=ws, check=False))
out.append(P.rlvla_logprob_fwd_bwd(x, torch.tensor([1, 2, 3, 4, 5, 99], dtype=torch.int32, device="cuda"),
                                   logp=lp, stats=st, ws=ws, check=False))          # bad target
print("CODES", out)
'''


def test_sync_check_turns_counters_into_status():
    if not torch.cuda.is_available():
        pytest.skip("GPU")
    env = dict(os.environ, RLVLA_SYNC_CHECK="1", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, cwd=ROOT, env=env,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("CODES")][-1]
    assert line == "CODES [0, 5, 0, 5]", line
