"""GPU parity for NEXT-3 — the Eq. (1) dynamic batching scheduler on the device
(rlvla_batch_offer / rlvla_batch_poll, reading R24) against oracle/batcher.py:
bit-exact batch contents (env ids, enqueue times, order), trigger ticks, counters, queue
state, and the gathered observation bytes."""
import itertools

import numpy as np
import pytest
import torch

from oracle import batcher as O_b
from tests import harness as H

pytestmark = pytest.mark.gpu


def _P():
    import paper_2602_05765_b200 as P
    return P


def _run(case, with_obs_src=True, fifo=False):
    """Replay a harness case tick by tick through the C ABI; compare every poll. fifo: the
    observation rows are kept in FIFO order and each batch is read in place (no out_obs)."""
    P = _P()
    q = P.BatchQueue.allocate(case.n_env, case.obs_bytes, obs_fifo=fifo,
                              max_batch=min(case.b_max, case.n_env) if fifo else 0)
    ws = P.workspace(1)
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    out_env = torch.full((case.b_max,), -7, dtype=torch.int32, device="cuda")
    out_time = torch.zeros(case.b_max, dtype=torch.int64, device="cuda")
    out_n = torch.zeros(1, dtype=torch.int32, device="cuda")
    out_obs = torch.zeros(case.b_max, max(case.obs_bytes, 16), dtype=torch.uint8, device="cuda") \
        if case.obs_bytes and not fifo else None
    last_payload = {}
    n_fired = 0
    for tk in case.ticks:
        now = tk["now"]
        if tk["env"]:
            env = torch.tensor(tk["env"], dtype=torch.int32, device="cuda")
            tim = torch.tensor(tk["time"], dtype=torch.int64, device="cuda")
            src = None
            if case.obs_bytes:
                rows = [H.payload(case, e, c) for e, c in zip(tk["env"], tk["cycle"])]
                if with_obs_src:
                    src = torch.from_numpy(np.stack(rows)).cuda()
                else:  # the env side writes its slot itself (zero-copy offer)
                    for e, c, r in zip(tk["env"], tk["cycle"], rows):
                        if c >= 0:
                            q.obs[e].copy_(torch.from_numpy(r))
            P.rlvla_batch_offer(q, env, tim, now, cnt, obs_src=src, ws=ws)
            for e, c in zip(tk["env"], tk["cycle"]):
                if c >= 0:
                    last_payload[e] = c
        P.rlvla_batch_poll(q, now, case.b_max, case.t_max, out_env, out_time, out_n,
                           out_obs=out_obs, ws=ws)
        b = int(out_n.item())
        exp = tk["expect"]
        assert b == len(exp), (now, b, len(exp))
        if b:
            n_fired += 1
            assert out_env[:b].cpu().tolist() == [e for e, _ in exp], now
            assert out_time[:b].cpu().tolist() == [t for _, t in exp], now
            if out_obs is not None or (fifo and case.obs_bytes):
                got = (q.batch_rows(b) if fifo else out_obs[:b, :case.obs_bytes]).cpu().numpy()
                for i, (e, _) in enumerate(exp):
                    assert np.array_equal(got[i], H.payload(case, e, last_payload[e])), (now, e)
    assert cnt.cpu().tolist() == case.counters.tolist()
    st = q.state.cpu().tolist()
    n_acc = int(case.counters[3])
    assert st[1] == n_acc and st[3] == n_fired
    return st


@pytest.mark.parametrize("fifo", [False, True])
@pytest.mark.parametrize("n_env,ticks,b_max,t_max,obs_bytes", [
    (300, 600, 64, 8, 3 * 16384 + 48),     # multi-chunk payload with a ragged tail
    (37, 400, 5, 0, 16),                    # T_max = 0: every non-empty poll fires
    (64, 500, 64, 10 ** 9, 1024),          # T_max = inf: only full batches (lockstep-like)
    (20, 300, 100, 15, 0),                  # B_max > n_env, no payload
])
def test_closed_loop_traffic(n_env, ticks, b_max, t_max, obs_bytes, fifo):
    case = H.batcher_case(n_env, ticks, b_max, t_max, obs_bytes=obs_bytes)
    assert sum(1 for t in case.ticks if t["expect"]) >= 5
    # the harness's bad offers are exactly the ones the oracle rejects
    assert sum(1 for t in case.ticks for c in t["cycle"] if c < 0) == case.counters[:3].sum()
    assert case.counters[:3].sum() > 0 or t_max == 10 ** 9
    if fifo and b_max > n_env:  # a FIFO-row queue bounds b_max by its mirror rows: same batches
        case = H.batcher_case(n_env, ticks, n_env, t_max, obs_bytes=obs_bytes)
    _run(case, fifo=fifo)


def test_zero_copy_offer():
    case = H.batcher_case(48, 300, 16, 6, obs_bytes=4096, seed=11)
    _run(case, with_obs_src=False)


def test_small_sequences_sample():
    """A seeded sample of the exhaustive space of the oracle pins: arrival
    sequences of <= 6 requests at integer times in [0, 10], (B_max, T_max) in
    {1..4} x {0..10}, every tick offered then polled."""
    rng = np.random.default_rng(5)
    seqs = [s for L in range(7) for s in itertools.combinations_with_replacement(range(11), L)]
    for k in rng.choice(len(seqs), 150, replace=False):
        times = seqs[k]
        b_max, t_max = int(rng.integers(1, 5)), int(rng.integers(0, 11))
        n = max(len(times), 1)
        case = H.BatcherCase(n, 32, b_max, t_max)
        bt = O_b.Batcher(n)
        horizon = (times[-1] if times else 0) + (t_max + 1) * (len(times) + 1)
        for now in range(horizon + 1):
            envs = [i for i, t in enumerate(times) if t == now]
            bt.offer(envs, [now] * len(envs), now)
            case.ticks.append(dict(now=now, env=envs, time=[now] * len(envs), cycle=[0] * len(envs),
                                   expect=bt.poll(now, b_max, t_max)))
        case.counters = bt.counters.copy()
        _run(case)


def test_oft_sized_gather():
    """OpenVLA-OFT observations (2 x 224x224x3 + proprio = 301,088 B), B_max = 64: one full
    batch leaves with every byte in place."""
    import synth
    P = _P()
    n_env, ob, b_max = 96, synth.OBS_BYTES_OFT, 64
    q = P.BatchQueue.allocate(n_env, ob)
    g = torch.Generator(device="cuda").manual_seed(3)
    q.obs.copy_(torch.randint(0, 256, (n_env, ob), generator=g, device="cuda", dtype=torch.uint8))
    order = torch.randperm(n_env, generator=torch.Generator().manual_seed(4))[:70].to(torch.int32)
    ws = P.workspace(1)
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    P.rlvla_batch_offer(q, order.cuda(), torch.zeros(70, dtype=torch.int64, device="cuda"), 0, cnt, ws=ws)
    out_env = torch.empty(b_max, dtype=torch.int32, device="cuda")
    out_time = torch.empty(b_max, dtype=torch.int64, device="cuda")
    out_n = torch.empty(1, dtype=torch.int32, device="cuda")
    out_obs = torch.empty(b_max, ob, dtype=torch.uint8, device="cuda")
    P.rlvla_batch_poll(q, 3, b_max, 50, out_env, out_time, out_n, out_obs=out_obs, ws=ws)
    assert int(out_n.item()) == 64                              # S:180 oversize rule
    assert out_env.cpu().tolist() == order[:64].tolist()
    assert torch.equal(out_obs, q.obs[order[:64].long().cuda()])
    assert q.state.cpu().tolist()[:4] == [64, 70, 3, 1]        # 6 remain, anchor re-set to 3
    assert int(q.pending.sum().item()) == 6
