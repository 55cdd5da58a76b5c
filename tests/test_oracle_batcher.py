"""Pins for the NEXT-3 oracle (oracle/batcher.py): the Dynamic Batching Scheduler of Eq. (1)
 with SPEC.md's offer/poll operations.

  * the SPEC's worked examples (tests/golden/batcher_examples.csv, each row cited);
  * exhaustive: every non-decreasing sequence of <= 5 arrival times in [0, 10] and every
    (B_max, T_max) in {1..4} x {0..10} — the replayed schedule satisfies the
    declarative Eq. (1) predicates (FIFO partition, sizes, trigger, minimality) and
    conserves requests;
  * special cases with closed forms: T_max = 0 fires on every non-empty poll; T_max = inf
    emits consecutive blocks of exactly B_max; lockstep degeneracy.
"""
import csv
import itertools
import os

import numpy as np

from oracle import batcher as B

GOLD = os.path.join(os.path.dirname(__file__), "golden", "batcher_examples.csv")
INF = 10 ** 9


def test_spec_examples():
    rows = [r for r in csv.DictReader(l for l in open(GOLD) if not l.startswith("#"))]
    assert len(rows) == 7
    for r in rows:
        n = int(r["n_pending"])
        bt = B.Batcher(max(n, 1))
        bt.offer(range(n), [int(r["t_offer"])] * n, int(r["t_offer"]))
        batch = bt.poll(int(r["t_poll"]), int(r["b_max"]), int(r["t_max"]))
        assert len(batch) == int(r["batch"]), r["case"]
        assert len(bt.fifo) == int(r["remaining"]), r["case"]
        assert [e for e, _ in batch] == list(range(len(batch))), r["case"]     # oldest first
        if bt.fifo:
            assert bt.anchor == int(r["anchor_after"]), r["case"]
            assert [e for e, _ in bt.fifo] == list(range(len(batch), n))
        else:
            assert int(r["anchor_after"]) == -1


def test_fifo_order_and_rejections():
    bt = B.Batcher(4)
    bt.offer([2, 0, 1], [0, 0, 0], 0)                 # FIFO r1, r2, r3
    bt.offer([0, 7, 3, -1], [0, 0, 5, 0], 1)          # pending env, OOB, future, OOB
    assert [e for e, _ in bt.fifo] == [2, 0, 1]
    assert bt.counters.tolist() == [2, 1, 1, 3]
    assert [e for e, _ in bt.poll(1, 2, 99)] == [2, 0]
    bt.offer([2], [1], 1)                             # env 2 left the queue: accepted again
    assert [e for e, _ in bt.fifo] == [1, 2]


def _sequences(max_len, t_hi):
    for L in range(max_len + 1):
        yield from itertools.combinations_with_replacement(range(t_hi + 1), L)


def test_exhaustive_small_sequences():
    """all arrival sequences of length <= 5, integer times in [0, 10],
    (B_max, T_max) in {1..4} x {0..10}: zero violations of the Eq. (1) predicates."""
    n_checked = 0
    for times in _sequences(5, 10):
        arrivals = [(t, i) for i, t in enumerate(times)]
        for b_max in range(1, 5):
            for t_max in range(0, 11):
                horizon = (times[-1] if times else 0) + (t_max + 1) * (len(times) + 1)
                events = [(now, [e for t, e in arrivals if t == now], [now] * sum(1 for t, _ in arrivals if t == now))
                          for now in range(horizon + 1)]
                fired, bt, _ = B.replay(events, len(times) or 1, b_max, t_max)
                bad = B.schedule_violations(arrivals, fired, range(horizon + 1), b_max, t_max)
                assert not bad, (times, b_max, t_max, bad, fired)
                emitted = sorted(e for _, batch in fired for e, _ in batch)
                assert emitted == list(range(len(times))) and not bt.fifo    # conservation
                n_checked += 1
    assert n_checked == 4368 * 44


def test_predicates_catch_wrong_schedules():
    """The declarative check is not vacuous: plausible mistakes are flagged."""
    arrivals = [(0, 0), (0, 1), (2, 2)]
    good, _, _ = B.replay([(0, [0, 1], [0, 0]), (1, [], []), (2, [2], [2]), (3, [], []), (4, [], [])], 3, 2, 2)
    assert not B.schedule_violations(arrivals, good, range(5), 2, 2)
    assert good == [(0, [(0, 0), (1, 0)]), (4, [(2, 2)])]
    assert B.schedule_violations(arrivals, [(0, [(1, 0), (0, 0)]), (4, [(2, 2)])], range(5), 2, 2)  # order
    assert B.schedule_violations(arrivals, [(0, [(0, 0)]), (1, [(1, 0)]), (4, [(2, 2)])], range(5), 2, 2)  # size
    assert B.schedule_violations(arrivals, [(0, [(0, 0), (1, 0)]), (3, [(2, 2)])], range(5), 2, 2)  # early
    assert B.schedule_violations(arrivals, [(0, [(0, 0), (1, 0)])], range(5), 2, 2)  # missed trigger


def test_tmax_zero_and_infinite():
    rng = np.random.default_rng(0)
    n_env = 50
    arr_t = np.sort(rng.integers(0, 40, n_env))
    events = [(now, list(np.nonzero(arr_t == now)[0]), [now] * int((arr_t == now).sum())) for now in range(60)]
    # T_max = 0: every non-empty poll fires with min(pending, B_max)
    fired, _, sizes = B.replay(events, n_env, 3, 0)
    pend = 0
    for (now, envs, _), s in zip(events, sizes):
        pend += len(envs)
        assert s == min(pend, 3)
        pend -= s
    # T_max = inf: consecutive blocks of exactly B_max in arrival order, the rest stays
    fired, bt, _ = B.replay(events, n_env, 7, INF)
    order = [int(e) for now, envs, _ in events for e in envs]
    assert all(len(b) == 7 for _, b in fired) and len(fired) == n_env // 7
    assert [e for _, b in fired for e, _ in b] == order[:7 * (n_env // 7)]
    assert [e for e, _ in bt.fifo] == order[7 * (n_env // 7):]


def test_lockstep_degeneracy():
    """rollout_async = false <=> B_max = n_env, T_max = inf: every inference
    batch is the whole env set."""
    n_env = 16
    bt = B.Batcher(n_env)
    rng = np.random.default_rng(1)
    for rnd in range(5):
        order = rng.permutation(n_env)
        for k, e in enumerate(order):
            now = 100 * rnd + k
            bt.offer([e], [now], now)
            batch = bt.poll(now, n_env, INF)
            assert (len(batch) == n_env) == (k == n_env - 1)
        assert [e for e, _ in batch] == list(order)
