"""NEXT-3 oracle: the Dynamic Batching Scheduler of Eq. (1) (TEST INFRASTRUCTURE ONLY).

Paper (§3.2): "This scheduler utilizes the maximum inference batch size (B_max)
and the maximum waiting latency (T_max) as constraints:
    Trigger Inference if: (Batch Size >= B_max) or (Wait Time >= T_max)"
Ready requests from a subset of environments enter the inference queue early.

The paper does not say what the wait clock measures, what happens with more than B_max
pending requests, or whether an empty queue can fire. Reading R24 takes
SPEC.md's operations, written out below in their own order:
  offer(req, now): append to the pending FIFO in arrival order; if the queue
                   was empty, the wait-clock anchor := now.
  poll(now): n = |pending|; fire iff n >= B_max or (n >= 1 and
                   now - anchor >= T_max) (empty-batch rule S:261); the batch is the
                   oldest min(n, B_max) requests (oversize rule S:262); if requests remain,
                   the anchor := now.
A request is (env_id, enqueue_time) with enqueue_time <= now; an environment waits for its
action, so it has at most one pending request (a second offer while pending is rejected
and counted). Offers that break the preconditions are rejected and counted:
counters = [env out of range, enqueue_time > now, env already pending, accepted].
Times are integers (ticks), so the comparison with T_max is exact.
"""
from __future__ import annotations

import numpy as np


class Batcher:
    """Plain FIFO state machine (one rollout worker's queue)."""

    def __init__(self, n_env: int):
        self.n_env = n_env
        self.fifo: list[tuple[int, int]] = []
        self.anchor = 0
        self.pending = np.zeros(n_env, bool)
        self.counters = np.zeros(4, np.int64)

    def offer(self, env_ids, enqueue_times, now: int):
        """Requests in arrival order (one call = one arrival chunk at time `now`)."""
        for e, t in zip(env_ids, enqueue_times):
            e, t = int(e), int(t)
            if not 0 <= e < self.n_env:
                self.counters[0] += 1
                continue
            if t > now:
                self.counters[1] += 1
                continue
            if self.pending[e]:
                self.counters[2] += 1
                continue
            if not self.fifo:
                self.anchor = now
            self.fifo.append((e, t))
            self.pending[e] = True
            self.counters[3] += 1

    def poll(self, now: int, b_max: int, t_max: int):
        """Eq. (1). Returns the emitted batch as a list of (env, enqueue_time), or []."""
        n = len(self.fifo)
        fire = n >= b_max or (n >= 1 and now - self.anchor >= t_max)
        if not fire:
            return []
        b = min(n, b_max)
        batch, self.fifo = self.fifo[:b], self.fifo[b:]
        for e, _ in batch:
            self.pending[e] = False
        if self.fifo:
            self.anchor = now
        return batch


def replay(events, n_env: int, b_max: int, t_max: int):
    """Run a tick-ordered event list through a Batcher: events = [(now, env_ids, times)],
    one offer chunk then one poll per tick. Returns [(now, batch)] for every firing poll,
    the final Batcher and the per-poll batch sizes."""
    bt = Batcher(n_env)
    fired, sizes = [], []
    for now, envs, times in events:
        bt.offer(envs, times, now)
        batch = bt.poll(now, b_max, t_max)
        sizes.append(len(batch))
        if batch:
            fired.append((now, batch))
    return fired, bt, sizes


def schedule_violations(arrivals, fired, poll_times, b_max: int, t_max: int):
    """Declarative check of a schedule against Eq. (1) + S:261-262, independent of the
    state machine: `arrivals` = [(time, env)] in FIFO order (every request offered at its
    enqueue time), `fired` = [(time, [(env, time), ...])], polls at `poll_times` (each
    after that tick's offers). Returns a list of violated properties (empty = valid):
      P1 FIFO partition: concatenated batches are a prefix of the arrivals in order;
      P2 size: 1 <= |batch| <= B_max, and |batch| = min(pending, B_max) at its poll;
      P3 trigger: at every firing poll, pending >= B_max or wait >= T_max;
      P4 minimality: at every non-firing poll, pending < B_max and (pending == 0 or
         wait < T_max);
    where pending(t) and the anchor are re-derived from the arrival times and the batch
    boundaries alone (anchor = time the queue last became non-empty, or the last firing
    poll that left requests behind)."""
    bad = []
    emitted = [r for _, batch in fired for r in batch]
    if emitted != [(e, t) for t, e in arrivals][:len(emitted)]:
        bad.append("P1")
    fire_at = {t: batch for t, batch in fired}
    n_out = 0
    anchor = None
    for now in poll_times:
        n_in = sum(1 for t, _ in arrivals if t <= now)
        # anchor: arrivals that found the queue empty (re-derived arrival by arrival)
        pend_before = n_in - n_out
        if pend_before > 0 and anchor is None:
            # the first request still pending arrived when the queue was empty
            anchor = arrivals[n_out][0]
        batch = fire_at.get(now, [])
        wait_ok = pend_before >= 1 and anchor is not None and now - anchor >= t_max
        should = pend_before >= b_max or wait_ok
        if batch:
            if not should:
                bad.append(f"P3@{now}")
            if len(batch) != min(pend_before, b_max):
                bad.append(f"P2@{now}")
            n_out += len(batch)
            anchor = now if n_in - n_out > 0 else None
        elif should:
            bad.append(f"P4@{now}")
    return bad
