"""S1 oracle: out-of-order step records -> trajectory buffer (TEST INFRASTRUCTURE ONLY).

Paper: trajectories carry the policy version they were generated with (§3.1);
ready requests from subsets of environments arrive early / out of order (§3.2);
samples accumulate in a "trajectory buffer" (§3.3). The paper never says what
happens when a step arrives twice; reading R6: sequential replay in
submission order, key = (version << 40) | seq, newest key wins, every extra arrival
counts as a duplicate.
"""
from __future__ import annotations

import numpy as np

VERSION_SHIFT = 40


def new_buffer(n_env: int, t_steps: int, a_tok: int) -> dict:
    """Empty buffer: slot_key 0 means 'never filled' (reading R6b)."""
    return dict(
        slot_key=np.zeros((n_env, t_steps), np.uint64),
        reward=np.zeros((n_env, t_steps), np.float32),
        done=np.zeros((n_env, t_steps), np.uint8),
        value=np.zeros((n_env, t_steps), np.float32),
        version=np.zeros((n_env, t_steps), np.int32),
        tokens=np.zeros((n_env, t_steps, a_tok), np.int32),
        logp_behav=np.zeros((n_env, t_steps, a_tok), np.float32),
    )


def scatter_steps(buf: dict, rec: dict, cur_version: int, seq_base: int) -> np.ndarray:
    """Replay records i = 0..M-1 in order; returns counters [oob, bad_version, dup, written].

    For record i with key_i = (version_i << 40) | (seq_base + i):
      1. env_id or step out of range          -> oob += 1, skip
      2. version_i < 0 or > cur_version        -> bad_version += 1, skip
      3. slot already filled                   -> dup += 1; overwrite whole slot iff
                                                  key_i > slot_key
      4. otherwise                             -> write, written += 1
    Payload fields are copied bit for bit (float32 stays float32).
    """
    E, T = buf["slot_key"].shape
    oob = bad = dup = written = 0
    M = len(rec["env_id"])
    for i in range(M):
        e = int(rec["env_id"][i])
        t = int(rec["step"][i])
        v = int(rec["version"][i])
        if e < 0 or e >= E or t < 0 or t >= T:
            oob += 1
            continue
        if v < 0 or v > cur_version:
            bad += 1
            continue
        key = (v << VERSION_SHIFT) | (seq_base + i)
        old = int(buf["slot_key"][e, t])
        if old != 0:
            dup += 1
            if key <= old:
                continue
        else:
            written += 1
        buf["slot_key"][e, t] = np.uint64(key)
        buf["reward"][e, t] = rec["reward"][i]
        buf["done"][e, t] = rec["done"][i]
        buf["value"][e, t] = rec["value"][i]
        buf["version"][e, t] = rec["version"][i]
        buf["tokens"][e, t, :] = rec["tokens"][i]
        buf["logp_behav"][e, t, :] = rec["logp_behav"][i]
    return np.array([oob, bad, dup, written], np.int64)
