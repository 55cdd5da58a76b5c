"""Pins for oracle.scatter (S1). Checked against properties the replay rule (reading R6)
must satisfy, never against the CUDA path."""
import itertools

import numpy as np

from oracle import scatter as S


def _recs(rows, A=3):
    """rows: list of (env, step, version, reward) -> record dict with distinct payloads."""
    M = len(rows)
    r = dict(env_id=np.array([x[0] for x in rows], np.int32),
             step=np.array([x[1] for x in rows], np.int32),
             version=np.array([x[2] for x in rows], np.int32),
             reward=np.array([x[3] for x in rows], np.float32),
             done=np.array([i % 2 for i in range(M)], np.uint8),
             value=np.arange(M, dtype=np.float32) * np.float32(0.5),
             tokens=(np.arange(M * A, dtype=np.int32).reshape(M, A) * 7),
             logp_behav=-np.arange(M * A, dtype=np.float32).reshape(M, A) / 8)
    return r


def _payload(buf):
    return {k: v.copy() for k, v in buf.items() if k != "slot_key"}


def test_permutation_invariance_all_720_orders():
    # 6 duplicate-free records on a 2x3 buffer: every arrival order gives the same buffer
    rows = [(e, t, 5 + e, float(10 * e + t)) for e in range(2) for t in range(3)]
    base = _recs(rows)
    ref = None
    for perm in itertools.permutations(range(6)):
        p = np.array(perm)
        rec = {k: v[p] for k, v in base.items()}
        buf = S.new_buffer(2, 3, 3)
        c = S.scatter_steps(buf, rec, cur_version=9, seq_base=1)
        assert c.tolist() == [0, 0, 0, 6]
        assert (buf["slot_key"] != 0).all()
        if ref is None:
            ref = _payload(buf)
        else:
            for k in ref:
                assert np.array_equal(ref[k].view(np.uint8), buf[k].view(np.uint8)), k


def test_conservation_with_faults():
    rng = np.random.default_rng(0)
    E, T, M = 4, 5, 200
    rows = [(int(rng.integers(-1, E + 1)), int(rng.integers(-1, T + 1)),
             int(rng.integers(-1, 4)), float(i)) for i in range(M)]
    rec = _recs(rows)
    buf = S.new_buffer(E, T, 3)
    oob, bad, dup, written = S.scatter_steps(buf, rec, cur_version=2, seq_base=100)
    assert oob + bad + dup + written == M
    inb = [(e, t) for e, t, v, _ in rows if 0 <= e < E and 0 <= t < T]
    ok = [(e, t) for e, t, v, _ in rows if 0 <= e < E and 0 <= t < T and 0 <= v <= 2]
    assert oob == M - len(inb)
    assert bad == len(inb) - len(ok)
    assert written == len(set(ok)) == int((buf["slot_key"] != 0).sum())


def test_round_trip_bitwise_including_nan_payloads():
    rows = [(0, 0, 1, 0.0), (1, 2, 1, 0.0), (0, 1, 0, 0.0)]
    rec = _recs(rows)
    nan_bits = np.array([0x7FC00001, 0xFFC12345, 0x7F800001], np.uint32)
    rec["reward"] = nan_bits.view(np.float32)
    rec["logp_behav"][1] = np.array([0x7FA00000, 0x00000001, 0x80000000], np.uint32).view(np.float32)
    buf = S.new_buffer(2, 3, 3)
    S.scatter_steps(buf, rec, cur_version=1, seq_base=1)
    for i, (e, t, _, _) in enumerate(rows):
        assert buf["reward"][e, t].view(np.uint32) == nan_bits[i]
        assert np.array_equal(buf["logp_behav"][e, t].view(np.uint32), rec["logp_behav"][i].view(np.uint32))
        assert np.array_equal(buf["tokens"][e, t], rec["tokens"][i])
        assert buf["done"][e, t] == rec["done"][i] and buf["version"][e, t] == rec["version"][i]
        assert buf["value"][e, t].view(np.uint32) == rec["value"][i].view(np.uint32)


def test_duplicate_brute_force_against_max_key_rule():
    """All sequences of 1..4 records on ONE slot with versions in {-1,0,1,2} (cur=1), with
    and without a pre-filled slot: the survivor is the valid record with the largest
    (version, position); dup = #valid arrivals - [slot was empty and any valid]."""
    cur = 1
    for n in range(1, 5):
        for versions in itertools.product([-1, 0, 1, 2], repeat=n):
            for prefilled in (False, True):
                rec = _recs([(0, 0, v, float(i)) for i, v in enumerate(versions)], A=2)
                buf = S.new_buffer(1, 1, 2)
                pre_key = 0
                if prefilled:
                    pre_key = (1 << 40) | 50  # version 1, an earlier call's seq 50
                    buf["slot_key"][0, 0] = np.uint64(pre_key)
                    buf["reward"][0, 0] = -9.0
                seq_base = 1000
                oob, bad, dup, written = S.scatter_steps(buf, rec, cur, seq_base)
                valid = [i for i, v in enumerate(versions) if 0 <= v <= cur]
                assert oob == 0 and bad == n - len(valid)
                keys = {i: (versions[i] << 40) | (seq_base + i) for i in valid}
                if not prefilled:
                    assert written == (1 if valid else 0)
                    assert dup == max(0, len(valid) - 1)
                else:
                    assert written == 0 and dup == len(valid)
                best = max(keys.values()) if keys else 0
                if best > pre_key:
                    win = [i for i in valid if keys[i] == best][0]
                    assert buf["reward"][0, 0] == np.float32(win)
                    assert int(buf["slot_key"][0, 0]) == best
                else:
                    assert int(buf["slot_key"][0, 0]) == pre_key
                    assert buf["reward"][0, 0] == (np.float32(-9.0) if prefilled else 0.0)
