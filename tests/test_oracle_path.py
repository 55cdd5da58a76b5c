"""Pins for the oracle glue that turns a trajectory buffer into per-token loss inputs
(oracle.advantages.episode_return / grpo_step_adv / step_counts, oracle.path.advantages /
token_view / rollout_to_loss): hand-built buffers whose answers are printed values, closed
forms or library routines, per-element brute force, and the P = 1 vs P = 8 logical-shard
identity (SURVEY §8(c) S2b pins (vi), (vii)). Never the CUDA path.

Anchor: the trajectory buffer micro-batches are cut from (§3.3) and the per-trajectory
policy version (§3.1); GRPO / GAE are textbook (readings R7-R10)."""
import math

import numpy as np
import pytest

from oracle import advantages as A
from oracle import path as OP
from oracle import scatter as OS

JUNK = 1.0e6      # what an unfilled slot holds: a stale reward / value from an old window


def _buf(E, T, Atok):
    b = OS.new_buffer(E, T, Atok)
    b["reward"][:] = JUNK            # unfilled slots keep stale payload; only slot_key says empty
    b["value"][:] = JUNK
    b["done"][:] = 1
    b["version"][:] = 7              # stale version of an old window
    b["tokens"][:] = 3
    return b


def _fill(b, e, t, *, r=0.0, v=0.0, d=0, ver=100, tok=None, key=1):
    b["slot_key"][e, t] = np.uint64(key)
    b["reward"][e, t] = r
    b["value"][e, t] = v
    b["done"][e, t] = d
    b["version"][e, t] = ver
    if tok is not None:
        b["tokens"][e, t, :] = tok


# ---------------------------------------------------------------------------------------
# S2b GRPO glue: brute force on 2 groups of 4 with unfilled slots
# ---------------------------------------------------------------------------------------

def _grpo_case():
    """8 envs x 5 steps, interleaved groups g(e) = e mod 2 (every group spans the buffer).
    Filled-step returns: group 0 (envs 0, 2, 4, 6) = {1, 0, 0, 0}; group 1 (envs 1, 3, 5, 7)
    = {2, 2, 0, 0}. Every env has at least one unfilled slot holding JUNK reward."""
    E, T = 8, 5
    b = _buf(E, T, 2)
    # env 0: success reward 1 at t = 3; t = 1 unfilled
    for t in (0, 2, 3, 4):
        _fill(b, 0, t, r=1.0 if t == 3 else 0.0)
    # env 1: 0.5 on each of t = 0..3; t = 4 unfilled
    for t in range(4):
        _fill(b, 1, t, r=0.5)
    # env 3: 2.0 at t = 0 only, t = 1, 2 unfilled
    _fill(b, 3, 0, r=2.0)
    _fill(b, 3, 3, r=0.0)
    _fill(b, 3, 4, r=0.0)
    # envs 2, 4, 5, 6, 7: zero reward, some unfilled
    for e, filled in ((2, (0, 1)), (4, (2,)), (5, (0, 1, 2, 3)), (6, (4,)), (7, (1, 3))):
        for t in filled:
            _fill(b, e, t, r=0.0)
    return b, np.arange(E) % 2


def test_episode_return_ignores_unfilled_slots():
    b, _ = _grpo_case()
    R = A.episode_return(b["reward"], b["slot_key"] != 0)
    assert R.tolist() == [1.0, 2.0, 0.0, 2.0, 0.0, 0.0, 0.0, 0.0]


def test_grpo_path_brute_force_two_groups_of_four():
    b, gid = _grpo_case()
    out = OP.advantages(b, None, mode="grpo", group_of_env=gid, cur_version=100)
    # printed / closed-form group advantages (unbiased std, eps = 1e-6 on sigma, R10):
    #   {1,0,0,0}: (1.499997000, -0.499999000 x 3)
    #   {2,2,0,0}: mu = 1, sigma = sqrt(4/3) => +-1/(sqrt(4/3) + 1e-6) = +-0.8660246537850883
    a_env = {0: 1.499997000, 2: -0.499999000, 4: -0.499999000, 6: -0.499999000,
             1: 0.8660246537850883, 3: 0.8660246537850883,
             5: -0.8660246537850883, 7: -0.8660246537850883}
    R_env = {0: 1.0, 1: 2.0, 2: 0.0, 3: 2.0, 4: 0.0, 5: 0.0, 6: 0.0, 7: 0.0}
    E, T = b["slot_key"].shape
    for e in range(E):
        for t in range(T):
            filled = b["slot_key"][e, t] != 0
            want = a_env[e] if filled else 0.0
            assert abs(out["adv"][e, t] - want) < 5e-9, (e, t, out["adv"][e, t], want)
            assert out["ret"][e, t] == (R_env[e] if filled else 0.0)
    # population flag: {1,0,0,0} -> (1.732046808, -0.577348936 x 3)
    pop = OP.advantages(b, None, mode="grpo", group_of_env=gid, std_unbiased=False,
                        cur_version=100)
    assert abs(pop["adv"][0, 0] - 1.732046808) < 5e-9
    assert abs(pop["adv"][2, 0] + 0.577348936) < 5e-9
    assert pop["adv"][0, 1] == 0.0                 # unfilled slot


def test_grpo_step_adv_broadcasts_only_to_filled_steps():
    v = np.array([[1, 0, 1], [0, 0, 0], [1, 1, 1]], bool)
    out = A.grpo_step_adv(np.array([2.5, -1.0, -3.0]), v)
    assert out.tolist() == [[2.5, 0.0, 2.5], [0.0, 0.0, 0.0], [-3.0, -3.0, -3.0]]


# ---------------------------------------------------------------------------------------
# S2a GAE glue: unfilled slots hold junk, the closed form still holds (R7, R8, R9)
# ---------------------------------------------------------------------------------------

def test_gae_path_ignores_junk_and_whitens_over_filled_steps():
    b = _buf(2, 6, 1)
    for t in (0, 1, 3, 4, 5):                     # env 0: t = 2 unfilled (JUNK, done = 1)
        _fill(b, 0, t, r=1.0, v=0.0)
    for t in range(6):                            # env 1: terminates at t = 2
        _fill(b, 1, t, r=1.0, v=0.0, d=1 if t == 2 else 0)
    lv = np.zeros(2)
    out = OP.advantages(b, lv, mode="gae", gamma=1.0, lam=1.0, cur_version=100)
    # gamma = lambda = 1, r = 1, V = 0: A_t = number of steps left in the segment
    assert out["adv"][0].tolist() == [2.0, 1.0, 0.0, 3.0, 2.0, 1.0]
    assert out["adv"][1].tolist() == [3.0, 2.0, 1.0, 3.0, 2.0, 1.0]
    assert out["ret"][0, 2] == 0.0 and out["ret"][0, 0] == 2.0
    assert out["whiten_stats"] == (11.0, 21.0, 47.0)      # sum A^2 = 19 + 28
    w = OP.advantages(b, lv, mode="gae", gamma=1.0, lam=1.0, whiten=True, cur_version=100)
    vals = np.array([2, 1, 3, 2, 1, 3, 2, 1, 3, 2, 1], np.float64)
    mu, sd = 21.0 / 11.0, vals.std(ddof=1)          # 1.909090..., 0.831209...
    assert abs(sd - 0.8312094145936334) < 1e-15
    filled = b["slot_key"] != 0
    np.testing.assert_allclose(w["adv"][filled], (out["adv"][filled] - mu) / (sd + 1e-8),
                               rtol=1e-13)
    assert w["adv"][0, 2] == 0.0


# ---------------------------------------------------------------------------------------
# counts and the per-token view
# ---------------------------------------------------------------------------------------

def test_step_counts_closed_form():
    """E x T x A = 4 x 5 x 3, all filled at lag 0 with every target >= 0 => n_tok = 60 and
    20 loss steps; then 2 steps at lag 2 (stale), 1 step at lag -1 (bad), 4 targets = -1 on
    ok steps, one ok step with all 3 targets = -1 (no loss step), and 2 unfilled steps (one
    of them at lag 5 and one with targets -1: both ignored)."""
    E, T, At, cur = 4, 5, 3, 100
    valid = np.ones((E, T), bool)
    version = np.full((E, T), cur)
    tokens = np.zeros((E, T, At), np.int64)
    assert A.step_counts(valid, version, tokens, cur, 1) == dict(
        n_valid=20, n_tok=60, n_stale=0, n_bad=0, n_loss_steps=20)
    version[0, 1] = version[2, 3] = cur - 2       # stale (lag 2 > eta = 1)
    version[1, 0] = cur + 1                       # future (lag -1)
    version[3, 4] = cur - 1                       # lag 1 == eta: still counted
    tokens[0, 0, 0] = tokens[0, 0, 2] = tokens[1, 1, 1] = tokens[3, 4, 0] = -1
    tokens[2, 0, :] = -1                          # an ok step without a usable token
    valid[2, 2] = valid[3, 0] = False
    version[2, 2] = cur - 5
    tokens[3, 0, :] = -1
    # n_valid = 20 - 2 unfilled = 18; ok steps = 18 - 2 stale - 1 bad = 15;
    # n_tok = 3 * 15 - 4 - 3 = 38; loss steps = 15 - 1 = 14
    assert A.step_counts(valid, version, tokens, cur, 1) == dict(
        n_valid=18, n_tok=38, n_stale=2, n_bad=1, n_loss_steps=14)
    # eta = 2 admits the two lag-2 steps: n_tok = 3 * 17 - 7 = 44, 16 loss steps
    c2 = A.step_counts(valid, version, tokens, cur, 2)
    assert (c2["n_tok"], c2["n_loss_steps"]) == (44, 16)


def test_token_view_row_to_step_and_lag_sign():
    """Row r of the token view is token r % A of decision step r // A, steps row-major
    [E, T]; lag = cur_version - version (rollout on pre-update weights => lag >= 0)."""
    E, T, At, cur = 2, 3, 2, 100
    b = _buf(E, T, At)
    vers = [[100, 99, 98], [97, 100, 99]]
    for e in range(E):
        for t in range(T):
            if (e, t) != (1, 2):                  # (1, 2) unfilled
                _fill(b, e, t, ver=vers[e][t], tok=[10 * (3 * e + t), 10 * (3 * e + t) + 1])
            b["logp_behav"][e, t, :] = [-(3 * e + t) - 0.25, -(3 * e + t) - 0.75]
    adv = np.array([[0.5, 1.5, 2.5], [3.5, 4.5, 5.5]])
    tv = OP.token_view(b, adv, At, cur)
    assert tv["valid"].tolist() == [True] * 10 + [False] * 2
    assert tv["lag"].tolist()[:10] == [0, 0, 1, 1, 2, 2, 3, 3, 0, 0]
    assert tv["lag"].tolist()[10:] == [93, 93]   # the unfilled slot's stale version (7)
    assert tv["adv"].tolist() == [0.5, 0.5, 1.5, 1.5, 2.5, 2.5, 3.5, 3.5, 4.5, 4.5, 5.5, 5.5]
    assert tv["target"].tolist()[:10] == [0, 1, 10, 11, 20, 21, 30, 31, 40, 41]
    assert tv["logp_behav"].tolist()[6] == -3.25 and tv["logp_behav"].tolist()[3] == -1.75


# ---------------------------------------------------------------------------------------
# P = 1 vs P = 8 logical shards
# ---------------------------------------------------------------------------------------

def _random_buffer(E, T, At, seed):
    rng = np.random.default_rng(seed)
    b = _buf(E, T, At)
    for e in range(E):
        for t in range(T):
            if rng.random() < 0.85:
                _fill(b, e, t, r=float(np.float32(rng.random() < 0.3)) + float(np.float32(rng.uniform(0, .1))),
                      v=float(np.float32(rng.normal(.5, .2))), d=int(rng.random() < 0.1),
                      ver=100 - int(rng.integers(0, 2)))
    return b


@pytest.mark.parametrize("P", [2, 8])
def test_grpo_logical_shards_bit_identical(P):
    E, T, G = 64, 6, 8
    b = _random_buffer(E, T, 2, 11)
    gid = np.arange(E) % (E // G)                 # interleaved: every group spans all shards
    full = OP.advantages(b, None, mode="grpo", group_of_env=gid, cur_version=100)
    Er = E // P
    shards = [{k: v[r * Er:(r + 1) * Er] for k, v in b.items()} for r in range(P)]
    # C2 emulated: every shard's per-env returns gathered in rank order
    R_all = np.concatenate([A.episode_return(s["reward"], s["slot_key"] != 0) for s in shards])
    parts = [OP.advantages(s, None, mode="grpo", group_of_env=gid, cur_version=100,
                           R_global=R_all, env_offset=r * Er)["adv"] for r, s in enumerate(shards)]
    assert np.array_equal(np.concatenate(parts), full["adv"])


@pytest.mark.parametrize("P", [2, 8])
def test_gae_whitening_logical_shards(P):
    E, T = 64, 6
    b = _random_buffer(E, T, 2, 12)
    lv = np.random.default_rng(13).normal(size=E)
    full = OP.advantages(b, lv, mode="gae", whiten=True, cur_version=100)
    Er = E // P
    shards = [{k: v[r * Er:(r + 1) * Er] for k, v in b.items()} for r in range(P)]
    raw = [OP.advantages(s, lv[r * Er:(r + 1) * Er], mode="gae", cur_version=100)
           for r, s in enumerate(shards)]
    st = tuple(np.sum([o["whiten_stats"] for o in raw], axis=0))      # C1 emulated
    parts = [OP.advantages(s, lv[r * Er:(r + 1) * Er], mode="gae", whiten=True, whiten_global=st,
                           cur_version=100)["adv"] for r, s in enumerate(shards)]
    # raw GAE is per env, so identical; the whitened values differ only by the order of the
    # fp64 sums behind (mu, sigma)
    assert np.array_equal(np.concatenate([o["raw"] for o in raw]), full["raw"])
    np.testing.assert_allclose(np.concatenate(parts), full["adv"], rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------------------------------
# the whole chain on a hand-evaluable case
# ---------------------------------------------------------------------------------------

def test_rollout_to_loss_closed_form():
    """2 envs x 2 decision steps, A = 1 token, V = 2 equal logits, one GRPO group of 2.
    env 0 fills both steps (success reward 1 at t = 1): R_0 = 1; env 1 fills t = 0 only
    (reward 0): R_1 = 0 => A = +-0.707105781. logp = -ln 2 on
    every row and logp_behav = f32(-ln 2), so rho = 1 up to one f32 rounding; no clip.
    N_tok = 3 => Loss = -(2 A_0 + A_1) / 3 = -0.707105781 / 3, g = -A rho / 3 per token,
    dx = g (1[j = a] - 1/2). An OOB record and a resend that loses are counted."""
    lb = np.float32(-math.log(2.0))
    rec = dict(env_id=np.array([1, 0, 5, 0, 0], np.int32), step=np.array([0, 1, 0, 0, 1], np.int32),
               version=np.array([100, 100, 100, 100, 99], np.int32),
               reward=np.array([0, 1, 0, 0, 9], np.float32), done=np.array([0, 1, 0, 0, 0], np.uint8),
               value=np.zeros(5, np.float32), tokens=np.array([[1], [0], [0], [1], [1]], np.int32),
               logp_behav=np.full((5, 1), lb, np.float32))
    cfg = dict(n_env=2, t_steps=2, a_tok=1, cur_version=100, max_staleness=1, mode="grpo",
               group_of_env=np.array([0, 0]), last_value=None)
    logits = np.zeros((4, 2))
    out = OP.rollout_to_loss(cfg, [{k: v[:3] for k, v in rec.items()},
                                   {k: v[3:] for k, v in rec.items()}], logits)
    assert out["counters"].tolist() == [1, 0, 1, 3]         # oob, bad_version, dup, written
    a = 0.707105781
    np.testing.assert_allclose(out["adv"]["adv"], [[a, a], [-a, 0.0]], atol=5e-9)
    assert out["adv"]["counts"]["n_tok"] == 3
    np.testing.assert_allclose(out["fwd"]["logp"], -math.log(2.0), rtol=1e-15)
    assert abs(out["stats"]["loss"] + a / 3) < 1e-7
    g = np.array([-a / 3, -a / 3, a / 3, 0.0])
    np.testing.assert_allclose(out["ppo"]["grad"], g, atol=1e-7)
    tgt = np.array([1, 0, 1, 0])                            # row 3: unfilled slot (token 0)
    want_dx = g[:, None] * ((np.arange(2)[None, :] == tgt[:, None]) - 0.5)
    np.testing.assert_allclose(out["dx"], want_dx, atol=1e-7)
