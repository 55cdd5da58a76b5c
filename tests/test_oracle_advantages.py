"""Pins for oracle.advantages (S2a GAE + whitening, S2b GRPO): closed forms, special cases
that reduce to simpler definitions, library routines and brute force — never the CUDA path."""
import itertools

import numpy as np
import pytest

from oracle import advantages as A
from tests.conftest import read_golden


def _gae(r, V, d, v, lv, g, l):
    return A.gae(np.asarray(r), np.asarray(V), np.asarray(d), np.asarray(v), lv, g, l)


@pytest.mark.parametrize("row", read_golden("gae_closed_form.csv"))
def test_gae_constant_reward_closed_form(row):
    T, t, expected = int(row[0]), int(row[1]), float(row[2])
    E = 3
    adv, ret = _gae(np.ones((E, T)), np.zeros((E, T)), np.zeros((E, T)), np.ones((E, T)),
                    np.zeros(E), 0.99, 0.95)
    assert abs(adv[0, t] - expected) < 5e-9
    gl = 0.99 * 0.95
    closed = (1 - gl ** (T - np.arange(T))) / (1 - gl)
    np.testing.assert_allclose(adv[1], closed, rtol=1e-13)


def test_gae_gamma_lambda_one_telescopes():
    # gamma = lambda = 1, no done: A_t = sum_{k>=t} r_k + V_T - V_t (any V)
    rng = np.random.default_rng(1)
    E, T = 4, 17
    r, V, lv = rng.normal(size=(E, T)), rng.normal(size=(E, T)), rng.normal(size=E)
    adv, _ = _gae(r, V, np.zeros((E, T)), np.ones((E, T)), lv, 1.0, 1.0)
    expect = np.cumsum(r[:, ::-1], axis=1)[:, ::-1] + lv[:, None] - V
    np.testing.assert_allclose(adv, expect, rtol=1e-12, atol=1e-12)
    adv2, _ = _gae(np.ones((2, 32)), np.zeros((2, 32)), np.zeros((2, 32)), np.ones((2, 32)),
                   np.zeros(2), 1.0, 1.0)
    assert adv2[0, 0] == 32.0 and adv2[0, 31] == 1.0


def test_gae_lambda_zero_is_td_error_and_lambda_one_is_return():
    rng = np.random.default_rng(2)
    E, T, g = 3, 12, 0.9
    r, V, lv = rng.normal(size=(E, T)), rng.normal(size=(E, T)), rng.normal(size=E)
    d = (rng.random((E, T)) < 0.2).astype(np.float64)
    adv0, _ = _gae(r, V, d, np.ones((E, T)), lv, g, 0.0)
    Vn = np.concatenate([V[:, 1:], lv[:, None]], axis=1)
    np.testing.assert_allclose(adv0, r + g * (1 - d) * Vn - V, rtol=1e-12, atol=1e-12)
    # lambda = 1: discounted return cut at done (bootstrap from last_value if no done)
    adv1, ret1 = _gae(r, V, d, np.ones((E, T)), lv, g, 1.0)
    for e in range(E):
        for t in range(T):
            G, k = 0.0, t
            while True:
                G += g ** (k - t) * r[e, k]
                if d[e, k]:
                    break
                if k == T - 1:
                    G += g ** (T - t) * lv[e]
                    break
                k += 1
            assert abs(adv1[e, t] - (G - V[e, t])) < 1e-11
            assert abs(ret1[e, t] - G) < 1e-11


def test_gae_done_everywhere():
    rng = np.random.default_rng(3)
    r, V = rng.normal(size=(2, 9)), rng.normal(size=(2, 9))
    adv, _ = _gae(r, V, np.ones((2, 9)), np.ones((2, 9)), rng.normal(size=2), 0.99, 0.95)
    np.testing.assert_allclose(adv, r - V, rtol=1e-14)


def test_gae_brute_force_double_sum_all_done_patterns():
    """A_t = sum_l (g l)^l prod_{k<l} nt_{t+k} delta_{t+l}, every done pattern, T <= 8,
    with random unfilled slots (R8)."""
    rng = np.random.default_rng(4)
    g, lam = 0.97, 0.9
    for T in (1, 2, 5, 8):
        for bits in itertools.product([0, 1], repeat=T):
            d = np.array([bits], np.float64)
            v = (rng.random((1, T)) > 0.15).astype(np.float64)
            r, V, lv = rng.normal(size=(1, T)), rng.normal(size=(1, T)), rng.normal(size=1)
            adv, _ = _gae(r, V, d, v, lv, g, lam)
            vn = np.append(v[0, 1:], 1.0)
            Vn = np.append(V[0, 1:], lv[0])
            nt = v[0] * (1 - d[0]) * vn
            delta = v[0] * (r[0] + g * nt * Vn - V[0])
            for t in range(T):
                s, prod = 0.0, 1.0
                for l in range(T - t):
                    s += (g * lam) ** l * prod * delta[t + l]
                    prod *= nt[t + l]
                assert abs(adv[0, t] - s) < 1e-12


def test_gae_unfilled_slots_cut_recursion():
    r = np.ones((1, 6))
    V = np.zeros((1, 6))
    v = np.array([[1, 1, 0, 1, 1, 1]], np.float64)
    adv, ret = _gae(r, V, np.zeros((1, 6)), v, np.zeros(1), 1.0, 1.0)
    assert adv[0].tolist() == [2.0, 1.0, 0.0, 3.0, 2.0, 1.0]
    assert ret[0, 2] == 0.0


def test_whiten_matches_numpy_std():
    rng = np.random.default_rng(5)
    a = rng.normal(3.0, 2.0, size=(6, 40))
    v = rng.random((6, 40)) > 0.3
    w = A.whiten(a, v, eps=1e-8)
    sel = a[v]
    mu, sd = sel.mean(), sel.std(ddof=1)
    np.testing.assert_allclose(w[v], (sel - mu) / (sd + 1e-8), rtol=1e-12)
    assert abs(w[v].mean()) < 1e-12
    assert abs(w[v].std(ddof=1) - sd / (sd + 1e-8)) < 1e-12
    assert (w[~v] == 0).all()
    # sharded stats give the same result
    st = A.whiten_stats(a, v)
    np.testing.assert_allclose(A.whiten(a, v, 1e-8, stats=st), w, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("row", read_golden("grpo_values.csv")[1:])
def test_grpo_printed_values(row):
    R = np.array([float(x) for x in row[0].split()])
    exp = np.array([float(x) for x in row[2].split()])
    got = A.grpo(R, np.zeros(len(R), int), eps=1e-6, unbiased=(row[1] == "unbiased"))
    np.testing.assert_allclose(got, exp, atol=5e-9)


def test_grpo_properties():
    rng = np.random.default_rng(6)
    R = rng.normal(size=24)
    gid = np.repeat(np.arange(6), 4)
    a = A.grpo(R, gid)
    for g in range(6):
        m = gid == g
        assert abs(a[m].sum()) < 1e-12
        sd = R[m].std(ddof=1)
        np.testing.assert_allclose(a[m], (R[m] - R[m].mean()) / (sd + 1e-6), rtol=1e-12)
        # population flag uses ddof=0
        ap = A.grpo(R[m], np.zeros(4, int), unbiased=False)
        np.testing.assert_allclose(ap, (R[m] - R[m].mean()) / (R[m].std() + 1e-6), rtol=1e-12)
    # affine invariance (up to eps)
    a2 = A.grpo(3.0 * R + 7.0, gid)
    np.testing.assert_allclose(a2, a, atol=1e-5)
    # all-equal groups and singletons give exactly 0
    assert (A.grpo(np.full(8, 0.3), np.repeat([0, 1], 4)) == 0).all()
    assert (A.grpo(np.array([1.0, 2.0]), np.array([0, 1])) == 0).all()
    # interleaved membership = same as contiguous after permutation
    perm = np.argsort(gid % 6 * 100 + np.arange(24))
    np.testing.assert_allclose(A.grpo(R[perm], gid[perm]), a[perm], rtol=1e-13)


def test_step_counts_brute_force():
    rng = np.random.default_rng(7)
    E, T, Atok = 3, 5, 4
    valid = rng.random((E, T)) > 0.2
    version = 10 - rng.integers(-1, 4, size=(E, T))
    tokens = rng.integers(-1, 5, size=(E, T, Atok))
    c = A.step_counts(valid, version, tokens, 10, 1)
    nv = nt = ns = nb = nls = 0
    for e in range(E):
        for t in range(T):
            if not valid[e, t]:
                continue
            nv += 1
            lag = 10 - version[e, t]
            if lag < 0:
                nb += 1
            elif lag > 1:
                ns += 1
            else:
                k = sum(1 for a in range(Atok) if tokens[e, t, a] >= 0)
                nt += k
                nls += k > 0
    assert c == dict(n_valid=nv, n_tok=nt, n_stale=ns, n_bad=nb, n_loss_steps=nls)
