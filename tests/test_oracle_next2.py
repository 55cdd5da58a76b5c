"""Pins for the NEXT-2 oracle functions (loss variants; paper-silent, readings R19-R23):
torch float64 autograd of the composed objectives, hand-evaluated tables and closed forms."""
import itertools

import numpy as np
import pytest
import torch

from oracle import advantages as A
from oracle import logprob as L
from oracle import path as P
from oracle import ppo as O


def _torch_objective(x, tgt, lb, adv, m, N, *, eps=(0.2, 0.2), dual=0.0, lref=None, kl=0.0,
                     ent=0.0):
    """The composed loss written with torch ops (log_softmax, minimum, clamp, exp)."""
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    ls = torch.log_softmax(xt, dim=1)
    logp = ls[torch.arange(len(tgt)), torch.tensor(tgt)]
    rho = torch.exp(logp - torch.tensor(lb))
    At = torch.tensor(adv)
    J = torch.minimum(rho * At, torch.clamp(rho, 1 - eps[0], 1 + eps[1]) * At)
    if dual:
        J = torch.where(At < 0, torch.maximum(J, dual * At), J)
    Lr = -J
    if lref is not None and kl:
        lr = torch.tensor(lref) - logp
        Lr = Lr + kl * (torch.exp(lr) - lr - 1)
    mt = torch.tensor(m, dtype=torch.float64)
    loss = (Lr * mt).sum() / N
    if ent:
        H = -(torch.exp(ls) * ls).sum(dim=1)
        loss = loss - ent * (H * mt).sum() / N
    loss.backward()
    return loss.item(), xt.grad.numpy()


def _far_from_ties(rho, eps=(0.2, 0.2), dual=0.0, tol=1e-3):
    bounds = [1 - eps[0], 1 + eps[1]] + ([dual] if dual else [])
    return all(np.all(np.abs(rho - b) > tol) for b in bounds)


@pytest.mark.parametrize("dual,kl,ent", [(0.0, 0.0, 0.0), (3.0, 0.0, 0.0), (0.0, 0.1, 0.0),
                                         (0.0, 0.0, 0.01), (2.5, 0.05, 0.02)])
def test_composed_loss_and_logit_gradient_match_autograd(dual, kl, ent):
    rng = np.random.default_rng(int(dual * 10 + kl * 100 + ent * 1000))
    R, V = 40, 17
    x = rng.normal(0, 1.5, size=(R, V))
    tgt = rng.integers(0, V, R)
    f = L.log_softmax_gather(x, tgt)
    # ratios spread over all branches incl. beyond the dual-clip bound, away from ties
    lr = rng.choice([-1.2, -0.5, -0.1, 0.05, 0.15, 0.5, 1.3], R) + rng.normal(0, 0.01, R)
    lb = f["logp"] - lr
    adv = rng.normal(0, 1, R)
    m = rng.random(R) > 0.1
    lref = f["logp"] + rng.normal(0, 0.3, R)
    assert _far_from_ties(np.exp(lr), dual=dual)
    N = 37.0
    tv = dict(valid=m, lag=np.zeros(R, int), adv=adv, target=tgt, logp_behav=lb)
    out = P.loss_and_grad(x, tv, n_tok=N, dual_clip=dual, logp_ref=lref, kl_coef=kl, ent_coef=ent)
    loss_t, grad_t = _torch_objective(x, tgt, lb, adv, m, N, dual=dual,
                                      lref=lref if kl else None, kl=kl, ent=ent)
    assert abs(out["stats"]["loss"] - loss_t) < 1e-12
    np.testing.assert_allclose(out["dx"], grad_t, rtol=1e-10, atol=1e-14)


def test_dual_clip_table():
    # A = -1, c = 3, eps = 0.2: J = min(-rho, -clip(rho)); dual branch when -3 > J (rho > 3)
    for rho, loss, grad, dual in ((0.5, 0.8, 0.0, False), (2.0, 2.0, 2.0, False),
                                  (4.0, 3.0, 0.0, True)):
        o = O.ppo_loss(np.array([np.log(rho)]), np.zeros(1), np.array([-1.0]), np.array([True]),
                       np.zeros(1, int), n_tok=1.0, dual_clip=3.0)
        assert abs(o["loss_tok"][0] - loss) < 1e-12 and abs(o["grad"][0] - grad) < 1e-12
        assert bool(o["dual"][0]) == dual
    # A > 0 never takes the dual branch
    o = O.ppo_loss(np.array([np.log(5.0)]), np.zeros(1), np.array([1.0]), np.array([True]),
                   np.zeros(1, int), n_tok=1.0, dual_clip=3.0)
    assert not o["dual"][0] and abs(o["loss_tok"][0] + 1.2) < 1e-12


def test_kl_reference_closed_forms():
    lp = np.array([-2.0, -2.0, -1.0])
    lref = np.array([-2.0, -2.0 + np.log(2.0), -1.0 - np.log(2.0)])
    o = O.ppo_loss(lp, lp, np.zeros(3), np.ones(3, bool), np.zeros(3, int), n_tok=1.0,
                   logp_ref=lref, kl_coef=0.5)
    k3 = o["loss_tok"] / 0.5
    np.testing.assert_allclose(k3, [0.0, 1 - np.log(2.0), 0.5 + np.log(2.0) - 1], atol=1e-15)
    np.testing.assert_allclose(o["grad"], 0.5 * np.array([0.0, 1 - 2.0, 1 - 0.5]), atol=1e-15)
    assert abs(o["stats"]["kl_ref_sum"] - k3.sum()) < 1e-15


def test_entropy_bonus_gradient_pins():
    # uniform row: entropy is maximal => zero gradient; finite differences elsewhere
    x = np.zeros((1, 8))
    f = L.log_softmax_gather(x, [0])
    assert np.abs(L.entropy_bonus_grad(x, f["lse"], f["entropy"], [1.0])).max() < 1e-15
    rng = np.random.default_rng(3)
    x = rng.normal(size=(2, 9))
    f = L.log_softmax_gather(x, [0, 1])
    g = L.entropy_bonus_grad(x, f["lse"], f["entropy"], [1.0, 1.0])   # d(-H)/dx
    h = 1e-6
    for r in range(2):
        for j in range(9):
            xp, xm = x.copy(), x.copy()
            xp[r, j] += h
            xm[r, j] -= h
            fd = -(L.log_softmax_gather(xp, [0, 1])["entropy"][r] -
                   L.log_softmax_gather(xm, [0, 1])["entropy"][r]) / (2 * h)
            assert abs(fd - g[r, j]) < 1e-8
    # -inf columns contribute nothing
    x2 = np.array([[0.0, 1.0, -np.inf]])
    f2 = L.log_softmax_gather(x2, [0])
    assert L.entropy_bonus_grad(x2, f2["lse"], f2["entropy"], [1.0])[0, 2] == 0.0


@pytest.mark.parametrize("prox,cap,dual", [(False, 0.0, 0.0), (True, 0.0, 0.0), (True, 1.05, 0.0),
                                            (False, 0.0, 1.3), (True, 1.1, 1.3)])
def test_chunk_ratio_matches_autograd_and_reduces_to_token_level(prox, cap, dual):
    rng = np.random.default_rng(4)
    S, Atok = 40, 5
    R = S * Atok
    logp = rng.normal(-3, 0.5, R)
    lb = logp - rng.normal(0, 0.08, R)
    lpp = lb + rng.normal(0, 0.03, R)
    adv = rng.normal(size=S)
    m = rng.random(R) > 0.15
    st = np.arange(R) // Atok
    kw = dict(logp_prox=lpp if prox else None, is_cap=cap, dual_clip=dual)
    o = O.ppo_loss_chunk(logp, lb, adv, m, st, S, **kw)
    assert not o["near_tie_step"].any()
    if dual:
        assert o["dual"].any()                     # the dual branch is exercised
    if cap:
        assert (o["w_step"] == cap).any()          # the cap binds somewhere
    t = torch.tensor(logp, requires_grad=True)
    mt = torch.tensor(m, dtype=torch.float64)
    base = torch.tensor(lpp if prox else lb)
    lr = torch.zeros(S, dtype=torch.float64).index_add(0, torch.tensor(st), (t - base) * mt)
    rho = torch.exp(lr)
    w = torch.ones(S, dtype=torch.float64)
    if prox:                                       # detached importance weight (R12)
        w = torch.exp(torch.zeros(S, dtype=torch.float64).index_add(
            0, torch.tensor(st), torch.tensor(lpp - lb) * mt))
        if cap:
            w = torch.clamp(w, max=cap)
    At = torch.tensor(adv)
    J = torch.minimum(rho * At, torch.clamp(rho, 0.8, 1.2) * At)
    if dual:
        J = torch.where(At < 0, torch.maximum(J, dual * At), J)
    ms = torch.tensor(o["mask_step"], dtype=torch.float64)
    loss = -(w * J * ms).sum() / ms.sum()
    loss.backward()
    assert abs(loss.item() - o["stats"]["loss"]) < 1e-13
    np.testing.assert_allclose(o["grad"], t.grad.numpy() * m, atol=1e-15)
    # one token per step == the token-level surrogate (same knobs)
    o1 = O.ppo_loss_chunk(logp[:S], lb[:S], adv, np.ones(S, bool), np.arange(S), S,
                          logp_prox=lpp[:S] if prox else None, is_cap=cap, dual_clip=dual)
    o2 = O.ppo_loss(logp[:S], lb[:S], adv, np.ones(S, bool), np.zeros(S, int),
                    logp_prox=lpp[:S] if prox else None, is_cap=cap, dual_clip=dual)
    np.testing.assert_allclose(o1["grad"], o2["grad"], rtol=1e-14, atol=1e-300)
    assert abs(o1["stats"]["loss"] - o2["stats"]["loss"]) < 1e-14
    assert o1["stats"]["n_dual_clipped"] == o2["stats"]["n_dual_clipped"]


def test_chunk_decoupled_with_prox_equal_behav_is_standard():
    rng = np.random.default_rng(9)
    S, Atok = 30, 4
    R = S * Atok
    logp = rng.normal(-3, 0.5, R)
    lb = logp - rng.normal(0, 0.1, R)
    adv = rng.normal(size=S)
    m = rng.random(R) > 0.1
    st = np.arange(R) // Atok
    a = O.ppo_loss_chunk(logp, lb, adv, m, st, S)
    b = O.ppo_loss_chunk(logp, lb, adv, m, st, S, logp_prox=lb)
    assert np.array_equal(a["grad"], b["grad"]) and a["stats"] == b["stats"]


def test_value_loss_matches_autograd_and_special_cases():
    rng = np.random.default_rng(5)
    n = 300
    v, vo, R = rng.normal(size=n), rng.normal(size=n), rng.normal(size=n)
    m = rng.random(n) > 0.1
    d = np.abs(v - vo)
    v = np.where(np.abs(d - 0.2) < 1e-3, v + 0.01, v)     # away from the clip boundary
    o = O.value_loss(v, vo, R, m, clip_eps=0.2)
    t = torch.tensor(v, requires_grad=True)
    vc = torch.tensor(vo) + torch.clamp(t - torch.tensor(vo), -0.2, 0.2)
    Lt = 0.5 * torch.maximum((t - torch.tensor(R)) ** 2, (vc - torch.tensor(R)) ** 2)
    loss = (Lt * torch.tensor(m, dtype=torch.float64)).sum() / m.sum()
    loss.backward()
    assert abs(loss.item() - o["stats"]["loss"]) < 1e-13
    np.testing.assert_allclose(o["grad"], t.grad.numpy(), atol=1e-15)
    plain = O.value_loss(v, vo, R, m, clip_eps=0.0)
    np.testing.assert_allclose(plain["grad"], np.where(m, v - R, 0) / m.sum(), rtol=1e-15)
    same = O.value_loss(vo, vo, R, m, clip_eps=0.2)       # v == v_old: no clipping possible
    assert same["stats"]["n_clipped"] == 0


def test_gae_truncation_pins():
    rng = np.random.default_rng(6)
    E, T, g = 3, 9, 0.97
    r, V, lv = rng.normal(size=(E, T)), rng.normal(size=(E, T)), rng.normal(size=E)
    B = rng.normal(size=(E, T))
    v = np.ones((E, T))
    # lambda = 0: a truncated step's advantage is the TD error against the bootstrap value
    d = np.zeros((E, T), int)
    d[:, 4] = 2
    a0, _ = A.gae(r, V, d, v, lv, g, 0.0, boot_value=B)
    assert np.allclose(a0[:, 4], r[:, 4] + g * B[:, 4] - V[:, 4], atol=1e-14)
    # truncation with B_t = V_{t+1} and lambda = 0 equals "not done"
    B2 = np.concatenate([V[:, 1:], lv[:, None]], axis=1)
    a_tr, _ = A.gae(r, V, d, v, lv, g, 0.0, boot_value=B2)
    a_nd, _ = A.gae(r, V, np.zeros((E, T), int), v, lv, g, 0.0)
    np.testing.assert_allclose(a_tr, a_nd, atol=1e-14)
    # brute force over all done codes {0,1,2} for T = 5
    lam = 0.9
    for codes in itertools.product([0, 1, 2], repeat=5):
        dd = np.array([codes])
        r1, V1, B1, lv1 = r[:1, :5], V[:1, :5], B[:1, :5], lv[:1]
        adv, _ = A.gae(r1, V1, dd, np.ones((1, 5)), lv1, g, lam, boot_value=B1)
        for t in range(5):
            # explicit: sum_l (g lam)^l prod nt * delta, delta with the bootstrap
            s, prod = 0.0, 1.0
            for k in range(t, 5):
                ntk = 1.0 if dd[0, k] == 0 else 0.0
                nV = V1[0, k + 1] if k + 1 < 5 else lv1[0]
                dk = r1[0, k] + g * (ntk * nV + (dd[0, k] == 2) * B1[0, k]) - V1[0, k]
                s += (g * lam) ** (k - t) * prod * dk
                prod *= ntk
            assert abs(adv[0, t] - s) < 1e-12
