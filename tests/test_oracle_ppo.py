"""Pins for oracle.ppo (S4) and the composed S3∘S4 gradient: hand-evaluated clip table,
ratio == 1, decoupled == standard, staleness, torch float64 autograd (library routine),
finite differences, micro-batch split invariance."""
import numpy as np
import pytest
import torch

from oracle import logprob as L
from oracle import path as P
from oracle import ppo as O
from tests.conftest import read_golden

CLIP = read_golden("ppo_clip_table.csv")


@pytest.mark.parametrize("row", CLIP)
def test_clip_table(row):
    a, rho, loss, grad = (float(v) for v in row)
    # N_tok = 1; logp_behav chosen so that exp(logp - logp_behav) == rho exactly
    lb = np.array([0.0])
    lp = np.array([np.log(rho)])
    out = O.ppo_loss(lp, lb, np.array([a]), np.array([True]), np.array([0]), n_tok=1.0)
    r = out["ratio"][0]
    assert abs(out["loss_tok"][0] - loss) < 1e-12 + 1e-12 * abs(loss) + 2 * abs(r - rho)
    if r == rho or a == 0 or rho not in (0.8, 1.2):
        assert abs(out["grad"][0] - grad) < 1e-12 + 2 * abs(r - rho)
    else:  # exp(log(rho)) missed the bound by an ulp: near-tie, either branch is correct
        assert out["near_tie"][0]


def test_ratio_one():
    rng = np.random.default_rng(0)
    n = 50
    lp = rng.normal(-3, 1, size=n)
    A = rng.normal(size=n)
    m = rng.random(n) > 0.2
    out = O.ppo_loss(lp, lp.copy(), A, m, np.zeros(n, int), n_tok=float(m.sum()))
    N = m.sum()
    assert abs(out["stats"]["loss"] - (-(A * m).sum() / N)) < 1e-14
    np.testing.assert_allclose(out["grad"], np.where(m, -A / N, 0.0), rtol=1e-15)
    assert out["stats"]["n_clipped"] == 0 and out["stats"]["kl_k3_sum"] == 0.0


def test_decoupled_with_prox_equal_behav_is_standard():
    rng = np.random.default_rng(1)
    n = 64
    lp, lb, A = rng.normal(-2, 1, n), rng.normal(-2, 1, n), rng.normal(size=n)
    m = np.ones(n, bool)
    s = O.ppo_loss(lp, lb, A, m, np.zeros(n, int))
    d = O.ppo_loss(lp, lb, A, m, np.zeros(n, int), logp_prox=lb.copy())
    assert np.array_equal(s["loss_tok"], d["loss_tok"]) and np.array_equal(s["grad"], d["grad"])


def test_decoupled_matches_autograd():
    rng = np.random.default_rng(2)
    n = 200
    lp, lb, lpp = rng.normal(-2, .3, n), rng.normal(-2, .3, n), rng.normal(-2, .3, n)
    A = rng.normal(size=n)
    out = O.ppo_loss(lp, lb, A, np.ones(n, bool), np.zeros(n, int), logp_prox=lpp, is_cap=2.0,
                     eps_low=0.1, eps_high=0.3, n_tok=float(n))
    t = torch.tensor(lp, dtype=torch.float64, requires_grad=True)
    w = torch.clamp(torch.exp(torch.tensor(lpp - lb)), max=2.0)
    rho = torch.exp(t - torch.tensor(lpp))
    At = torch.tensor(A)
    loss = (-w * torch.minimum(rho * At, torch.clamp(rho, 0.9, 1.3) * At)).sum() / n
    loss.backward()
    assert abs(loss.item() - out["stats"]["loss"]) < 1e-13
    np.testing.assert_allclose(out["grad"], t.grad.numpy(), rtol=1e-12, atol=1e-15)


def test_staleness_bound():
    lp = np.full(4, -1.0)
    out = O.ppo_loss(lp, lp, np.ones(4), np.ones(4, bool), np.array([0, 1, 2, -1]),
                     max_staleness=1)
    assert out["mask"].tolist() == [True, True, False, False]
    assert out["stats"]["n_stale_tok"] == 1 and out["stats"]["n_bad_lag"] == 1
    assert out["grad"][2] == 0 and out["grad"][3] == 0


def _composed_loss(x, tgt, lb, A, lag, n_tok):
    f = L.log_softmax_gather(x, tgt)
    o = O.ppo_loss(f["logp"], lb, A, f["status"] == 0, lag, n_tok=n_tok)
    return f, o


def test_composed_finite_differences_wrt_logits():
    rng = np.random.default_rng(3)
    R, V = 6, 12
    x = rng.normal(0, 1, size=(R, V))
    tgt = rng.integers(0, V, size=R)
    f0 = L.log_softmax_gather(x, tgt)
    lb = f0["logp"] + rng.normal(0, 0.05, R)     # ratios well inside (0.8, 1.2)
    A = rng.normal(size=R)
    lag = np.zeros(R, int)
    f, o = _composed_loss(x, tgt, lb, A, lag, float(R))
    dx = L.log_softmax_grad(x, tgt, f["lse"], o["grad"])
    h = 1e-5
    for r in range(R):
        for j in range(V):
            xp, xm = x.copy(), x.copy()
            xp[r, j] += h
            xm[r, j] -= h
            fd = (_composed_loss(xp, tgt, lb, A, lag, float(R))[1]["stats"]["loss"] -
                  _composed_loss(xm, tgt, lb, A, lag, float(R))[1]["stats"]["loss"]) / (2 * h)
            assert abs(fd - dx[r, j]) <= 1e-6 * max(1e-3, abs(dx[r, j])) + 1e-10


def test_micro_batch_split_invariance():
    rng = np.random.default_rng(4)
    R, V = 40, 33
    x = rng.normal(size=(R, V))
    tv = dict(valid=rng.random(R) > 0.1, lag=rng.integers(0, 3, R), adv=rng.normal(size=R),
              target=rng.integers(-1, V, R), logp_behav=rng.normal(-3.5, 0.3, R))
    full = P.loss_and_grad(x, tv, n_tok=37.0)
    parts = [np.arange(0, 13), np.arange(13, 30), np.arange(30, 40)]
    outs = [P.loss_and_grad(x[p], tv, n_tok=37.0, rows=p) for p in parts]
    for k in ("loss", "n_clipped", "kl_k3_sum", "entropy_sum", "ratio_sum", "n_loss_tok"):
        assert abs(sum(o["stats"][k] for o in outs) - full["stats"][k]) <= 1e-12 * max(1, abs(full["stats"][k]))
    assert np.array_equal(np.concatenate([o["dx"] for o in outs]), full["dx"])
