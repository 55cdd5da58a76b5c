"""Pins for the NEXT-4 oracle (oracle/flow.py): the log-likelihood of a flow/diffusion
policy's action chunk as a chain of K Gaussian denoising transitions (reading R25;
P:39/Table 2 "Model Num Step" = 4).

  * hand-evaluated normal densities (tests/golden/gaussian_logpdf.csv);
  * the chain sum equals scipy's multivariate normal log-density of the flattened chunk
    with diagonal covariance (an independent formulation);
  * gradients and entropy equal torch.distributions.Normal (fp64 autograd / entropy);
  * central finite differences of logp w.r.t. mu and ln sigma;
  * x = mu: logp = -sum ln sigma - K D ln(2 pi)/2 (closed form); the chunk ratio composed
    with the PPO oracle is exactly 1 on-policy.
"""
import csv
import os

import numpy as np
import torch
from scipy import stats

from oracle import flow as F
from oracle import ppo as O_ppo

GOLD = os.path.join(os.path.dirname(__file__), "golden", "gaussian_logpdf.csv")


def _case(R=6, K=4, D=70, seed=0, learned=False):
    rng = np.random.default_rng(seed)
    mu = rng.normal(size=(R, K, D))
    sig_k = np.array([0.8, 0.5, 0.3, 0.1])[:K]
    log_std = rng.normal(-1.0, 0.4, size=(R, K, D)) if learned else None
    s = np.exp(log_std) if learned else sig_k[None, :, None]
    x = mu + s * rng.normal(size=(R, K, D))
    return mu, x, sig_k, log_std


def test_golden_values():
    rows = list(csv.DictReader(l for l in open(GOLD) if not l.startswith("#")))
    assert len(rows) == 4
    for r in rows:
        o = F.chain_logprob(np.array([[[float(r["mu"])]]]), np.array([[[float(r["x"])]]]),
                            sigma_k=np.array([float(r["sigma"])]))
        assert abs(o["logp"][0] - float(r["logp"])) < 1e-14, r


def test_matches_multivariate_normal():
    for learned in (False, True):
        mu, x, sk, ls = _case(learned=learned)
        o = F.chain_logprob(mu, x, sigma_k=sk, log_std=ls)
        R, K, D = mu.shape
        for r in range(R):
            var = (np.exp(2 * ls[r]) if learned else np.broadcast_to((sk ** 2)[:, None], (K, D))).ravel()
            ref = stats.multivariate_normal(mean=mu[r].ravel(), cov=np.diag(var)).logpdf(x[r].ravel())
            assert abs(o["logp"][r] - ref) <= 1e-10 * max(1.0, abs(ref))


def test_grads_and_entropy_vs_torch():
    for learned in (False, True):
        mu, x, sk, ls = _case(seed=3, learned=learned)
        R, K, D = mu.shape
        g = np.linspace(-2.0, 1.5, R)
        m = torch.tensor(mu, requires_grad=True)
        l_t = torch.tensor(ls if learned else np.broadcast_to(np.log(sk)[None, :, None], (R, K, D)).copy(),
                           requires_grad=True)
        dist = torch.distributions.Normal(m, l_t.exp())
        lp = dist.log_prob(torch.tensor(x)).sum(dim=(1, 2))
        (lp * torch.tensor(g)).sum().backward()
        o = F.chain_logprob(mu, x, sigma_k=sk, log_std=ls)
        gr = F.chain_grads(mu, x, g, sigma_k=sk, log_std=ls)
        np.testing.assert_allclose(o["logp"], lp.detach().numpy(), rtol=1e-12, atol=1e-10)
        np.testing.assert_allclose(gr["dmu"], m.grad.numpy(), rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(gr["dlog_std"], l_t.grad.numpy(), rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(o["entropy"], dist.entropy().sum(dim=(1, 2)).detach().numpy(), rtol=1e-12)


def test_finite_differences():
    mu, x, _, ls = _case(R=2, K=2, D=3, seed=5, learned=True)
    g = np.array([0.7, -1.3])
    gr = F.chain_grads(mu, x, g, log_std=ls)
    h = 1e-6
    for idx in [(0, 0, 0), (1, 1, 2), (0, 1, 1)]:
        for name, arr in (("dmu", mu), ("dlog_std", ls)):
            a1, a2 = arr.copy(), arr.copy()
            a1[idx] += h
            a2[idx] -= h
            f = lambda a: (F.chain_logprob(a if name == "dmu" else mu, x, log_std=a if name == "dlog_std" else ls)["logp"] * g).sum()  # noqa: E731
            fd = (f(a1) - f(a2)) / (2 * h)
            assert abs(fd - gr[name][idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx)


def test_on_policy_closed_forms():
    mu, _, sk, _ = _case(R=5, seed=7)
    R, K, D = mu.shape
    o = F.chain_logprob(mu, mu, sigma_k=sk)                       # x = mu
    np.testing.assert_allclose(o["logp"], -D * np.log(sk).sum() - K * D * F.LN_2PI / 2, rtol=1e-14)
    gr = F.chain_grads(mu, mu, np.ones(R), sigma_k=sk)
    assert not gr["dmu"].any()
    np.testing.assert_array_equal(gr["dlog_std"], -1.0)
    # chunk ratio through the PPO oracle, one "token" per decision step: on-policy => rho = 1
    mu2, x2, sk2, _ = _case(R=8, seed=9)
    lp = F.chain_logprob(mu2, x2, sigma_k=sk2)["logp"]
    adv = np.linspace(-1, 1, 8)
    p = O_ppo.ppo_loss(lp, lp, adv, np.ones(8, bool), np.zeros(8, int), n_tok=8.0)
    np.testing.assert_array_equal(p["ratio"], 1.0)
    np.testing.assert_allclose(p["grad"], -adv / 8.0, rtol=1e-15)
