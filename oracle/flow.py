"""NEXT-4 oracle: log-likelihood of a flow/diffusion policy's action chunk as a chain of
Gaussian denoising transitions (TEST INFRASTRUCTURE ONLY).

Paper: pi_0 / pi_0.5 (flow matching) and GR00T N1.5 (diffusion) are trained with the same
asynchronous pipeline ("VLA models often integrate Diffusion modules ...
multi-step denoising"); Table 2 fixes "Model Num Step" = 4 denoising steps and the
chunk sizes. The paper never writes the policy likelihood the PPO ratio needs.
Reading R25: the sampled chunk is the end of a K-step stochastic denoising
chain x_0 -> x_1 -> ... -> x_K with Gaussian transitions
    x_{k+1} ~ N(mu_theta(x_k, k), diag(sigma_{k,d}^2)),   k = 0 .. K-1,
so the log-likelihood of the decision step is the sum of the K transition log-densities
    logp = sum_k sum_d [ -(x_{k+1,d} - mu_{k,d})^2 / (2 sigma_{k,d}^2) - ln sigma_{k,d}
                         - ln(2 pi) / 2 ],
with sigma either a per-step schedule sigma_k (no gradient) or a learned ln sigma_{k,d}.
Gradients of a loss L through g = dL/dlogp:
    dL/dmu_{k,d}        = g (x - mu) / sigma^2
    dL/d ln sigma_{k,d} = g ((x - mu)^2 / sigma^2 - 1).
Entropy of the chain's transitions (a statistic): H = sum_k sum_d (ln sigma + ln(2 pi e)/2).
The PPO surrogate over these per-step log-probs is oracle.ppo.ppo_loss with one "token"
per decision step (the chunk's ratio). Everything is float64.
"""
from __future__ import annotations

import numpy as np

LN_2PI = float(np.log(2.0 * np.pi))


def _sigma(rows, K, D, sigma_k=None, log_std=None):
    if log_std is not None:
        ls = np.asarray(log_std, np.float64).reshape(rows, K, D)
        return np.exp(ls), ls
    s = np.broadcast_to(np.asarray(sigma_k, np.float64).reshape(1, K, 1), (rows, K, D))
    return s, np.log(s)


def chain_logprob(mu, x, sigma_k=None, log_std=None):
    """mu, x: [rows, K, D]. Returns dict(logp [rows], entropy [rows], z [rows, K, D])."""
    mu = np.asarray(mu, np.float64)
    x = np.asarray(x, np.float64)
    R, K, D = mu.shape
    s, ls = _sigma(R, K, D, sigma_k, log_std)
    z = (x - mu) / s
    logp = (-0.5 * z * z - ls - 0.5 * LN_2PI).sum(axis=(1, 2))
    ent = (ls + 0.5 * (LN_2PI + 1.0)).sum(axis=(1, 2))
    return dict(logp=logp, entropy=ent, z=z)


def chain_grads(mu, x, g, sigma_k=None, log_std=None):
    """dL/dmu and dL/dln sigma for per-row g = dL/dlogp."""
    mu = np.asarray(mu, np.float64)
    x = np.asarray(x, np.float64)
    R, K, D = mu.shape
    s, _ = _sigma(R, K, D, sigma_k, log_std)
    z = (x - mu) / s
    gr = np.asarray(g, np.float64)[:, None, None]
    return dict(dmu=gr * z / s, dlog_std=gr * (z * z - 1.0))
