"""S2 oracle: GAE (+ global whitening) and GRPO group normalisation (TEST INFRASTRUCTURE ONLY).

The paper does not define the learning algorithm ("Hyperparameters related to the
optimizer and learning algorithm ... are omitted", App. A). The
definitions below are the textbook ones, written out in their own order:
  * GAE: Schulman, Moritz, Levine, Jordan, Abbeel 2016, eq. (16) recursion
    A_t = delta_t + gamma*lambda*A_{t+1}, delta_t = r_t + gamma V_{t+1} - V_t.
  * GRPO: Shao et al. 2024, outcome supervision A_i = (r_i - mean(r)) / std(r).
Readings R7 (done = termination), R8 (unfilled slots cut the recursion), R9 (global,
unbiased whitening, eps on sigma), R10 (unbiased group std, eps on sigma) are listed in
DESIGN.md §2. Everything is float64.
"""
from __future__ import annotations

import numpy as np


def gae(reward, value, done, valid, last_value, gamma: float, lam: float, boot_value=None):
    """Per env, t = T-1 .. 0 (truncation = NEXT-2 reading R23):
        v_t   = valid(e, t);                 v_T := 1
        nt_t  = v_t * [done_t == 0] * v_{t+1}
        tr_t  = [done_t == 2]  (time-limit truncation: bootstrap B_t = boot_value, then cut)
        nV_t  = last_value[e] if t == T-1 else V_{t+1}
        delta = v_t * (r_t + gamma * (nt_t * nV_t + tr_t * B_t) - V_t)
        A_t   = delta + gamma * lam * nt_t * A_{t+1},   A_T = 0
        R_t   = A_t + V_t  (valid steps; 0 elsewhere)
    done_t = 1 is a termination (reading R7). Returns (adv, ret) float64 [E, T].
    """
    r = np.asarray(reward, np.float64)
    V = np.asarray(value, np.float64)
    d = np.asarray(done, np.int64)
    v = np.asarray(valid, np.float64)
    E, T = r.shape
    lv = np.zeros(E) if last_value is None else np.asarray(last_value, np.float64)
    B = np.zeros((E, T)) if boot_value is None else np.asarray(boot_value, np.float64)
    adv = np.zeros((E, T))
    A_next = np.zeros(E)
    for t in range(T - 1, -1, -1):
        v_next = v[:, t + 1] if t + 1 < T else np.ones(E)
        V_next = V[:, t + 1] if t + 1 < T else lv
        nt = v[:, t] * (d[:, t] == 0) * v_next
        tr = (d[:, t] == 2).astype(np.float64)
        delta = v[:, t] * (r[:, t] + gamma * (nt * V_next + tr * B[:, t]) - V[:, t])
        A = delta + gamma * lam * nt * A_next
        adv[:, t] = A
        A_next = A
    ret = np.where(v > 0, adv + V, 0.0)
    return adv, ret


def whiten_stats(adv, valid):
    """(n, sum A, sum A^2) over valid steps — the quantities allreduced across ranks."""
    m = np.asarray(valid, bool)
    a = np.asarray(adv, np.float64)[m]
    return float(m.sum()), float(a.sum()), float((a * a).sum())


def whiten(adv, valid, eps: float = 1e-8, stats=None):
    """Reading R9: mu = sum vA / sum v; sigma = sqrt(sum v (A - mu)^2 / (sum v - 1));
    A_hat = (A - mu) / (sigma + eps) on valid steps, 0 elsewhere. `stats` = global
    (n, sum A, sum A^2) when the buffer is one shard of several."""
    m = np.asarray(valid, bool)
    a = np.asarray(adv, np.float64)
    if stats is None:
        n = m.sum()
        mu = a[m].sum() / n if n > 0 else 0.0
        var = ((a[m] - mu) ** 2).sum() / (n - 1) if n > 1 else 0.0
    else:
        n, s1, s2 = stats
        mu = s1 / n if n > 0 else 0.0
        var = (s2 - n * mu * mu) / (n - 1) if n > 1 else 0.0
        var = max(var, 0.0)
    sigma = np.sqrt(var)
    return np.where(m, (a - mu) / (sigma + eps), 0.0)


def episode_return(reward, valid):
    """R_e = sum_t valid * r_t (undiscounted outcome return)."""
    return (np.asarray(reward, np.float64) * np.asarray(valid, np.float64)).sum(axis=1)


def grpo(R, group_of_env, eps: float = 1e-6, unbiased: bool = True):
    """Per group g (members in ascending env id):
         mu_g = mean R;  sigma_g = sqrt(sum (R - mu_g)^2 / (n_g - 1))   [unbiased, R10]
                         sigma_g = sqrt(sum (R - mu_g)^2 / n_g)         [population flag]
         A_e  = (R_e - mu_g) / (sigma_g + eps);   n_g == 1 => A_e = 0.
    Returns A float64 [E]."""
    R = np.asarray(R, np.float64)
    g = np.asarray(group_of_env)
    A = np.zeros_like(R)
    for gid in np.unique(g):
        idx = np.nonzero(g == gid)[0]
        n = len(idx)
        if n < 2:
            A[idx] = 0.0
            continue
        mu = R[idx].sum() / n
        ss = ((R[idx] - mu) ** 2).sum()
        sigma = np.sqrt(ss / (n - 1 if unbiased else n))
        A[idx] = (R[idx] - mu) / (sigma + eps)
    return A


def grpo_step_adv(A_env, valid):
    """Broadcast A_e to every valid step of env e; 0 on unfilled slots."""
    v = np.asarray(valid, bool)
    return np.where(v, np.asarray(A_env, np.float64)[:, None], 0.0)


def step_counts(valid, version, tokens, cur_version: int, max_staleness: int):
    """Counts over decision steps (pre-loss bookkeeping, SURVEY §8(b) stats slots 0,3,4,5):
         n_valid  = #valid steps
         n_tok    = #tokens with target >= 0 on valid steps with 0 <= lag <= eta
         n_stale  = #valid steps with lag > eta
         n_bad    = #valid steps with lag < 0
         n_loss_steps = #valid steps with 0 <= lag <= eta and >= 1 token with target >= 0
                    (the chunk-ratio normaliser N_steps, reading R21)
    lag = cur_version - version (rollout runs on pre-update weights => lag <= 1)."""
    v = np.asarray(valid, bool)
    lag = cur_version - np.asarray(version, np.int64)
    ok = v & (lag >= 0) & (lag <= max_staleness)
    tok_ok = (np.asarray(tokens) >= 0).sum(axis=2)
    return dict(n_valid=int(v.sum()), n_tok=int((tok_ok * ok).sum()),
                n_stale=int((v & (lag > max_staleness)).sum()),
                n_bad=int((v & (lag < 0)).sum()),
                n_loss_steps=int((ok & (tok_ok > 0)).sum()))
