"""S4 oracle: PPO / decoupled clipped surrogate with a staleness bound (TEST INFRASTRUCTURE ONLY).

Paper: rollout continues on the pre-update policy until the actor finishes the update
(§3.1) => every trajectory carries a behaviour version with lag <= 1; the paper's
asynchronous design cites AReaL's decoupled objective (`fu2025areal`, §1) but
never writes a loss. Definitions written out per token row r of decision
step (e, t) (readings R11-R14 in DESIGN.md §2):

  1. lag = cur_version - version[e, t]
  2. m_r = valid * [target_ok] * [0 <= lag <= eta]
  3. standard:  rho = exp(logp - logp_behav),  w = 1
     decoupled: w = min(exp(logp_prox - logp_behav), cap) (no gradient),
                rho = exp(logp - logp_prox)                         (Fu et al. 2025)
  4. L_r = -w * min(rho * A, clip(rho, 1 - eps_lo, 1 + eps_hi) * A)  (Schulman et al. 2017)
  5. Loss = sum_r m_r L_r / N_tok
  6. dLoss/dlogp_r = -m_r w A rho [active] / N_tok,
     active <=> not ((A > 0 and rho > 1 + eps_hi) or (A < 0 and rho < 1 - eps_lo))
     (ties at the bound are active: autograd of min + clamp, reading R11)
  7. stats: sum m (rho - 1 - ln rho) (k3 KL), sum m rho, #clipped
"""
from __future__ import annotations

import numpy as np

NEAR_TIE_REL = 1e-5


def ppo_loss(logp, logp_behav, adv_tok, mask_base, lag_tok, *, eps_low=0.2, eps_high=0.2,
             max_staleness=1, n_tok=None, logp_prox=None, is_cap=0.0):
    """Per-token PPO/decoupled loss in float64.

    logp, logp_behav, logp_prox, adv_tok: [R]; mask_base: bool [R] = valid step and
    usable target (finite logp); lag_tok: int [R].
    Returns dict(loss_tok, grad, mask, stale, bad_lag, clipped, near_tie, ratio, w,
    stats) where loss_tok is the unnormalised L_r (0 where masked) and grad is
    dLoss/dlogp including the 1/N_tok factor.
    """
    logp = np.asarray(logp, np.float64)
    lb = np.asarray(logp_behav, np.float64)
    A = np.asarray(adv_tok, np.float64)
    lag = np.asarray(lag_tok, np.int64)
    base = np.asarray(mask_base, bool)
    stale = base & (lag > max_staleness)
    bad_lag = base & (lag < 0)
    m = base & (lag >= 0) & (lag <= max_staleness)
    if n_tok is None:
        n_tok = float(m.sum())
    with np.errstate(over="ignore", invalid="ignore"):
        if logp_prox is None:
            w = np.ones_like(logp)
            lr = logp - lb
        else:
            lp = np.asarray(logp_prox, np.float64)
            w = np.exp(lp - lb)
            if is_cap and is_cap > 0:
                w = np.minimum(w, is_cap)
            lr = logp - lp
        rho = np.exp(lr)
        lo, hi = 1.0 - eps_low, 1.0 + eps_high
        surr1 = rho * A
        surr2 = np.clip(rho, lo, hi) * A
        L = -w * np.minimum(surr1, surr2)
        clipped = ((A > 0) & (rho > hi)) | ((A < 0) & (rho < lo))
        grad = np.where(clipped, 0.0, -w * A * rho) / n_tok
        near_tie = (np.abs(rho / hi - 1.0) <= NEAR_TIE_REL) | (np.abs(rho / lo - 1.0) <= NEAR_TIE_REL)
    L = np.where(m, L, 0.0)
    grad = np.where(m, grad, 0.0)
    clipped = clipped & m
    k3 = np.where(m, rho - 1.0 - lr, 0.0)
    stats = dict(loss=L.sum() / n_tok if n_tok > 0 else 0.0,
                 n_clipped=float(clipped.sum()), kl_k3_sum=float(k3.sum()),
                 ratio_sum=float(np.where(m, rho, 0.0).sum()),
                 n_loss_tok=float(m.sum()), n_stale_tok=float(stale.sum()),
                 n_bad_lag=float(bad_lag.sum()),
                 logp_sum=float(np.where(m, logp, 0.0).sum()), denom=float(n_tok))
    return dict(loss_tok=L, grad=grad, mask=m, stale=stale, bad_lag=bad_lag, clipped=clipped,
                near_tie=near_tie & m, ratio=rho, w=w, stats=stats)
