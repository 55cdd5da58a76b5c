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
             max_staleness=1, n_tok=None, logp_prox=None, is_cap=0.0, dual_clip=0.0,
             logp_ref=None, kl_coef=0.0):
    """Per-token PPO/decoupled loss in float64.

    logp, logp_behav, logp_prox, logp_ref, adv_tok: [R]; mask_base: bool [R] = valid step
    and usable target (finite logp); lag_tok: int [R].
    Optional terms (NEXT-2; the paper is silent, readings R19-R20):
      dual_clip c > 1 (Ye et al. 2020): for A < 0 the objective is max(J, c A), so tokens
        with c A > J carry no gradient ("dual-clipped");
      kl_coef b with logp_ref (k3 estimator, Schulman 2020; as in GRPO): L += b k3,
        k3 = e^{lr} - lr - 1, lr = logp_ref - logp, dk3/dlogp = 1 - e^{lr}.
    Returns dict(loss_tok, grad, mask, stale, bad_lag, clipped, dual, near_tie, ratio, w,
    stats): loss_tok is the unnormalised per-token loss (0 where masked), grad is dLoss/dlogp
    including the 1/N_tok factor.
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
    inv_n = 1.0 / n_tok if n_tok > 0 else 0.0
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
        J = np.minimum(surr1, surr2)
        clipped = ((A > 0) & (rho > hi)) | ((A < 0) & (rho < lo))
        dual = np.zeros_like(clipped)
        if dual_clip and dual_clip > 1.0:
            dual = (A < 0) & (dual_clip * A > J)
            J = np.where(dual, dual_clip * A, J)
        L = -w * J
        gpg = np.where(clipped | dual, 0.0, -w * A * rho)
        near_tie = (np.abs(rho / hi - 1.0) <= NEAR_TIE_REL) | (np.abs(rho / lo - 1.0) <= NEAR_TIE_REL)
        if dual_clip and dual_clip > 1.0:
            near_tie = near_tie | (np.abs(rho / dual_clip - 1.0) <= NEAR_TIE_REL)
        k3ref = np.zeros_like(logp)
        gkl = np.zeros_like(logp)
        if logp_ref is not None and kl_coef:
            lref = np.asarray(logp_ref, np.float64) - logp
            k3ref = np.exp(lref) - lref - 1.0
            gkl = kl_coef * (1.0 - np.exp(lref))
    Lpg = np.where(m, L, 0.0)
    Ltot = np.where(m, L + kl_coef * k3ref, 0.0)
    grad = np.where(m, (gpg + gkl) * inv_n, 0.0)
    clipped = clipped & m
    dual = dual & m
    k3 = np.where(m, rho - 1.0 - lr, 0.0)
    stats = dict(loss=Ltot.sum() * inv_n, pg_loss=Lpg.sum() * inv_n,
                 n_clipped=float(clipped.sum()), n_dual_clipped=float(dual.sum()),
                 kl_k3_sum=float(k3.sum()), kl_ref_sum=float(np.where(m, k3ref, 0.0).sum()),
                 ratio_sum=float(np.where(m, rho, 0.0).sum()),
                 n_loss_tok=float(m.sum()), n_stale_tok=float(stale.sum()),
                 n_bad_lag=float(bad_lag.sum()),
                 logp_sum=float(np.where(m, logp, 0.0).sum()), denom=float(n_tok))
    return dict(loss_tok=Ltot, grad=grad, mask=m, stale=stale, bad_lag=bad_lag, clipped=clipped,
                dual=dual, near_tie=near_tie & m, ratio=rho, w=w, stats=stats)


def ppo_loss_chunk(logp, logp_behav, adv_step, mask_tok, step_of_tok, n_steps_total, *,
                   eps_low=0.2, eps_high=0.2, n_den=None, logp_prox=None, is_cap=0.0,
                   dual_clip=0.0):
    """Chunk-level ratio (NEXT-2, reading R21): one ratio per decision step = the action
    chunk's likelihood ratio rho_s = exp(sum_{a in s, m_a} (logp_a - logp_behav_a)) (an
    OpenVLA-OFT action chunk is one inference); L_s = -min(rho_s A_s, clip(rho_s) A_s)
    over steps with >= 1 masked token; Loss = sum_s L_s / N_steps; every token of step s gets
    dLoss/dlogp = -A_s rho_s [active_s] / N_steps.
    Decoupled (R12 at step level): w_s = min(exp(sum m (logp_prox - logp_behav)), cap)
    (detached), rho_s = exp(sum m (logp - logp_prox)), L_s = -w_s J_s. Dual clip (R19 at step
    level): for A_s < 0, J_s = max(J_s, c A_s); steps with c A_s > J_s carry no gradient."""
    logp = np.asarray(logp, np.float64)
    lb = np.asarray(logp_behav, np.float64)
    m = np.asarray(mask_tok, bool)
    st = np.asarray(step_of_tok, np.int64)
    A = np.asarray(adv_step, np.float64)
    lpp = None if logp_prox is None else np.asarray(logp_prox, np.float64)
    lr = np.zeros(n_steps_total)
    lw = np.zeros(n_steps_total)
    cnt = np.zeros(n_steps_total)
    for r in range(len(logp)):
        if m[r]:
            if lpp is None:
                lr[st[r]] += logp[r] - lb[r]
            else:
                lr[st[r]] += logp[r] - lpp[r]
                lw[st[r]] += lpp[r] - lb[r]
            cnt[st[r]] += 1
    ms = cnt > 0
    N = float(ms.sum()) if n_den is None else n_den
    inv = 1.0 / N if N > 0 else 0.0
    rho = np.exp(lr)
    w = np.ones(n_steps_total) if lpp is None else np.exp(lw)
    if lpp is not None and is_cap and is_cap > 0:
        w = np.minimum(w, is_cap)
    lo, hi = 1.0 - eps_low, 1.0 + eps_high
    J = np.minimum(rho * A, np.clip(rho, lo, hi) * A)
    clipped = ((A > 0) & (rho > hi)) | ((A < 0) & (rho < lo))
    dual = np.zeros(n_steps_total, bool)
    if dual_clip and dual_clip > 1.0:
        dual = (A < 0) & (dual_clip * A > J)
        J = np.where(dual, dual_clip * A, J)
    g_step = np.where(ms & ~clipped & ~dual, -w * A * rho * inv, 0.0)
    grad = np.where(m, g_step[st], 0.0)
    L = np.where(ms, -w * J, 0.0)
    near = (np.abs(rho / hi - 1.0) <= NEAR_TIE_REL) | (np.abs(rho / lo - 1.0) <= NEAR_TIE_REL)
    if dual_clip and dual_clip > 1.0:
        near = near | (np.abs(rho / dual_clip - 1.0) <= NEAR_TIE_REL)
    return dict(grad=grad, loss_step=L, rho_step=rho, w_step=w, mask_step=ms,
                clipped=clipped & ms, dual=dual & ms, near_tie_step=near & ms,
                stats=dict(loss=L.sum() * inv, n_clipped=float((clipped & ms).sum()),
                           n_dual_clipped=float((dual & ms).sum()),
                           n_steps=float(ms.sum()), denom=N))


def value_loss(v_new, v_old, ret, mask, *, clip_eps=0.2, n_den=None):
    """Clipped value loss per decision step (PPO value head, NEXT-2; paper-silent, reading
    R22): L = 0.5 max((v - R)^2, (v_old + clip(v - v_old, -e, e) - R)^2); e <= 0 => plain
    0.5 (v - R)^2. Loss = sum m L / N; dLoss/dv from the larger branch; the clipped branch
    counts only where the clip moved v (|v - v_old| > e), and there d clip/dv = 0."""
    v = np.asarray(v_new, np.float64)
    vo = np.asarray(v_old, np.float64)
    R = np.asarray(ret, np.float64)
    m = np.asarray(mask, bool)
    N = float(m.sum()) if n_den is None else n_den
    inv = 1.0 / N if N > 0 else 0.0
    u = (v - R) ** 2
    if clip_eps and clip_eps > 0:
        d = v - vo
        vc = vo + np.clip(d, -clip_eps, clip_eps)
        c = (vc - R) ** 2
        # the clipped branch counts only where the clip moved v (|d| > e); inside the
        # interval v_clip == v and both branches agree (reading R22)
        use_c = (np.abs(d) > clip_eps) & (c > u)
        g = np.where(use_c, 0.0, v - R)
        L = 0.5 * np.maximum(u, c)
    else:
        use_c = np.zeros_like(m)
        g = v - R
        L = 0.5 * u
    return dict(loss_step=np.where(m, L, 0.0), grad=np.where(m, g * inv, 0.0),
                clipped=use_c & m,
                stats=dict(loss=np.where(m, L, 0.0).sum() * inv, n_clipped=float((use_c & m).sum()),
                           n_steps=float(m.sum()), denom=N))
