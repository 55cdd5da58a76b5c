"""S3 oracle: log-softmax + gather, forward and backward (TEST INFRASTRUCTURE ONLY).

Paper: OpenVLA "discretizes the action space into tokens to generate actions
autoregressively" (§2); OpenVLA-OFT predicts a chunk of actions (§4.1;
chunk 8 in Table 2). The action-token log-probability is the textbook
log-softmax of the token logits evaluated at the sampled token; the paper does not
write it out. Two-pass definition, float64:
    m   = max_j x_j
    S   = sum_j exp(x_j - m)
    lse = m + ln S
    logp = x_a - lse
    H   = lse - sum_j p_j x_j          (p_j = exp(x_j - lse); p_j x_j := 0 where p_j = 0)
    dx_j = g * (1[j = a] - p_j)        (backward with upstream g = dL/dlogp)
           at j = a the factor 1 - p_a is evaluated as sum_{j != a} p_j (the same number;
           written this way because 1 - p_a cancels to 0 in float64 once p_a > 1 - 1e-16,
           e.g. a saturated row, DESIGN.md §2 reading R15b)
Readings: R3 (normalise over the V columns supplied), R4 (target -1 = ignore, other
out-of-range targets counted), R5 (-inf allowed in non-target columns; NaN/+inf or an
all -inf row give a non-finite result that is counted).
"""
from __future__ import annotations

import numpy as np


def log_softmax_gather(x, target):
    """x: [R, V] (any float dtype, decoded exactly to float64); target: int [R].
    Returns dict(logp, lse, entropy, status) with status 0 ok, 1 ignore (target -1),
    2 bad target, 3 non-finite. logp = 0 for ignore/bad rows."""
    x = np.asarray(x, np.float64)
    tgt = np.asarray(target, np.int64)
    R, V = x.shape
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        m = x.max(axis=1)
        S = np.exp(x - m[:, None]).sum(axis=1)
        lse = m + np.log(S)
        p = np.exp(x - lse[:, None])
        px = np.where(p > 0, p * x, 0.0)
        H = lse - px.sum(axis=1)
    status = np.zeros(R, np.int8)
    logp = np.zeros(R)
    for r in range(R):
        a = tgt[r]
        if a == -1:
            status[r] = 1
            continue
        if a < 0 or a >= V:
            status[r] = 2
            continue
        logp[r] = x[r, a] - lse[r]
        if not (np.isfinite(lse[r]) and np.isfinite(logp[r])):
            status[r] = 3
            logp[r] = np.nan if not np.isfinite(logp[r]) else logp[r]
    return dict(logp=logp, lse=lse, entropy=H, status=status)


def log_softmax_grad(x, target, lse, g):
    """dx[r, j] = g_r * (1[j = a_r] - exp(x[r, j] - lse_r)); rows with g_r == 0 are 0
    (masked rows carry no gradient even if their logits are non-finite)."""
    x = np.asarray(x, np.float64)
    tgt = np.asarray(target, np.int64)
    g = np.asarray(g, np.float64)
    R, V = x.shape
    with np.errstate(invalid="ignore", over="ignore"):
        p = np.exp(x - np.asarray(lse, np.float64)[:, None])
    dx = -g[:, None] * p
    ok = (tgt >= 0) & (tgt < V)
    for r in np.nonzero(ok)[0]:
        a = tgt[r]
        rest = p[r, :a].sum() + p[r, a + 1:].sum()       # = 1 - p_a
        dx[r, a] = g[r] * rest
    dx[g == 0] = 0.0
    return dx


def entropy_bonus_grad(x, lse, H, coef_r):
    """Gradient of -coef * H w.r.t. the logits (entropy bonus, NEXT-2, reading R20):
    dH/dx_j = -p_j (log p_j + H)  =>  d(-c H)/dx_j = c p_j (log p_j + H). coef_r: [R]
    (the per-row weight m_r beta / N_tok). -inf columns (p_j = 0) contribute 0."""
    x = np.asarray(x, np.float64)
    lse = np.asarray(lse, np.float64)
    with np.errstate(invalid="ignore", over="ignore"):
        logp_all = x - lse[:, None]
        p = np.exp(logp_all)
        t = np.where(p > 0, p * (logp_all + np.asarray(H, np.float64)[:, None]), 0.0)
    return np.asarray(coef_r, np.float64)[:, None] * t
