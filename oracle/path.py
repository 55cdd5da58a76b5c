"""S1..S4 composed: one rollout-to-loss pass on the CPU (TEST INFRASTRUCTURE ONLY).

Order of the hot path as SURVEY §3.2 lays it out and the paper places it (§3.3:
"Whenever the number of samples accumulated in the trajectory buffer reaches the size of
a single micro-batch, the actor initiates a forward and backward computation"):
    scatter arrival chunks -> advantages -> action-token log-probs -> PPO loss -> dlogits.
Also Eq. (2), the paper's throughput unit (§4.1).
"""
from __future__ import annotations

import numpy as np

from . import advantages as adv_mod
from . import logprob as lp_mod
from . import ppo as ppo_mod
from . import scatter as sc_mod


def throughput_eq2(n_re: float, n_env: float, n_es: float, t_s: float) -> float:
    """Eq. (2): Throughput = N_re * N_env * N_es / T_s. T_s is the run's wall
    time (the tables reproduce with T_s = 'Time (s)')."""
    return n_re * n_env * n_es / t_s


def advantages(buf, last_value, *, mode, gamma=0.99, lam=0.95, whiten=False,
               whiten_eps=1e-8, group_of_env=None, grpo_eps=1e-6, std_unbiased=True,
               cur_version=0, max_staleness=1, R_global=None, env_offset=0,
               whiten_global=None):
    """Advantages on one buffer (shard). For GRPO across shards pass R_global (all envs'
    returns) and env_offset; for global whitening pass whiten_global=(n, s1, s2)."""
    valid = buf["slot_key"] != 0
    counts = adv_mod.step_counts(valid, buf["version"], buf["tokens"], cur_version,
                                 max_staleness)
    if mode == "gae":
        a, ret = adv_mod.gae(buf["reward"], buf["value"], buf["done"], valid, last_value,
                             gamma, lam)
        raw = a
        st = adv_mod.whiten_stats(a, valid)
        if whiten:
            a = adv_mod.whiten(a, valid, whiten_eps, stats=whiten_global or st)
    else:
        R = adv_mod.episode_return(buf["reward"], valid)
        E = R.shape[0]
        Rg = R if R_global is None else np.asarray(R_global, np.float64)
        Ag = adv_mod.grpo(Rg, group_of_env, grpo_eps, std_unbiased)
        A_env = Ag[env_offset:env_offset + E]
        a = adv_mod.grpo_step_adv(A_env, valid)
        ret = adv_mod.grpo_step_adv(R, valid)
        raw = a
        st = adv_mod.whiten_stats(a, valid)
    return dict(adv=a, ret=ret, raw=raw, counts=counts, whiten_stats=st, valid=valid)


def token_view(buf, adv, a_tok, cur_version):
    """Per-token (row) views of per-step arrays: row r <-> step r // A."""
    valid = (buf["slot_key"] != 0).reshape(-1)
    lag = (cur_version - buf["version"].astype(np.int64)).reshape(-1)
    return dict(valid=np.repeat(valid, a_tok), lag=np.repeat(lag, a_tok),
                adv=np.repeat(np.asarray(adv, np.float64).reshape(-1), a_tok),
                target=buf["tokens"].reshape(-1), logp_behav=buf["logp_behav"].reshape(-1))


def loss_and_grad(logits, tv, *, eps_low=0.2, eps_high=0.2, max_staleness=1, n_tok=None,
                  logp_prox=None, is_cap=0.0, rows=None, dual_clip=0.0, logp_ref=None,
                  kl_coef=0.0, ent_coef=0.0):
    """S3 + S4 on the given logit rows. `rows` = indices into the token view (defaults to
    all); `logits` holds exactly those rows."""
    rows = np.arange(len(tv["target"])) if rows is None else np.asarray(rows)
    tgt = tv["target"][rows]
    f = lp_mod.log_softmax_gather(logits, tgt)
    valid = tv["valid"][rows]
    base = valid & (f["status"] == 0)
    lpp = None if logp_prox is None else np.asarray(logp_prox)[rows]
    lpr = None if logp_ref is None else np.asarray(logp_ref)[rows]
    p = ppo_mod.ppo_loss(f["logp"], tv["logp_behav"][rows], tv["adv"][rows], base,
                         tv["lag"][rows], eps_low=eps_low, eps_high=eps_high,
                         max_staleness=max_staleness, n_tok=n_tok, logp_prox=lpp,
                         is_cap=is_cap, dual_clip=dual_clip, logp_ref=lpr, kl_coef=kl_coef)
    dx = lp_mod.log_softmax_grad(logits, tgt, f["lse"], p["grad"])
    N = p["stats"]["denom"]
    if ent_coef:
        coef = np.where(p["mask"], ent_coef / N if N > 0 else 0.0, 0.0)
        dx = dx + lp_mod.entropy_bonus_grad(logits, f["lse"], f["entropy"], coef)
    bad = valid & ((f["status"] == 2) | (f["status"] == 3))
    n_bad_tok = float(bad.sum() + p["bad_lag"].sum())
    ent = float(np.where(p["mask"], f["entropy"], 0.0).sum())
    stats = dict(p["stats"])
    stats.update(entropy_sum=ent, n_bad_tok=n_bad_tok)
    if ent_coef and N > 0:
        stats["loss"] -= ent_coef * ent / N
    return dict(fwd=f, ppo=p, dx=dx, stats=stats)


def rollout_to_loss(cfg_params: dict, records_chunks, logits, *, seq_base=1):
    """Whole path on one shard: scatter every arrival chunk, advantages, S3+S4.
    cfg_params: n_env, t_steps, a_tok, cur_version, max_staleness, mode, group_of_env,
    last_value, whiten, gamma, lam."""
    c = cfg_params
    buf = sc_mod.new_buffer(c["n_env"], c["t_steps"], c["a_tok"])
    counters = np.zeros(4, np.int64)
    seq = seq_base
    for ch in records_chunks:
        counters += sc_mod.scatter_steps(buf, ch, c["cur_version"], seq)
        seq += len(ch["env_id"])
    adv = advantages(buf, c.get("last_value"), mode=c["mode"], gamma=c.get("gamma", 0.99),
                     lam=c.get("lam", 0.95), whiten=c.get("whiten", False),
                     group_of_env=c.get("group_of_env"), cur_version=c["cur_version"],
                     max_staleness=c["max_staleness"])
    tv = token_view(buf, adv["adv"], c["a_tok"], c["cur_version"])
    out = loss_and_grad(logits, tv, max_staleness=c["max_staleness"],
                        n_tok=float(adv["counts"]["n_tok"]), rows=c.get("rows"))
    return dict(buf=buf, counters=counters, adv=adv, tv=tv, **out)
