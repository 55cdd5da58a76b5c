"""GPU parity for NEXT-4 — the flow/diffusion chunk log-likelihood (chain of K Gaussian
denoising transitions, reading R25) through rlvla_flow_logprob against oracle/flow.py and the
PPO oracle: forward, fused PPO (one ratio per decision step) with its backward to mu and
ln sigma, and the external backward; f32 and bf16 means, sigma schedule and learned ln sigma,
rows inside and beyond the 512-element register cache."""
import numpy as np
import pytest
import torch

from oracle import flow as F
from oracle import ppo as O_ppo
from tests import harness as H

pytestmark = pytest.mark.gpu
SIG_K = np.array([0.8, 0.5, 0.3, 0.1], np.float32)


def _P():
    import paper_2602_05765_b200 as P
    return P


def _case(R, K, D, dtype, learned, seed=0):
    rng = np.random.default_rng(seed)
    mu = torch.from_numpy(rng.normal(size=(R, K, D)).astype(np.float32)).to(dtype)
    mu64 = mu.double().numpy()                      # what the kernel reads
    ls = rng.normal(-1.2, 0.5, size=(R, K, D)).astype(np.float32) if learned else None
    s = np.exp(ls.astype(np.float64)) if learned else SIG_K[:K].astype(np.float64)[None, :, None]
    x = (mu64 + s * rng.normal(size=(R, K, D))).astype(np.float32)
    if R > 10:
        x[3] = np.float32(np.nan)   # a non-finite row: counted and masked
    return mu, mu64, x, ls


def _err_scale(mu64, x, ls, K):
    """fp32 error scale of logp: the magnitudes of its terms (0.5 z^2, |ln sigma|, ln 2pi/2)."""
    s = np.exp(ls.astype(np.float64)) if ls is not None else SIG_K[:K].astype(np.float64)[None, :, None]
    z = (x.astype(np.float64) - mu64) / s
    lsig = np.log(np.broadcast_to(s, z.shape))
    return np.nan_to_num((0.5 * z * z + np.abs(lsig) + 1.0).sum(axis=(1, 2)), nan=1.0)


SHAPES = [(300, 4, 70), (257, 4, 35), (50, 3, 200), (33, 1, 7), (3, 4, 70)]  # (3, ...): a lone partial tile


@pytest.mark.parametrize("R,K,D", SHAPES)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("learned", [False, True])
def test_forward(R, K, D, dtype, learned):
    P = _P()
    mu, mu64, x, ls = _case(R, K, D, dtype, learned)
    ch = P.GaussChain(mu.cuda(), torch.from_numpy(x).cuda(), torch.from_numpy(SIG_K[:K]).cuda(),
                      None if ls is None else torch.from_numpy(ls).cuda())
    logp = torch.empty(R, device="cuda")
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    P.rlvla_flow_logprob(ch, logp=logp, stats=st, ws=P.workspace(1))
    o = F.chain_logprob(mu64, x, sigma_k=SIG_K[:K], log_std=ls)
    es = _err_scale(mu64, x, ls, K)
    got = logp.cpu().numpy()
    fin = np.isfinite(o["logp"])
    assert (~fin).sum() == (1 if R > 10 else 0) and not np.isfinite(got[~fin]).any()
    # fp32 lane partials of <= 16 terms: |error| <= ~16 eps32 x (sum of the terms' magnitudes)
    H.assert_close_rel(got[fin], o["logp"][fin], 2e-7, es[fin], "logp")
    s = st.cpu().numpy()
    assert s[11] == fin.sum() and s[13] == (~fin).sum()
    assert abs(s[9] - o["entropy"][fin].sum()) <= 1e-5 * np.abs(o["entropy"][fin]).sum()
    assert abs(s[14] - o["logp"][fin].sum()) <= 1e-5 * es[fin].sum()


VARS = [dict(), dict(dual_clip=3.0, kl_coef=0.1), dict(ent_coef=0.01)]


@pytest.mark.parametrize("R,K,D", SHAPES[:3] + SHAPES[4:])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("learned", [False, True])
@pytest.mark.parametrize("var", VARS)
def test_fused_ppo(R, K, D, dtype, learned, var):
    _run_fused(R, K, D, dtype, learned, var)


@pytest.mark.parametrize("R,K,D", SHAPES[:2])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("learned", [False, True])
@pytest.mark.parametrize("which", ["data", "meta"])
def test_fused_ppo_unaligned(R, K, D, dtype, learned, which):
    """Arrays 8 bytes off a 16-byte boundary. data: the paper's shapes then skip the TMA-staged
    kernel (bulk copies need 16-byte aligned tiles) and run the direct one (bf16 4-wide, f32
    scalar); meta: the staged kernel loads the PPO inputs from global memory instead."""
    _run_fused(R, K, D, dtype, learned, dict(kl_coef=0.1) if which == "meta" else {},
               offset_bytes=8, offset_what=which)


def _offset(t, nbytes):
    """A copy of t whose data pointer sits `nbytes` past a 256-byte aligned allocation."""
    k = nbytes // t.element_size()
    buf = torch.empty(t.numel() + k, dtype=t.dtype, device=t.device)
    v = buf[k:].view(t.shape)
    v.copy_(t)
    assert v.data_ptr() % 16 == nbytes % 16
    return v


def _run_fused(R, K, D, dtype, learned, var, offset_bytes=0, offset_what="data"):
    P = _P()
    mu, mu64, x, ls = _case(R, K, D, dtype, learned, seed=1)
    o = F.chain_logprob(mu64, x, sigma_k=SIG_K[:K], log_std=ls)
    rng = np.random.default_rng(2)
    lp = np.nan_to_num(o["logp"])
    lb = (lp - rng.choice([-1.0, -0.05, 0.02, 0.1, 0.9], R) - rng.normal(0, 0.01, R)).astype(np.float32)
    lref = (lp + rng.normal(0, 0.3, R)).astype(np.float32)
    adv = rng.normal(size=R).astype(np.float32)
    ver = (100 - rng.choice([0, 1, 2], size=R, p=[0.6, 0.3, 0.1])).astype(np.int32)
    key = np.where(rng.random(R) < 0.95, 5, 0).astype(np.int64)
    N = float(R)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    cm = cu  # the PPO inputs
    if offset_bytes and offset_what == "meta":
        cm = lambda a: _offset(cu(a), offset_bytes)  # noqa: E731
    g = torch.empty(R, device="cuda")
    lt = torch.empty(R, device="cuda")
    fa = P.ppo_args(logp_behav=cm(lb), adv=cm(adv), version=cm(ver), slot_key=cm(key), a_tok=1,
                    cur_version=100, tok_denominator=N, out_grad_logp=g, out_loss_tok=lt,
                    logp_ref=cm(lref) if var.get("kl_coef") else None, **var)
    mu_d, x_d, ls_d = mu.cuda(), cu(x), None if ls is None else cu(ls)
    dmu = torch.empty_like(mu_d)
    dls = torch.empty(R, K, D, device="cuda") if learned else None
    if offset_bytes and offset_what == "data":
        mu_d, x_d, dmu = _offset(mu_d, offset_bytes), _offset(x_d, offset_bytes), _offset(dmu, offset_bytes)
        ls_d = None if ls_d is None else _offset(ls_d, offset_bytes)
        dls = None if dls is None else _offset(dls, offset_bytes)
    ch = P.GaussChain(mu_d, x_d, cu(SIG_K[:K]), ls_d)
    logp = torch.empty(R, device="cuda")
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    P.rlvla_flow_logprob(ch, logp=logp, fused=fa, dmu=dmu, dlog_std=dls, stats=st, ws=P.workspace(1))
    # oracle: PPO over the chain log-probs, one token per decision step
    base = (key != 0) & np.isfinite(o["logp"])
    p = O_ppo.ppo_loss(lp, lb, adv, base, 100 - ver.astype(np.int64), n_tok=N,
                       dual_clip=var.get("dual_clip", 0.0), logp_ref=lref if var.get("kl_coef") else None,
                       kl_coef=var.get("kl_coef", 0.0))
    nt = p["near_tie"]
    es = _err_scale(mu64, x, ls, K)
    dlogp = 2e-7 * es                                   # logp tolerance (test_forward)
    sens = np.abs(adv) * np.nan_to_num(p["ratio"])
    if var.get("kl_coef"):
        sens = sens + var["kl_coef"] * np.exp(np.minimum(lref - lp, 50.0))
    gtol = np.maximum(sens * dlogp / N, 1e-12)
    ok = ~nt
    H.assert_close_rel(g.cpu().numpy()[ok], p["grad"][ok], 1e-5, (gtol / 1e-5)[ok], "grad_logp")
    c = np.where(p["mask"], var.get("ent_coef", 0.0) / N, 0.0)
    gr = F.chain_grads(mu64, x, p["grad"], sigma_k=SIG_K[:K], log_std=ls)
    s_ = np.exp(ls.astype(np.float64)) if learned else SIG_K[:K].astype(np.float64)[None, :, None]
    z = np.nan_to_num((x - mu64) / s_)
    # dmu = g z / sigma carries g's tolerance; rows near a clip bound are excluded
    dmu_ref = np.where(p["mask"][:, None, None], gr["dmu"], 0.0)
    fl = (gtol[:, None, None] + 1e-5 * np.abs(p["grad"])[:, None, None]) * np.abs(z / s_) / 1e-5
    got = dmu.float().cpu().numpy()
    if dtype == torch.bfloat16:
        bits = dmu.view(torch.int16).cpu().numpy().astype(np.int32) & 0xFFFF
        H.assert_bf16_ulp(bits[ok], dmu_ref[ok], 1, abs_floor=1e-5 * fl[ok])
    else:
        H.assert_close_rel(got[ok], dmu_ref[ok], 1e-5, fl[ok], "dmu")
    if learned:
        dls_ref = np.where(p["mask"][:, None, None], gr["dlog_std"] - c[:, None, None], 0.0)
        fl2 = (gtol[:, None, None] + 1e-5 * np.abs(p["grad"])[:, None, None]) * (z * z + 1) / 1e-5 + c[:, None, None]
        H.assert_close_rel(dls.cpu().numpy()[ok], dls_ref[ok], 1e-5, fl2[ok], "dlog_std")
    s = st.cpu().numpy()
    rs = p["stats"]
    ent = float(np.where(p["mask"], o["entropy"], 0.0).sum())
    loss = rs["loss"] - var.get("ent_coef", 0.0) * ent / N
    # the loss is a mean of mixed-sign terms: its error is the propagated logp error
    tol_loss = float((sens * dlogp)[base].sum()) / N + 1e-5 * max(1e-3, abs(loss))
    assert abs(s[6] - loss) <= tol_loss, (s[6], loss, tol_loss)
    assert s[11] == rs["n_loss_tok"] and s[12] == rs["n_stale_tok"]
    assert abs(s[9] - ent) <= 1e-5 * max(1.0, abs(ent))
    assert abs(s[16] - rs["n_dual_clipped"]) <= nt.sum()


def test_external_backward():
    P = _P()
    R, K, D = 120, 4, 70
    mu, mu64, x, ls = _case(R, K, D, torch.float32, True, seed=4)
    g = np.random.default_rng(6).normal(size=R).astype(np.float32)
    ch = P.GaussChain(mu.cuda(), torch.from_numpy(x).cuda(), None, torch.from_numpy(ls).cuda())
    dmu = torch.empty(R, K, D, device="cuda")
    dls = torch.empty(R, K, D, device="cuda")
    P.rlvla_flow_logprob(ch, grad_logp=torch.from_numpy(g).cuda(), dmu=dmu, dlog_std=dls)
    gr = F.chain_grads(mu64, x, g, log_std=ls)
    fin = np.isfinite(gr["dmu"]).all(axis=(1, 2))
    H.assert_close_rel(dmu.cpu().numpy()[fin], gr["dmu"][fin], 1e-5, 1e-30, "dmu")
    H.assert_close_rel(dls.cpu().numpy()[fin], gr["dlog_std"][fin], 1e-5, np.abs(g[fin])[:, None, None], "dlog_std")


def test_rerun_bit_identical():
    """Fixed-order reductions: two identical fused calls give identical bits."""
    P = _P()
    R, K, D = 500, 4, 70
    mu, mu64, x, ls = _case(R, K, D, torch.bfloat16, False, seed=9)
    rng = np.random.default_rng(3)
    lb = (np.nan_to_num(F.chain_logprob(mu64, x, sigma_k=SIG_K)["logp"]) - rng.normal(0, 0.05, R)).astype(np.float32)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    outs = []
    for _ in range(2):
        g = torch.empty(R, device="cuda")
        fa = P.ppo_args(logp_behav=cu(lb), adv=cu(rng.normal(size=R).astype(np.float32) * 0 + 0.7),
                        version=cu(np.full(R, 100, np.int32)), slot_key=cu(np.ones(R, np.int64)),
                        a_tok=1, cur_version=100, tok_denominator=float(R), out_grad_logp=g)
        ch = P.GaussChain(mu.cuda(), cu(x), cu(SIG_K))
        logp = torch.empty(R, device="cuda")
        dmu = torch.empty_like(ch.mu)
        st = torch.zeros(24, dtype=torch.float64, device="cuda")
        P.rlvla_flow_logprob(ch, logp=logp, fused=fa, dmu=dmu, stats=st, ws=P.workspace(1))
        outs.append((logp.view(torch.int32).cpu(), g.view(torch.int32).cpu(), dmu.view(torch.int16).cpu(),
                     st.view(torch.int64).cpu()))
    for a_, b_ in zip(*outs):
        assert torch.equal(a_, b_)  # bitwise (the crafted non-finite step included)
