"""GPU parity for the NEXT-2 loss variants (paper-silent; readings R19-R23) against the oracle:
dual-clip, reference-KL (k3), entropy bonus (gradient through the logits) on all three
log-prob kernel paths; chunk-level ratio and token-level variants through rlvla_ppo_loss;
the clipped value loss; GAE with time-limit truncation."""
import numpy as np
import pytest
import torch

from oracle import advantages as O_adv
from oracle import logprob as O_lp
from oracle import path as O_path
from oracle import ppo as O_ppo
from tests import harness as H

pytestmark = pytest.mark.gpu


def _P():
    import paper_2602_05765_b200 as P
    return P


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _case(R, V, dtype, A, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = (torch.randn(R, V, generator=g) * 1.5)
    x[1] = -30.0
    x[1, 3] = 30.0                                   # saturated row (target 3)
    x[2, [1, 2, V // 2]] = float("-inf")             # -inf columns (target 0)
    x = x.to(dtype)
    rng = np.random.default_rng(seed)
    t = rng.integers(0, V, R).astype(np.int32)
    t[1], t[2], t[4] = 3, 0, -1
    x64 = x.double().numpy()
    f = O_lp.log_softmax_gather(x64, t)
    lp = np.nan_to_num(f["logp"])
    lr = rng.choice([-1.3, -0.4, -0.05, 0.03, 0.1, 0.4, 1.4], R) + rng.normal(0, 0.01, R)
    lb = (lp - lr).astype(np.float32)
    lref = (lp + rng.normal(0, 0.3, R)).astype(np.float32)
    S = R // A
    adv = rng.normal(size=S).astype(np.float32)
    ver = (100 - rng.choice([0, 1, 2], size=S, p=[0.6, 0.3, 0.1])).astype(np.int32)
    key = np.where(rng.random(S) < 0.95, 7, 0).astype(np.int64)
    return x, t, x64, f, lb, lref, adv, ver, key


VARIANTS = [dict(dual_clip=3.0), dict(kl_coef=0.05), dict(ent_coef=0.01),
            dict(dual_clip=2.5, kl_coef=0.1, ent_coef=0.02)]
SHAPES = [(280, 256, torch.float32), (280, 1000, torch.bfloat16), (140, 32000, torch.bfloat16),
          (56, 5003, torch.float32), (56, 8192, torch.float32)]


@pytest.mark.parametrize("R,V,dtype", SHAPES)
@pytest.mark.parametrize("var", VARIANTS)
def test_fused_variants(R, V, dtype, var):
    P = _P()
    A = 7
    x, t, x64, f, lb, lref, adv, ver, key = _case(R, V, dtype, A)
    N = 250.0
    g = torch.empty(R, device="cuda")
    lt = torch.empty(R, device="cuda")
    logp = torch.empty(R, device="cuda")
    xd = x.cuda()
    dx = torch.empty_like(xd)
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    fa = P.ppo_args(logp_behav=_cuda(lb), adv=_cuda(adv), version=_cuda(ver), slot_key=_cuda(key),
                    a_tok=A, cur_version=100, tok_denominator=N, out_grad_logp=g, out_loss_tok=lt,
                    logp_ref=_cuda(lref) if var.get("kl_coef") else None, **var)
    P.rlvla_logprob_fwd_bwd(xd, _cuda(t), logp=logp, fused=fa, dlogits=dx, stats=st, ws=P.workspace(1))
    valid = np.repeat(key != 0, A)
    lag = np.repeat(100 - ver.astype(np.int64), A)
    tv = dict(valid=valid, lag=lag, adv=np.repeat(adv, A).astype(np.float64), target=t, logp_behav=lb)
    ref = O_path.loss_and_grad(x64, tv, n_tok=N, dual_clip=var.get("dual_clip", 0.0),
                               logp_ref=lref if var.get("kl_coef") else None,
                               kl_coef=var.get("kl_coef", 0.0), ent_coef=var.get("ent_coef", 0.0))
    p, rs = ref["ppo"], ref["stats"]
    nt = p["near_tie"]
    H.assert_close_rel(logp.cpu().numpy(), ref["fwd"]["logp"], 1e-5, 1.0, "logp")
    # g = (-w A rho + kl (1 - e^{lref - logp})) / N inherits the logp tolerance through
    # dg/dlogp = (-w A rho + kl e^{lref - logp}) / N; the floor is that sensitivity times the
    # allowed logp error scale max(1, |logp|) (the two terms may cancel, so |g| is no scale)
    lpo = np.nan_to_num(ref["fwd"]["logp"], neginf=0.0)
    sens = np.abs(np.repeat(adv, A)) * np.nan_to_num(p["ratio"])
    if var.get("kl_coef"):
        sens = sens + var["kl_coef"] * np.exp(np.minimum(lref - lpo, 50.0))
    gfl = np.maximum(sens * np.maximum(1.0, np.abs(lpo)) / N, 1e-7)
    if not var.get("kl_coef"):
        # without the KL term g = -w A rho / N is a single product (no cancellation): the
        # plain 1e-5 relative bar of north_star, no sensitivity floor
        H.assert_close_rel(g.cpu().numpy()[~nt], p["grad"][~nt], 1e-5, 1e-30, "grad_logp (1e-5 rel)")
    # with the KL term (R20) the two terms may cancel: the floor above is derived in DESIGN §6
    H.assert_close_rel(g.cpu().numpy()[~nt], p["grad"][~nt], 1e-5, gfl[~nt], "grad_logp")
    H.assert_close_rel(lt.cpu().numpy()[~nt], p["loss_tok"][~nt], 1e-5, 1e-4, "loss_tok")
    d = dx.cpu()
    # error scale of dx_j = p_j (-g + c (log p_j + H)) [+ g at the target]: g carries its own
    # tolerance (gfl above), and the entropy bracket may cancel to ~0, so the scale is the
    # terms' magnitudes p_j (|g| + gfl + |c| (|log p_j| + |H| + 1))
    with np.errstate(invalid="ignore", over="ignore"):
        lpa = x64 - ref["fwd"]["lse"][:, None]
        pj = np.nan_to_num(np.exp(lpa))
        esc = np.abs(p["grad"])[:, None] + gfl[:, None]
        if var.get("ent_coef"):
            cr = np.where(p["mask"], var["ent_coef"] / N, 0.0)[:, None]
            Hr = np.nan_to_num(ref["fwd"]["entropy"])[:, None]
            esc = esc + cr * (np.abs(np.nan_to_num(lpa, neginf=0.0)) + np.abs(Hr) + 1.0)
        esc = pj * esc
        ta = np.nonzero(t >= 0)[0]
        esc[ta, t[ta]] += np.abs(p["grad"][ta]) + gfl[ta]      # the target's g (1 - p_a) term
    if dtype == torch.bfloat16:
        bits = d.view(torch.int16).numpy().astype(np.int32) & 0xFFFF
        H.assert_bf16_ulp(bits[~nt], ref["dx"][~nt], 1, abs_floor=1e-5 * esc[~nt])
    else:
        rsc = np.abs(ref["dx"]).max(axis=1, keepdims=True) * 1e-6
        fl = np.maximum(np.maximum(rsc, 1e-30), esc)
        H.assert_close_rel(d.numpy()[~nt], ref["dx"][~nt], 1e-5, fl[~nt], "dx")
    s = st.cpu().numpy()
    tol = lambda v: 1e-5 * max(1e-3, abs(v)) + 1e-6  # noqa: E731
    assert abs(s[6] - rs["loss"]) <= tol(rs["loss"]), (s[6], rs["loss"])
    assert abs(s[17] - rs["pg_loss"]) <= tol(rs["pg_loss"])
    assert abs(s[15] - rs["kl_ref_sum"]) <= tol(rs["kl_ref_sum"])
    assert abs(s[16] - rs["n_dual_clipped"]) <= nt.sum()
    assert abs(s[9] - rs["entropy_sum"]) <= tol(rs["entropy_sum"])
    assert s[11] == rs["n_loss_tok"] and s[18] == N


@pytest.mark.parametrize("var", [dict(), dict(dual_clip=3.0), dict(kl_coef=0.2)])
def test_ppo_loss_token_variants(var):
    P = _P()
    R, A = 700, 7
    rng = np.random.default_rng(1)
    logp = rng.normal(-4, 1, R).astype(np.float32)
    lb = (logp - rng.choice([-1.3, -0.1, 0.05, 1.4], R) - rng.normal(0, 0.01, R)).astype(np.float32)
    lref = (logp + rng.normal(0, 0.3, R)).astype(np.float32)
    adv = rng.normal(size=R // A).astype(np.float32)
    ver = np.full(R // A, 100, np.int32)
    key = np.ones(R // A, np.int64)
    g = torch.empty(R, device="cuda")
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    fa = P.ppo_args(logp_behav=_cuda(lb), adv=_cuda(adv), version=_cuda(ver), slot_key=_cuda(key),
                    a_tok=A, cur_version=100, tok_denominator=float(R),
                    logp_ref=_cuda(lref) if var.get("kl_coef") else None, **var)
    P.rlvla_ppo_loss(_cuda(logp), None, fa, g, None, st, P.workspace(1))
    o = O_ppo.ppo_loss(logp, lb, np.repeat(adv, A), np.ones(R, bool), np.zeros(R, int),
                       n_tok=float(R), dual_clip=var.get("dual_clip", 0.0),
                       logp_ref=lref if var.get("kl_coef") else None, kl_coef=var.get("kl_coef", 0.0))
    nt = o["near_tie"]
    # the PG and KL terms may cancel: the scale is the sum of their magnitudes
    sc = np.abs(np.repeat(adv, A)) * o["ratio"]
    if var.get("kl_coef"):
        lq = lref.astype(np.float64) - logp
        sc = sc + var["kl_coef"] * np.maximum(np.exp(lq), np.abs(np.expm1(lq)))
    H.assert_close_rel(g.cpu().numpy()[~nt], o["grad"][~nt], 1e-5, np.maximum(sc / R, 1e-9)[~nt], "grad")
    s = st.cpu().numpy()
    assert abs(s[6] - o["stats"]["loss"]) <= 1e-5 * abs(o["stats"]["loss"]) + 1e-7


def _chunk_case(S=300, A=56, seed=2):
    rng = np.random.default_rng(seed)
    R = S * A
    logp = rng.normal(-4, 1, R).astype(np.float32)
    lb = (logp - rng.normal(0, 0.004, R)).astype(np.float32)     # step ratios ~ e^{N(0, 0.03)}
    lpp = (lb + rng.normal(0, 0.003, R)).astype(np.float32)
    t = np.where(rng.random(R) < 0.03, -1, 5).astype(np.int32)
    t[7 * A:8 * A] = -1                                           # a step with no usable token
    adv = rng.normal(size=S).astype(np.float32)
    ver = (100 - rng.choice([0, 1, 2], size=S, p=[0.7, 0.2, 0.1])).astype(np.int32)
    key = np.where(rng.random(S) < 0.95, 3, 0).astype(np.int64)
    lag = np.repeat(100 - ver.astype(np.int64), A)
    m = np.repeat(key != 0, A) & (t >= 0) & (lag >= 0) & (lag <= 1)
    return R, logp, lb, lpp, t, adv, ver, key, m


CHUNK_VARIANTS = [dict(), dict(prox=True), dict(prox=True, is_cap=1.01), dict(dual_clip=1.02),
                  dict(prox=True, is_cap=1.01, dual_clip=1.02)]


@pytest.mark.parametrize("den", ["explicit", "adv_stats", "implicit"])
@pytest.mark.parametrize("var", CHUNK_VARIANTS)
def test_ppo_loss_chunk_ratio(var, den):
    """Chunk-level ratio (R21) incl. decoupled weights, the cap and dual clip at step level;
    N_steps explicit, from a stats vector's N_LOSS_STEPS slot, or the call's own count."""
    P = _P()
    S, A = 300, 56
    R, logp, lb, lpp, t, adv, ver, key, m = _chunk_case(S, A)
    prox = var.get("prox", False)
    kw = {k: v for k, v in var.items() if k != "prox"}
    o_kw = dict(logp_prox=lpp if prox else None, is_cap=var.get("is_cap", 0.0),
                dual_clip=var.get("dual_clip", 0.0))
    o_own = O_ppo.ppo_loss_chunk(logp, lb, adv, m, np.arange(R) // A, S, **o_kw)
    N = {"explicit": 777.0, "adv_stats": 555.0, "implicit": o_own["stats"]["n_steps"]}[den]
    o = O_ppo.ppo_loss_chunk(logp, lb, adv, m, np.arange(R) // A, S, n_den=N, **o_kw)
    if var.get("dual_clip"):
        assert o["stats"]["n_dual_clipped"] > 0
    g = torch.empty(R, device="cuda")
    lt = torch.empty(R, device="cuda")
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    ast = torch.zeros(24, dtype=torch.float64, device="cuda")
    ast[23] = 555.0
    fa = P.ppo_args(logp_behav=_cuda(lb), adv=_cuda(adv), version=_cuda(ver), slot_key=_cuda(key),
                    a_tok=A, cur_version=100, ratio_level=1,
                    logp_prox=_cuda(lpp) if prox else None,
                    tok_denominator=777.0 if den == "explicit" else 0.0,
                    adv_stats=ast if den == "adv_stats" else None, **kw)
    P.rlvla_ppo_loss(_cuda(logp), _cuda(t), fa, g, lt, st, P.workspace(1))
    okt = ~np.repeat(o["near_tie_step"], A)
    H.assert_close_rel(g.cpu().numpy()[okt], o["grad"][okt], 1e-5, 1e-9, "chunk grad")
    s = st.cpu().numpy()
    assert abs(s[6] - o["stats"]["loss"]) <= 1e-5 * abs(o["stats"]["loss"]) + 1e-7
    assert s[18] == N and s[11] == m.sum()
    assert s[16] == o["stats"]["n_dual_clipped"] and s[7] == o["stats"]["n_clipped"]
    assert abs(lt.double().sum().item() - o["loss_step"].sum()) <= 1e-4 * abs(o["loss_step"].sum()) + 1e-5


def test_ppo_loss_chunk_micro_batches_and_guards():
    """Streamer micro-batches of the chunk path (accumulate) with N_steps from the stats
    vector: grads bit-identical to one call, stats within 1e-12; the call's own count with
    accumulate, or a KL term, are refused; rows = 0 with stats writes zeros."""
    P = _P()
    S, A = 300, 56
    R, logp, lb, lpp, t, adv, ver, key, m = _chunk_case(S, A, seed=5)
    ast = torch.zeros(24, dtype=torch.float64, device="cuda")
    ast[23] = 290.0
    base = dict(logp_behav=_cuda(lb), adv=_cuda(adv), version=_cuda(ver), slot_key=_cuda(key),
                a_tok=A, cur_version=100, ratio_level=1, adv_stats=ast, logp_prox=_cuda(lpp))
    g1 = torch.empty(R, device="cuda")
    st1 = torch.zeros(24, dtype=torch.float64, device="cuda")
    ws = P.workspace(1)
    P.rlvla_ppo_loss(_cuda(logp), _cuda(t), P.ppo_args(**base), g1, None, st1, ws)
    g2 = torch.empty(R, device="cuda")
    st2 = torch.zeros(24, dtype=torch.float64, device="cuda")
    lpd, td = _cuda(logp), _cuda(t)
    for s0, s1 in ((0, 64), (64, 65), (65, 200), (200, 300)):
        r0, r1 = s0 * A, s1 * A
        fa = P.ppo_args(logp_behav=base["logp_behav"][r0:r1], adv=base["adv"][s0:s1],
                        version=base["version"][s0:s1], slot_key=base["slot_key"][s0:s1], a_tok=A,
                        cur_version=100, ratio_level=1, adv_stats=ast, logp_prox=base["logp_prox"][r0:r1],
                        accumulate=1)
        P.rlvla_ppo_loss(lpd[r0:r1], td[r0:r1], fa, g2[r0:r1], None, st2, ws)
    assert torch.equal(g1, g2)
    a, b = st1.cpu().numpy(), st2.cpu().numpy()
    for k in range(6, 19):
        assert abs(a[k] - b[k]) <= 1e-12 * max(1.0, abs(a[k])), (k, a[k], b[k])
    o = O_ppo.ppo_loss_chunk(logp, lb, adv, m, np.arange(R) // A, S, n_den=290.0, logp_prox=lpp)
    assert abs(a[6] - o["stats"]["loss"]) <= 1e-5 * abs(o["stats"]["loss"]) + 1e-7
    # refused: accumulate without a known N_steps, KL on the chunk path
    bad = dict(base, adv_stats=None, accumulate=1)
    with pytest.raises(P.RlvlaError) as e:
        P.rlvla_ppo_loss(lpd, td, P.ppo_args(**bad), g2, None, st2, ws)
    assert e.value.status == 1
    with pytest.raises(P.RlvlaError) as e:
        P.rlvla_ppo_loss(lpd, td, P.ppo_args(**dict(base, logp_ref=lpd, kl_coef=0.1)), g2, None, st2, ws)
    assert e.value.status == 2
    # rows = 0 with stats: this call's totals (zeros), DENOM = N
    st3 = torch.full((24,), 9.0, dtype=torch.float64, device="cuda")
    e0 = torch.empty(0, device="cuda")
    fa0 = P.ppo_args(logp_behav=e0, adv=e0, version=torch.empty(0, dtype=torch.int32, device="cuda"),
                     slot_key=torch.empty(0, dtype=torch.int64, device="cuda"), a_tok=A,
                     cur_version=100, ratio_level=1, adv_stats=ast)
    P.rlvla_ppo_loss(e0, None, fa0, e0, None, st3, ws)
    s3 = st3.cpu().numpy()
    assert (s3[6:18] == 0).all() and s3[18] == 290.0 and (s3[:6] == 9.0).all()


@pytest.mark.parametrize("clip_eps,denom", [(0.2, 0.0), (0.0, 0.0), (0.5, 1234.0)])
def test_value_loss(clip_eps, denom):
    P = _P()
    n = 5000
    rng = np.random.default_rng(3)
    v, vo, R = (rng.normal(size=n).astype(np.float32) for _ in range(3))
    key = np.where(rng.random(n) < 0.9, 1, 0).astype(np.int64)
    ver = (100 - rng.choice([0, 1, 2], size=n, p=[0.7, 0.2, 0.1])).astype(np.int32)
    gv = torch.empty(n, device="cuda")
    ls = torch.empty(n, device="cuda")
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    P.rlvla_value_loss(_cuda(v), _cuda(vo), _cuda(R), _cuda(key), _cuda(ver), 100, gv,
                       clip_eps=clip_eps, denominator=denom, loss_step=ls, stats=st, ws=P.workspace(1))
    lag = 100 - ver.astype(np.int64)
    m = (key != 0) & (lag >= 0) & (lag <= 1)
    o = O_ppo.value_loss(v, vo, R, m, clip_eps=clip_eps, n_den=denom if denom > 0 else None)
    d = np.abs(v.astype(np.float64) - vo)
    ok = np.abs(d - clip_eps) > 1e-5 if clip_eps > 0 else np.ones(n, bool)
    H.assert_close_rel(gv.cpu().numpy()[ok], o["grad"][ok], 1e-5, 1e-9, "value grad")
    s = st.cpu().numpy()
    assert abs(s[19] - o["stats"]["loss"]) <= 1e-5 * o["stats"]["loss"]
    assert s[21] == m.sum() and s[22] == o["stats"]["denom"]
    assert abs(s[20] - o["stats"]["n_clipped"]) <= (~ok).sum()


def test_gae_truncation():
    P = _P()
    E, T = 64, 200
    rng = np.random.default_rng(4)
    r, V = rng.normal(size=(E, T)).astype(np.float32), rng.normal(size=(E, T)).astype(np.float32)
    B = rng.normal(size=(E, T)).astype(np.float32)
    d = rng.choice([0, 1, 2], size=(E, T), p=[0.96, 0.02, 0.02]).astype(np.uint8)
    lv = rng.normal(size=E).astype(np.float32)
    buf = P.TrajectoryBuffer.allocate(E, T, 1)
    buf.reward.copy_(_cuda(r))
    buf.value.copy_(_cuda(V))
    buf.done.copy_(_cuda(d))
    buf.version.fill_(100)
    buf.slot_key.fill_(1)
    adv = torch.zeros(E, T, device="cuda")
    ret = torch.zeros(E, T, device="cuda")
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    P.rlvla_advantages(buf, _cuda(lv), P.adv_params("gae", gamma=0.99, lam=0.95, n_env_global=E,
                                                    cur_version=100, boot_value=_cuda(B)),
                       adv, ret, st, P.workspace(E))
    a, rr = O_adv.gae(r, V, d, np.ones((E, T)), lv, 0.99, 0.95, boot_value=B)
    fl = max(1e-3, float(np.sqrt(np.mean(a ** 2))))
    H.assert_close_rel(adv.cpu().numpy(), a, 1e-5, fl, "adv (truncation)")
    H.assert_close_rel(ret.cpu().numpy(), rr, 1e-5, fl, "ret (truncation)")
