"""GPU parity for rlvla_logprob_fwd_bwd in all three modes and all four kernel paths
(warp / TMA / row / generic), plus rlvla_ppo_loss, against the oracle; crafted edge rows,
ragged vocabularies, ignore/bad targets, non-finite rows, in-place dlogits, determinism."""
import numpy as np
import pytest
import torch

from oracle import logprob as O_lp
from oracle import ppo as O_ppo
from tests import harness as H

pytestmark = pytest.mark.gpu


def _P():
    import paper_2602_05765_b200 as P
    return P


def _rows(R, V, dtype, seed=0, scale=1.5):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = torch.randn(R, V, generator=g) * scale
    # crafted rows
    if R >= 8:
        x[0] = 0.0                                   # uniform
        x[1] = -30.0
        x[1, 3 % V] = 30.0                            # saturated (target 3)
        x[2] = -1.0
        x[2, 5 % V] = 4.0
        x[2, 9 % V] = 4.0                             # tied max incl. target 5
        x[3, [1 % V, 2 % V, (V // 2) % V]] = float("-inf")  # -inf columns (target 0)
    return x.to(dtype)


def _targets(R, V, seed=1):
    g = np.random.default_rng(seed)
    t = g.integers(0, V, size=R).astype(np.int32)
    if R >= 8:
        t[0], t[1], t[2], t[3] = 7 % V, 3 % V, 5 % V, 0
        t[4] = -1          # ignore
        t[5] = V           # bad target (counted)
        t[6] = -5          # bad target (counted)
    return t


def _bits(x: torch.Tensor):
    return x.view(torch.int16).cpu().numpy().astype(np.int32) & 0xFFFF


def _check_dx(dx_gpu, ref64, dtype):
    if dtype == torch.bfloat16:
        H.assert_bf16_ulp(_bits(dx_gpu), ref64, 1)
    else:
        rs = np.abs(ref64).max(axis=1, keepdims=True)
        H.assert_close_rel(dx_gpu.cpu().numpy(), ref64, 1e-5, np.maximum(rs * 1e-6, 1e-30), "dx")


CASES = [
    # (R, V, dtype, expected path)
    (300, 256, torch.float32, "warp"),
    (300, 1000, torch.float32, "warp"),
    (300, 256, torch.bfloat16, "warp"),
    (300, 2048, torch.bfloat16, "warp"),
    (700, 32000, torch.bfloat16, "tma"),
    (150, 4104, torch.bfloat16, "tma"),
    (150, 32768, torch.bfloat16, "tma"),
    (64, 31999, torch.bfloat16, "generic"),    # ragged: V % 8 != 0
    (64, 5003, torch.float32, "generic"),      # ragged: V % 4 != 0
    (64, 5000, torch.float32, "row"),          # aligned fp32 beyond the warp path
    (300, 32000, torch.float32, "row"),        # fp32 logits at the OpenVLA vocabulary
    (40, 40000, torch.bfloat16, "row"),        # bf16 beyond the TMA stage
]


@pytest.mark.parametrize("R,V,dtype,path", CASES)
def test_forward_and_external_backward(R, V, dtype, path):
    P = _P()
    x = _rows(R, V, dtype).cuda()
    t = _targets(R, V)
    tgt = torch.from_numpy(t).cuda()
    logp = torch.full((R,), 123.0, device="cuda")
    lse = torch.empty(R, device="cuda")
    stats = torch.zeros(24, dtype=torch.float64, device="cuda")
    ws = P.workspace(1)
    P.rlvla_logprob_fwd_bwd(x, tgt, logp=logp, lse=lse, stats=stats, ws=ws)
    x64 = x.double().cpu().numpy()
    f = O_lp.log_softmax_gather(x64, t)
    H.assert_close_rel(logp.cpu().numpy(), f["logp"], 1e-5, 1.0, "logp")
    H.assert_close_rel(lse.cpu().numpy(), f["lse"], 1e-5, 1.0, "lse")
    st = stats.cpu().numpy()
    ok = f["status"] == 0
    assert st[11] == ok.sum() and st[13] == ((f["status"] == 2) | (f["status"] == 3)).sum()
    assert abs(st[9] - f["entropy"][ok].sum()) <= 1e-5 * max(1, abs(f["entropy"][ok].sum()))
    assert abs(st[14] - f["logp"][ok].sum()) <= 1e-5 * max(1, abs(f["logp"][ok].sum()))
    # external-gradient backward with the oracle's own lse? No: with the GPU lse just
    # produced (the call's contract), compared with the oracle gradient at the oracle lse.
    g = np.random.default_rng(3).normal(size=R).astype(np.float32)
    gg = torch.from_numpy(g).cuda()
    dx = torch.full_like(x, 7.0)
    P.rlvla_logprob_fwd_bwd(x, tgt, lse=lse, grad_logp=gg, dlogits=dx)
    gref = np.where(ok | (f["status"] == 3), g.astype(np.float64), 0.0)
    gref[~ok] = 0.0
    ref = O_lp.log_softmax_grad(x64, t, f["lse"], gref)
    fin = np.nonzero(np.isfinite(f["lse"]))[0]
    d = dx[torch.from_numpy(fin).cuda()]
    r = ref[fin].copy()
    # target column: given only an fp32 lse, 1 - p_a = -expm1(x_a - lse) carries the
    # rounding of lse (half an fp32 ulp of |lse|); compare it at that precision, the rest
    # of the row at 1 ulp / 1e-5
    tf = t[fin]
    tok = (tf >= 0) & (tf < V)
    ri, ci = np.nonzero(tok)[0], tf[tok]
    gd = d[torch.from_numpy(ri).cuda(), torch.from_numpy(ci).cuda()].float().cpu().numpy()
    lse32 = lse.cpu().numpy()[fin][ri].astype(np.float64)
    tol = np.abs(g[fin][ri]) * (np.spacing(np.abs(lse32).astype(np.float32)).astype(np.float64) * 2
                                + 1e-5 * np.abs(r[ri, ci] / np.where(g[fin][ri] == 0, 1, g[fin][ri])))
    tol = np.maximum(tol, np.abs(r[ri, ci]) * (2 ** -8 if dtype == torch.bfloat16 else 1e-5))
    assert np.all(np.abs(gd - r[ri, ci]) <= tol), np.max(np.abs(gd - r[ri, ci]) - tol)
    d[torch.from_numpy(ri).cuda(), torch.from_numpy(ci).cuda()] = 0
    r[ri, ci] = 0.0
    _check_dx(d, r, dtype)
    torch.cuda.synchronize()


def _ppo_inputs(R, A, seed=5):
    rng = np.random.default_rng(seed)
    S = R // A
    adv = rng.normal(size=S).astype(np.float32)
    ver = (100 - rng.choice([0, 1, 2, -1], size=S, p=[0.6, 0.3, 0.08, 0.02])).astype(np.int32)
    key = np.where(rng.random(S) < 0.95, (ver.astype(np.uint64) << np.uint64(40)) + np.uint64(1),
                   np.uint64(0)).astype(np.uint64)
    return adv, ver, key


@pytest.mark.parametrize("R,V,dtype,path", [c for c in CASES if c[0] % 2 == 0] + [(301, 256, torch.float32, "warp")])
@pytest.mark.parametrize("decoupled", [False, True])
def test_fused_ppo(R, V, dtype, path, decoupled):
    P = _P()
    A = 7 if R % 7 == 0 else (2 if R % 2 == 0 else 1)
    x = _rows(R, V, dtype).cuda()
    t = _targets(R, V)
    x64 = x.double().cpu().numpy()
    f = O_lp.log_softmax_gather(x64, t)
    rng = np.random.default_rng(11)
    lb = (np.nan_to_num(f["logp"], nan=-3.0) + rng.normal(0, 0.15, R)).astype(np.float32)
    lpp = (np.nan_to_num(f["logp"], nan=-3.0) + rng.normal(0, 0.05, R)).astype(np.float32) if decoupled else None
    adv, ver, key = _ppo_inputs(R, A)
    cuda = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    g = torch.empty(R, device="cuda")
    lt = torch.empty(R, device="cuda")
    logp = torch.empty(R, device="cuda")
    dx = torch.empty_like(x)
    stats = torch.zeros(24, dtype=torch.float64, device="cuda")
    ws = P.workspace(1)
    N = 1000.0
    fa = P.ppo_args(logp_behav=cuda(lb), logp_prox=cuda(lpp) if decoupled else None,
                    adv=cuda(adv), version=cuda(ver), slot_key=cuda(key.view(np.int64)), a_tok=A,
                    cur_version=100, max_staleness=1, eps_low=0.2, eps_high=0.28,
                    is_cap=3.0 if decoupled else 0.0, tok_denominator=N, out_grad_logp=g,
                    out_loss_tok=lt)
    P.rlvla_logprob_fwd_bwd(x, cuda(t), logp=logp, fused=fa, dlogits=dx, stats=stats, ws=ws)
    valid = np.repeat(key != 0, A)
    lag = np.repeat(100 - ver.astype(np.int64), A)
    base = valid & (f["status"] == 0)
    o = O_ppo.ppo_loss(f["logp"], lb, np.repeat(adv, A), base, lag, eps_low=0.2, eps_high=0.28,
                       n_tok=N, logp_prox=lpp, is_cap=3.0 if decoupled else 0.0)
    nt = o["near_tie"]
    H.assert_close_rel(logp.cpu().numpy(), f["logp"], 1e-5, 1.0, "logp")
    H.assert_close_rel(g.cpu().numpy()[~nt], o["grad"][~nt], 1e-5, 1e-6, "grad")
    H.assert_close_rel(lt.cpu().numpy(), o["loss_tok"], 1e-5, 1e-4, "loss_tok")
    ref = O_lp.log_softmax_grad(x64, t, f["lse"], o["grad"])
    _check_dx(dx[torch.from_numpy(np.nonzero(~nt)[0]).cuda()], ref[~nt], dtype)
    st = stats.cpu().numpy()
    s = o["stats"]
    assert abs(st[6] - s["loss"]) <= 1e-5 * max(1e-3, abs(s["loss"]))
    assert st[11] == s["n_loss_tok"] and st[12] == s["n_stale_tok"]
    bad = valid & ((f["status"] == 2) | (f["status"] == 3))
    assert st[13] == bad.sum() + s["n_bad_lag"]
    assert abs(st[8] - s["kl_k3_sum"]) <= 1e-5 * max(1e-3, abs(s["kl_k3_sum"])) + 1e-6 * s["n_loss_tok"]
    assert abs(st[10] - s["ratio_sum"]) <= 1e-5 * max(1.0, s["ratio_sum"])
    ent = np.where(o["mask"], f["entropy"], 0).sum()
    assert abs(st[9] - ent) <= 1e-5 * max(1.0, abs(ent))
    assert st[18] == N
    # the same epilogue through rlvla_ppo_loss on the GPU log-probs (fused == unfused)
    g2 = torch.empty(R, device="cuda")
    lt2 = torch.empty(R, device="cuda")
    st2 = torch.zeros(24, dtype=torch.float64, device="cuda")
    tg = cuda(np.where((t >= 0) & (t < V), t, np.where(t == -1, -1, -2)).astype(np.int32))
    P.rlvla_ppo_loss(logp, tg, fa, g2, lt2, st2, ws)
    assert torch.equal(g2, g) and torch.equal(lt2, lt)


def test_in_place_dlogits_and_determinism():
    P = _P()
    R, V = 300, 32000
    x = _rows(R, V, torch.bfloat16, seed=9).cuda()
    t = torch.from_numpy(_targets(R, V)).cuda()
    A = 3
    adv, ver, key = _ppo_inputs(R, A)
    cuda = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    lb = torch.full((R,), -8.0, device="cuda")
    fa = P.ppo_args(logp_behav=lb, adv=cuda(adv), version=cuda(ver),
                    slot_key=cuda(key.view(np.int64)), a_tok=A, cur_version=100,
                    tok_denominator=512.0)
    outs = []
    for _ in range(2):
        logp = torch.empty(R, device="cuda")
        dx = torch.empty_like(x)
        st = torch.zeros(24, dtype=torch.float64, device="cuda")
        P.rlvla_logprob_fwd_bwd(x, t, logp=logp, fused=fa, dlogits=dx, stats=st, ws=P.workspace(1))
        outs.append((logp, dx, st))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    assert torch.equal(outs[0][2], outs[1][2])
    y = x.clone()
    logp = torch.empty(R, device="cuda")
    P.rlvla_logprob_fwd_bwd(y, t, logp=logp, fused=fa, dlogits=y, stats=None)
    assert torch.equal(y, outs[0][1]) and torch.equal(logp, outs[0][0])


def test_fwd_only_equals_fused_logp():
    P = _P()
    R, V = 512, 32000
    x = _rows(R, V, torch.bfloat16, seed=4).cuda()
    t = torch.from_numpy(_targets(R, V)).cuda()
    l1 = torch.empty(R, device="cuda")
    P.rlvla_logprob_fwd_bwd(x, t, logp=l1)
    adv, ver, key = _ppo_inputs(R, 4)
    cuda = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    fa = P.ppo_args(logp_behav=torch.zeros(R, device="cuda"), adv=cuda(adv), version=cuda(ver),
                    slot_key=cuda(key.view(np.int64)), a_tok=4, cur_version=100,
                    tok_denominator=1.0)
    l2 = torch.empty(R, device="cuda")
    P.rlvla_logprob_fwd_bwd(x, t, logp=l2, fused=fa, dlogits=torch.empty_like(x))
    assert torch.equal(l1, l2)


def test_ratio_one_pin_through_gpu():
    """logp_behav := the GPU's own logp => rho = exp(0) = 1 exactly: loss = -sum m A / N,
    no clipping, k3 = 0 (SURVEY §8(c) S4 pin (i))."""
    P = _P()
    R, V, A = 700, 32000, 7
    x = _rows(R, V, torch.bfloat16, seed=2).cuda()
    t = torch.from_numpy(np.random.default_rng(0).integers(0, V, R).astype(np.int32)).cuda()
    lp0 = torch.empty(R, device="cuda")
    P.rlvla_logprob_fwd_bwd(x, t, logp=lp0)
    adv = np.random.default_rng(1).normal(size=R // A).astype(np.float32)
    cuda = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    key = torch.ones(R // A, dtype=torch.int64, device="cuda")
    ver = torch.full((R // A,), 100, dtype=torch.int32, device="cuda")
    g = torch.empty(R, device="cuda")
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    fa = P.ppo_args(logp_behav=lp0, adv=cuda(adv), version=ver, slot_key=key, a_tok=A,
                    cur_version=100, tok_denominator=float(R), out_grad_logp=g)
    P.rlvla_logprob_fwd_bwd(x, t, logp=torch.empty(R, device="cuda"), fused=fa,
                            dlogits=torch.empty_like(x), stats=st, ws=P.workspace(1))
    s = st.cpu().numpy()
    A_tok = np.repeat(adv.astype(np.float64), A)
    assert abs(s[6] - (-A_tok.sum() / R)) < 1e-6
    assert s[7] == 0 and s[8] == 0.0 and s[10] == R
    np.testing.assert_allclose(g.cpu().numpy(), -A_tok / R, rtol=1e-6)
