"""GPU parity: the whole rollout-to-loss path (S1 -> S2 -> S3+S4) through the C ABI vs the
oracle, element by element, on the tiny config (everything) and on a LIBERO-OFT-shaped
reduction (bf16 V=32000, TMA path; S1/S2 in full, S3/S4 on every row of a few envs).

Un-isolated, as bench.py runs it: the GPU chain feeds its OWN buffer, advantages and loss
token count (adv_stats) into S3+S4; the oracle chain runs on its own from the same records
and logits. Nothing crosses between the two. S2's tolerance (1e-5 of max(|A|, rms A)) is
propagated into S4 and S3's backward through the sensitivities dg/dA = -w rho / N,
dL/dA = -w max(rho, clip rho) and d dx_j / dg = 1[j = a] - p_j."""
import numpy as np
import pytest
import torch

import synth
from oracle import path as O_path
from tests import harness as H

pytestmark = pytest.mark.gpu

CUR = synth.CUR_VERSION


def _gpu_advantages(case, mode, buf, whiten=False):
    import paper_2602_05765_b200 as P
    cfg = case.cfg
    E, T = case.n_env, cfg.t_steps
    dev = "cuda"
    ws = P.workspace(E, device=dev)
    stats = torch.zeros(24, dtype=torch.float64, device=dev)
    adv = torch.zeros(E, T, dtype=torch.float32, device=dev)
    ret = torch.zeros(E, T, dtype=torch.float32, device=dev)
    lv = torch.from_numpy(case.traj.last_value[case.env_lo:case.env_hi]).to(dev)
    gid = torch.from_numpy(case.traj.group_id).to(dev)
    prm = P.adv_params(mode, whiten=whiten, group_id=gid if mode == "grpo" else None,
                       group_size=cfg.group_size, n_env_global=E, cur_version=CUR,
                       max_staleness=1)
    P.rlvla_advantages(buf, lv, prm, adv, ret, stats, ws)
    torch.cuda.synchronize()
    return adv, ret, stats, ws


def _gpu_loss(case, buf, adv, stats, ws, tok_den=0.0):
    import paper_2602_05765_b200 as P
    cfg = case.cfg
    E, T, A = case.n_env, cfg.t_steps, cfg.a_tok
    dev = "cuda"
    R = E * T * A
    logits = case.logits.to(dev)
    logp = torch.empty(R, dtype=torch.float32, device=dev)
    lse = torch.empty(R, dtype=torch.float32, device=dev)
    g = torch.empty(R, dtype=torch.float32, device=dev)
    lt = torch.empty(R, dtype=torch.float32, device=dev)
    dx = torch.empty_like(logits)
    fa = P.ppo_args(logp_behav=buf.logp_behav.view(-1), adv=adv.view(-1), version=buf.version.view(-1),
                    slot_key=buf.slot_key.view(-1), a_tok=A, cur_version=CUR, max_staleness=1,
                    tok_denominator=tok_den, adv_stats=stats, out_grad_logp=g, out_loss_tok=lt)
    st2 = torch.zeros(24, dtype=torch.float64, device=dev)
    P.rlvla_logprob_fwd_bwd(logits, buf.tokens.view(-1), logp=logp, lse=lse, fused=fa,
                            dlogits=dx, stats=st2, ws=ws)
    torch.cuda.synchronize()
    stats_all = stats.cpu().numpy().copy()
    stats_all[6:] = st2.cpu().numpy()[6:]
    return dict(logp=logp.cpu().numpy(), lse=lse.cpu().numpy(), g=g.cpu().numpy(),
                lt=lt.cpu().numpy(), dx=dx, stats=stats_all)


def _compare_path(case, mode, whiten=False, rows=None):
    """S1, S2 and S3+S4 each compared, the GPU chain running on its own outputs."""
    cfg = case.cfg
    # S1: bit-exact buffer and counters
    gbuf, gcnt = H.gpu_scatter(case)
    obuf, ocnt = H.oracle_scatter(case)
    gb = H.buf_to_np(gbuf)
    for k in obuf:
        assert np.array_equal(gb[k].view(np.uint8), obuf[k].view(np.uint8)), f"buffer.{k}"
    assert gcnt.cpu().numpy().tolist() == ocnt.tolist()
    # S2
    adv, ret, stats, ws = _gpu_advantages(case, mode, gbuf, whiten=whiten)
    oadv = H.oracle_advantages(case, obuf, mode, whiten=whiten)
    floor = max(1e-3, float(np.sqrt(np.mean(oadv["adv"] ** 2))))
    H.assert_close_rel(adv.cpu().numpy(), oadv["adv"], 1e-5, floor, "adv")
    H.assert_close_rel(ret.cpu().numpy(), oadv["ret"], 1e-5, floor, "ret")
    c = oadv["counts"]
    st = stats.cpu().numpy()
    assert st[0] == c["n_valid"] and st[3] == c["n_tok"] and st[4] == c["n_stale"] and st[5] == c["n_bad"]
    # S3+S4 on the GPU's own advantages and count; the oracle on its own
    out = _gpu_loss(case, gbuf, adv, stats, ws)
    tol_adv = 1e-5 * np.maximum(np.abs(oadv["adv"]), floor)           # the S2 bar, per step
    tv = O_path.token_view(obuf, oadv["adv"], cfg.a_tok, CUR)
    tol_tok = np.repeat(tol_adv.reshape(-1), cfg.a_tok)
    rows = np.arange(len(tv["target"])) if rows is None else rows
    refs = []
    for s in range(0, len(rows), 2048):
        rr = rows[s:s + 2048]
        refs.append(_compare_rows(case, out, tv, rr, float(c["n_tok"]), tol_tok[rr]))
    ref = _merge(refs)
    return out, ref, oadv


def _compare_rows(case, out, tv, rows, n_tok, tol_adv):
    xr = case.logits[torch.from_numpy(rows).to(case.logits.device)].double().cpu().numpy()
    loc = {k: (v[rows] if k != "dx" else v[torch.from_numpy(rows).cuda()]) for k, v in out.items()
           if k in ("logp", "lse", "g", "lt", "dx")}
    return check_rows(xr, loc, tv, rows, n_tok, tol_adv, case.logits.dtype)


def check_rows(xr, loc, tv, rows, n_tok, tol_adv, dtype):
    """The GPU outputs of token rows `rows` (loc: logp, lse, g, lt as numpy arrays and dx as a
    device tensor, all in the order of `rows`) against the oracle chain on the same logits xr,
    with S2's tolerance tol_adv (per row) propagated into S4 and S3's backward."""
    ref = O_path.loss_and_grad(xr, tv, n_tok=n_tok, rows=rows)
    f, p = ref["fwd"], ref["ppo"]
    H.assert_close_rel(loc["logp"], f["logp"], 1e-5, 1.0, "logp")
    fin = np.isfinite(f["lse"])
    if "lse" in loc:
        H.assert_close_rel(loc["lse"][fin], f["lse"][fin], 1e-5, 1.0, "lse")
    # S2's tolerance propagated: |dg/dA| = w rho / N, |dL/dA| <= w max(rho, 1 + eps)
    m = p["mask"]
    wr = np.where(m, np.nan_to_num(p["w"] * p["ratio"]), 0.0)
    g_extra = wr * tol_adv / n_tok
    l_extra = np.where(m, np.nan_to_num(p["w"] * np.maximum(p["ratio"], 1.2)), 0.0) * tol_adv
    # near-ties (|rho/bound - 1| <= 1e-5) may take either branch (reading R11)
    nt = p["near_tie"]
    ga = np.abs(p["grad"])
    H.assert_close_rel(loc["g"][~nt], p["grad"][~nt], 1e-5, np.maximum(ga + g_extra / 1e-5, 1e-30)[~nt],
                       "grad_logp")
    if "lt" in loc:
        la = np.abs(p["loss_tok"])
        H.assert_close_rel(loc["lt"], p["loss_tok"], 1e-5, np.maximum(la, 1e-3) + l_extra / 1e-5, "loss_tok")
    dx = loc["dx"]
    # dx_j = g (1[j = a] - p_j): g's tolerance times |1[j = a] - p_j|
    with np.errstate(invalid="ignore", over="ignore"):
        pj = np.nan_to_num(np.exp(xr - f["lse"][:, None]))
    ind = np.zeros_like(pj)
    ta = np.nonzero(tv["target"][rows] >= 0)[0]
    ind[ta, tv["target"][rows][ta]] = 1.0
    dg = (1e-5 * ga + g_extra)[:, None] * np.abs(ind - pj)
    if dtype == torch.bfloat16:
        bits = dx.view(torch.int16).cpu().numpy().astype(np.int32) & 0xFFFF
        # within 1 ulp of RNE(ref'), ref' within dg of ref: |gpu - ref| <= dg + 1.5 ulp(ref)
        with np.errstate(divide="ignore"):
            ulp = np.exp2(np.floor(np.log2(np.maximum(np.abs(ref["dx"]), 2.0 ** -126))) - 7)
        H.assert_bf16_ulp(bits[~nt], ref["dx"][~nt], 1, abs_floor=(dg + 1.5 * ulp)[~nt])
    else:
        d = dx.cpu().numpy()
        rowscale = np.abs(ref["dx"]).max(axis=1, keepdims=True)
        fl = np.maximum(rowscale * 1e-6, 1e-30) + dg / 1e-5
        H.assert_close_rel(d[~nt], ref["dx"][~nt], 1e-5, np.maximum(np.abs(ref["dx"]), fl)[~nt], "dlogits")
    return dict(stats=ref["stats"], near_tie=int(nt.sum()), loss_extra=float(l_extra.sum() / n_tok))


def _merge(refs):
    st = {k: sum(r["stats"][k] for r in refs) for k in refs[0]["stats"] if k != "denom"}
    st["denom"] = refs[0]["stats"]["denom"]
    return dict(stats=st, near_tie=sum(r["near_tie"] for r in refs),
                loss_extra=sum(r["loss_extra"] for r in refs))


def test_tiny_full_path_grpo():
    case = H.build_case(synth.CONFIGS["tiny"], device="cpu")
    out, ref, oadv = _compare_path(case, "grpo")
    st, rs = out["stats"], ref["stats"]
    assert abs(st[6] - rs["loss"]) <= 1e-5 * max(1.0, abs(rs["loss"])) + ref["loss_extra"]
    for slot, key in ((8, "kl_k3_sum"), (9, "entropy_sum"), (10, "ratio_sum"), (14, "logp_sum")):
        assert abs(st[slot] - rs[key]) <= 1e-5 * max(1.0, abs(rs[key])), key
    assert st[11] == rs["n_loss_tok"] and st[12] == rs["n_stale_tok"] and st[13] == rs["n_bad_tok"]
    assert abs(st[7] - rs["n_clipped"]) <= ref["near_tie"]
    assert st[18] == oadv["counts"]["n_tok"]
    # the fault injections really happened
    assert rs["n_stale_tok"] > 0 and rs["n_bad_tok"] == 0


def test_tiny_full_path_gae_whitened():
    case = H.build_case(synth.CONFIGS["tiny"], device="cpu")
    out, ref, _ = _compare_path(case, "gae", whiten=True)
    assert abs(out["stats"][6] - ref["stats"]["loss"]) <= 1e-5 * max(1.0, abs(ref["stats"]["loss"])) + ref["loss_extra"]


def test_oft_shape_reduced_tma_path():
    """LIBERO-Spatial OFT recipe (bf16, V=32000, A=56, T=64) on 2 envs: S1/S2 in full,
    S3/S4 on every row (7,168 rows x 32000)."""
    cfg = synth.scaled(synth.CONFIGS["libero_spatial_oft"], n_env=2)
    case = H.build_case(cfg, device="cuda")
    out, ref, _ = _compare_path(case, "grpo")
    assert np.abs(out["logp"] - 0).max() > 0
    st, rs = out["stats"], ref["stats"]
    assert abs(st[6] - rs["loss"]) <= 1e-5 * max(1e-3, abs(rs["loss"])) + ref["loss_extra"]
    assert st[11] == rs["n_loss_tok"]


@pytest.mark.parametrize("mode,whiten", [("grpo", False), ("gae", True)])
def test_oft_shape_two_groups_bench_chain(mode, whiten):
    """The bench's chain on a 16-env OFT-shaped slice (two GRPO groups of 8 / GAE with
    whitening): 1,024 records in 16 arrival chunks, advantages, one fused launch over all
    57,344 rows with the GPU's own advantages and N_tok; S3/S4 compared on 4,096 sampled
    rows plus the crafted ones."""
    cfg = synth.scaled(synth.CONFIGS["libero_spatial_oft"], n_env=16)
    case = H.build_case(cfg, device="cuda", behav_sample=64)
    rng = np.random.default_rng(3)
    crafted = np.concatenate([np.asarray(v) for v in case.traj.crafted.values()])
    rows = np.unique(np.concatenate([rng.choice(case.logits.shape[0], 4096, replace=False), crafted]))
    _compare_path(case, mode, whiten=whiten, rows=rows)
