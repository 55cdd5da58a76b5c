"""Streamer (§3.3): the fused S3+S4 pass run micro-batch by micro-batch
as the trajectory buffer fills, with a fixed global token denominator and statistics
accumulated in call order, equals the single full-batch call: per-row
outputs and dlogits bit-identical (rows are independent), statistics equal to fp64
rounding; and both equal the oracle."""
import numpy as np
import pytest
import torch

import synth
from oracle import path as O_path
from tests import harness as H

pytestmark = pytest.mark.gpu


def _fused(P, x, tgt, buf, adv, rows, A, N, stats, ws, accumulate, comm=None):
    r0, r1 = rows
    s0, s1 = r0 // A, r1 // A
    g = torch.empty(r1 - r0, device="cuda")
    logp = torch.empty(r1 - r0, device="cuda")
    dx = torch.empty(r1 - r0, x.shape[1], dtype=x.dtype, device="cuda")
    fa = P.ppo_args(logp_behav=buf.logp_behav.view(-1)[r0:r1], adv=adv.view(-1)[s0:s1],
                    version=buf.version.view(-1)[s0:s1], slot_key=buf.slot_key.view(-1)[s0:s1],
                    a_tok=A, cur_version=synth.CUR_VERSION, tok_denominator=N, out_grad_logp=g,
                    accumulate=accumulate)
    P.rlvla_logprob_fwd_bwd(x[r0:r1], tgt[r0:r1], logp=logp, fused=fa, dlogits=dx, stats=stats,
                            ws=ws, comm=comm)
    return logp, g, dx


@pytest.mark.parametrize("cfg_name,n_env", [("tiny", 8), ("libero_spatial_oft", 2)])
def test_streamer_equals_full_batch(cfg_name, n_env):
    import paper_2602_05765_b200 as P
    cfg = synth.scaled(synth.CONFIGS[cfg_name], n_env=n_env)
    case = H.build_case(cfg, device="cuda")
    buf, _ = H.gpu_scatter(case)
    obuf, _ = H.oracle_scatter(case)
    oadv = H.oracle_advantages(case, obuf, "grpo")
    A, T = cfg.a_tok, cfg.t_steps
    # the GPU chain's own advantages (GRPO: fp32 rounding of the oracle's, checked here)
    adv = torch.zeros(n_env, T, device="cuda")
    P.rlvla_advantages(buf, None, P.adv_params("grpo", group_id=torch.from_numpy(case.traj.group_id).cuda(),
                                               group_size=cfg.group_size, n_env_global=n_env,
                                               cur_version=synth.CUR_VERSION),
                       adv, torch.zeros(n_env, T, device="cuda"),
                       torch.zeros(24, dtype=torch.float64, device="cuda"), P.workspace(n_env))
    H.assert_close_rel(adv.cpu().numpy(), oadv["adv"], 1e-5, 1e-3, "adv")
    x = case.logits.cuda()
    tgt = buf.tokens.view(-1)
    R = x.shape[0]
    N = float(oadv["counts"]["n_tok"])
    ws = P.workspace(n_env)
    st_full = torch.zeros(24, dtype=torch.float64, device="cuda")
    lf, gf, df = _fused(P, x, tgt, buf, adv, (0, R), A, N, st_full, ws, False)
    # uneven micro-batches of whole decision steps, in arrival order
    cuts = [0, 3 * A, 17 * A, (R // A // 2) * A, R]
    st_mb = torch.zeros(24, dtype=torch.float64, device="cuda")
    outs = [_fused(P, x, tgt, buf, adv, (a, b), A, N, st_mb, ws, True) for a, b in zip(cuts, cuts[1:])]
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([o[0] for o in outs]), lf)
    assert torch.equal(torch.cat([o[1] for o in outs]), gf)
    assert torch.equal(torch.cat([o[2] for o in outs]), df)
    a, b = st_full.cpu().numpy(), st_mb.cpu().numpy()
    np.testing.assert_allclose(b[6:18], a[6:18], rtol=1e-12, atol=1e-15)
    assert b[18] == a[18] == N
    # and the accumulated stats equal the oracle's
    tv = O_path.token_view(obuf, oadv["adv"], A, synth.CUR_VERSION)
    tot = {}
    for s in range(0, R, 2048):
        rr = np.arange(s, min(R, s + 2048))
        ref = O_path.loss_and_grad(x[torch.from_numpy(rr).cuda()].double().cpu().numpy(), tv,
                                   n_tok=N, rows=rr)["stats"]
        for k, v in ref.items():
            tot[k] = tot.get(k, 0.0) + v
    assert abs(b[6] - tot["loss"]) <= 1e-5 * max(1e-3, abs(tot["loss"]))
    assert b[11] == tot["n_loss_tok"]


def _sub_buffer(P, buf, e0, e1):
    """Envs [e0, e1) of a trajectory buffer as a buffer of its own (views, no copy)."""
    return P.TrajectoryBuffer(e1 - e0, buf.t_steps, buf.a_tok, *(getattr(buf, f)[e0:e1] for f in (
        "slot_key", "reward", "done", "value", "version", "tokens", "logp_behav")))


@pytest.mark.parametrize("reserve", [0, 1])
def test_streamer_interleaved_two_streams(reserve):
    """The Streamer schedule (§3.3) on two streams: micro-batch k = whole GRPO groups;
    its records are scattered and its advantages computed on a rollout-side stream while the
    actor stream runs the fused S3+S4 of micro-batch k-1 (explicit global denominator,
    statistics accumulated in micro-batch order; the persistent kernel leaves `reserve` SMs
    free). Buffer, advantages, logp, grad and dlogits are bit-identical to the serial
    full-batch path, statistics within 1e-12."""
    import paper_2602_05765_b200 as P
    G = 2
    cfg = synth.scaled(synth.CONFIGS["libero_spatial_oft"], n_env=6, group_size=G)
    case = H.build_case(cfg, device="cuda")
    A, T = cfg.a_tok, cfg.t_steps
    E = cfg.n_env
    x = case.logits.cuda()
    R = x.shape[0]
    obuf, _ = H.oracle_scatter(case)
    N = float(H.oracle_advantages(case, obuf, "grpo")["counts"]["n_tok"])
    # serial reference: whole batch on one stream
    buf_s, _ = H.gpu_scatter(case)
    adv_s = torch.zeros(E, T, device="cuda")
    P.rlvla_advantages(buf_s, None, P.adv_params("grpo", group_size=G, n_env_global=E, cur_version=synth.CUR_VERSION),
                       adv_s, torch.zeros(E, T, device="cuda"), torch.zeros(24, dtype=torch.float64, device="cuda"),
                       P.workspace(E))
    st_s = torch.zeros(24, dtype=torch.float64, device="cuda")
    ref = _fused(P, x, buf_s.tokens.view(-1), buf_s, adv_s, (0, R), A, N, st_s, P.workspace(E), False)
    # streamer: micro-batch k = group k (envs [kG, kG + G)), its records in arrival order
    rec = H.to_dev_batch(case)
    env_np = case.rec.env_id
    buf = P.TrajectoryBuffer.allocate(E, T, A)
    adv = torch.zeros(E, T, device="cuda")
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    ws_roll, ws_act = P.workspace(G), P.workspace(E)
    side = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    prev = P.rlvla_set_reserved_sms(reserve)
    outs, seq = [], 1
    nmb = E // G
    mbs, idxs = [], []
    for k in range(nmb):          # each micro-batch's records (local env ids), built up front
        e0 = k * G
        idx = np.nonzero((env_np >= e0) & (env_np < e0 + G))[0]
        it = torch.from_numpy(idx).cuda()
        mb = P.StepBatch(*(getattr(rec, f)[it].contiguous() for f in (
            "env_id", "step", "version", "reward", "done", "value", "tokens", "logp_behav")))
        mb.env_id.sub_(e0)
        mbs.append(mb)
        idxs.append(idx)
    try:
        side.wait_stream(main)
        ready = [torch.cuda.Event() for _ in range(nmb)]
        for k in range(nmb):
            e0, e1 = k * G, (k + 1) * G
            sub = _sub_buffer(P, buf, e0, e1)
            idx, mb = idxs[k], mbs[k]
            with torch.cuda.stream(side):
                cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
                for c0 in range(0, len(idx), synth.B_MAX):
                    c1 = min(len(idx), c0 + synth.B_MAX)
                    P.rlvla_scatter_steps(sub, mb.slice(slice(c0, c1)), synth.CUR_VERSION, seq + c0, cnt,
                                          stream=side)
                P.rlvla_advantages(sub, None, P.adv_params("grpo", group_size=G, n_env_global=G,
                                                           cur_version=synth.CUR_VERSION),
                                   adv[e0:e1], torch.zeros(G, T, device="cuda"),
                                   torch.zeros(24, dtype=torch.float64, device="cuda"), ws_roll, stream=side)
                ready[k].record(side)
            seq += len(idx)
            main.wait_event(ready[k])
            outs.append(_fused(P, x, buf.tokens.view(-1), buf, adv, (e0 * T * A, e1 * T * A), A, N, st,
                               ws_act, k > 0))
        torch.cuda.synchronize()
    finally:
        P.rlvla_set_reserved_sms(prev)
    gb, gs = H.buf_to_np(buf), H.buf_to_np(buf_s)
    for k in gb:
        assert np.array_equal(gb[k].view(np.uint8), gs[k].view(np.uint8)) or k == "slot_key", k
    assert np.array_equal(gb["slot_key"] != 0, gs["slot_key"] != 0)
    assert torch.equal(adv, adv_s)
    for j in range(3):
        assert torch.equal(torch.cat([o[j] for o in outs]), ref[j]), j
    a, b = st_s.cpu().numpy(), st.cpu().numpy()
    np.testing.assert_allclose(b[6:18], a[6:18], rtol=1e-12, atol=1e-15)
