"""Small inputs through every kernel path, for compute-sanitizer (one tool per run):
  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_drive.py
Paths: single-CTA and multi-CTA scatter, GAE(+whiten) and GRPO, warp / TMA / generic
log-prob kernels in fwd, fused (with and without dlogits, standard and decoupled,
accumulate, every NEXT-2 knob) and external-bwd modes, in-place dlogits, rlvla_ppo_loss
(token and chunk ratio), rlvla_value_loss, the NEXT-3 batcher (both observation layouts) and
the NEXT-4 flow kernels (tile and scalar paths, fused and external backward)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2602_05765_b200 as P  # noqa: E402
from tests import harness as H  # noqa: E402


def main():
    torch.cuda.set_device(0)
    # tiny path (warp kernels), then a 2-env OpenVLA-shaped case (TMA kernel)
    for cfg in (synth.CONFIGS["tiny"], synth.scaled(synth.CONFIGS["libero_spatial_oft"], n_env=2)):
        case = H.build_case(cfg, device="cuda", behav_sample=8)
        buf, cnt = H.gpu_scatter(case, chunk=64)
        buf2, _ = H.gpu_scatter(case, chunk=5000)           # multi-CTA claim/write kernels
        E, T, A = case.n_env, cfg.t_steps, cfg.a_tok
        ws = P.workspace(E)
        stats = torch.zeros(24, dtype=torch.float64, device="cuda")
        adv = torch.zeros(E, T, device="cuda")
        ret = torch.zeros(E, T, device="cuda")
        lv = torch.from_numpy(case.traj.last_value).cuda()
        P.rlvla_advantages(buf, lv, P.adv_params("gae", whiten=True, n_env_global=E, cur_version=100),
                           adv, ret, stats, ws)
        gid = torch.from_numpy(case.traj.group_id).cuda()
        P.rlvla_advantages(buf, lv, P.adv_params("grpo", group_id=gid, group_size=cfg.group_size,
                                                 n_env_global=E, cur_version=100), adv, ret, stats, ws)
        x = case.logits
        R = x.shape[0]
        tgt = buf.tokens.view(-1)
        logp = torch.empty(R, device="cuda")
        lse = torch.empty(R, device="cuda")
        g = torch.empty(R, device="cuda")
        dx = torch.empty_like(x)
        st = torch.zeros(24, dtype=torch.float64, device="cuda")
        P.rlvla_logprob_fwd_bwd(x, tgt, logp=logp, lse=lse, stats=st, ws=ws)
        for prox in (None, buf.logp_behav.view(-1)):
            fa = P.ppo_args(logp_behav=buf.logp_behav.view(-1), logp_prox=prox, adv=adv.view(-1),
                            version=buf.version.view(-1), slot_key=buf.slot_key.view(-1), a_tok=A,
                            cur_version=100, adv_stats=stats, out_grad_logp=g, is_cap=2.0)
            P.rlvla_logprob_fwd_bwd(x, tgt, logp=logp, lse=lse, fused=fa, dlogits=dx, stats=st, ws=ws)
            P.rlvla_logprob_fwd_bwd(x, tgt, logp=logp, fused=fa, stats=st, ws=ws)   # no dlogits
        fa2 = P.ppo_args(logp_behav=buf.logp_behav.view(-1), adv=adv.view(-1),
                         version=buf.version.view(-1), slot_key=buf.slot_key.view(-1), a_tok=A,
                         cur_version=100, tok_denominator=100.0, accumulate=True)
        P.rlvla_logprob_fwd_bwd(x[:A * 3], tgt[:A * 3], logp=logp[:A * 3], fused=fa2,
                                dlogits=dx[:A * 3], stats=st, ws=ws)
        P.rlvla_logprob_fwd_bwd(x, tgt, lse=lse, grad_logp=g, dlogits=dx)          # external bwd
        y = x.clone()
        P.rlvla_logprob_fwd_bwd(y, tgt, logp=logp, fused=fa, dlogits=y)           # in place
        P.rlvla_ppo_loss(logp, tgt, fa, g, torch.empty(R, device="cuda"), st, ws)
        # NEXT-2: every loss knob on the fused call (x-path pass C with the entropy bonus),
        # the chunk-level ratio and the value loss
        fa3 = P.ppo_args(logp_behav=buf.logp_behav.view(-1), adv=adv.view(-1),
                         version=buf.version.view(-1), slot_key=buf.slot_key.view(-1), a_tok=A,
                         cur_version=100, adv_stats=stats, out_grad_logp=g, dual_clip=3.0,
                         logp_ref=buf.logp_behav.view(-1), kl_coef=0.1, ent_coef=0.01)
        P.rlvla_logprob_fwd_bwd(x, tgt, logp=logp, fused=fa3, dlogits=dx, stats=st, ws=ws)
        fa4 = P.ppo_args(logp_behav=buf.logp_behav.view(-1), adv=adv.view(-1),
                         version=buf.version.view(-1), slot_key=buf.slot_key.view(-1), a_tok=A,
                         cur_version=100, ratio_level=1)
        P.rlvla_ppo_loss(logp, tgt, fa4, g, None, st, ws)
        nsteps = E * T
        P.rlvla_value_loss(buf.value.view(-1), buf.value.view(-1), ret.view(-1), buf.slot_key.view(-1),
                           buf.version.view(-1), 100, torch.empty(nsteps, device="cuda"),
                           loss_step=torch.empty(nsteps, device="cuda"), stats=st, ws=ws)
    # generic path: ragged vocabulary, fp32 and bf16
    for dt in (torch.float32, torch.bfloat16):
        x = (torch.randn(20, 1003, device="cuda") * 2).to(dt)
        t = torch.randint(-1, 1003, (20,), device="cuda", dtype=torch.int32)
        lp = torch.empty(20, device="cuda")
        ls = torch.empty(20, device="cuda")
        P.rlvla_logprob_fwd_bwd(x, t, logp=lp, lse=ls)
        P.rlvla_logprob_fwd_bwd(x, t, lse=ls, grad_logp=torch.ones(20, device="cuda"),
                                dlogits=torch.empty_like(x))
    # NEXT-3: both observation layouts, offers with rejections, firing and idle polls
    for fifo in (False, True):
        q = P.BatchQueue.allocate(40, 4096 + 48, obs_fifo=fifo, max_batch=8 if fifo else 0)
        ws = P.workspace(1)
        cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
        src = torch.randint(0, 256, (12, 4096 + 48), dtype=torch.uint8, device="cuda")
        oe = torch.empty(8, dtype=torch.int32, device="cuda")
        ot = torch.empty(8, dtype=torch.int64, device="cuda")
        on = torch.empty(1, dtype=torch.int32, device="cuda")
        oo = torch.empty(8, 4096 + 48, dtype=torch.uint8, device="cuda")
        for k in range(12):
            env = torch.tensor([(3 * k + j) % 45 for j in range(12)], dtype=torch.int32, device="cuda")
            P.rlvla_batch_offer(q, env, torch.full((12,), k, dtype=torch.int64, device="cuda"), k, cnt,
                                obs_src=src, ws=ws)
            P.rlvla_batch_poll(q, k, 8, 2, oe, ot, on, out_obs=None if fifo else oo, ws=ws)
    # NEXT-4: chains, fused (schedule and learned ln sigma, tile and scalar paths), external bwd
    for K, D in ((4, 70), (3, 7)):
        R = 37
        mu = torch.randn(R, K, D, device="cuda").to(torch.bfloat16)
        x = torch.randn(R, K, D, device="cuda")
        ls = torch.randn(R, K, D, device="cuda") * 0.3 - 1.0
        sig = torch.linspace(0.8, 0.2, K, device="cuda")
        lb = torch.full((R,), -100.0, device="cuda")
        fa5 = P.ppo_args(logp_behav=lb, adv=torch.randn(R, device="cuda"),
                         version=torch.full((R,), 100, dtype=torch.int32, device="cuda"),
                         slot_key=torch.ones(R, dtype=torch.int64, device="cuda"), a_tok=1,
                         cur_version=100, tok_denominator=float(R), ent_coef=0.01)
        st = torch.zeros(24, dtype=torch.float64, device="cuda")
        ws = P.workspace(1)
        for learned in (None, ls):
            ch = P.GaussChain(mu, x, sig, learned)
            P.rlvla_flow_logprob(ch, logp=torch.empty(R, device="cuda"), fused=fa5, dmu=torch.empty_like(mu),
                                 dlog_std=None if learned is None else torch.empty_like(x), stats=st, ws=ws)
        P.rlvla_flow_logprob(P.GaussChain(mu, x, None, ls), grad_logp=torch.ones(R, device="cuda"),
                             dmu=torch.empty_like(mu), dlog_std=torch.empty_like(x))
    torch.cuda.synchronize()
    print("SANITIZE DRIVE OK")


if __name__ == "__main__":
    main()
