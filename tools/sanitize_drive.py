"""Small inputs through every kernel path, for compute-sanitizer (one tool per run):
  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_drive.py
Paths: single-CTA and multi-CTA scatter, GAE(+whiten) and GRPO, warp / TMA / generic
log-prob kernels in fwd, fused (with and without dlogits, standard and decoupled,
accumulate) and external-bwd modes, in-place dlogits, rlvla_ppo_loss."""
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
    # generic path: ragged vocabulary, fp32 and bf16
    for dt in (torch.float32, torch.bfloat16):
        x = (torch.randn(20, 1003, device="cuda") * 2).to(dt)
        t = torch.randint(-1, 1003, (20,), device="cuda", dtype=torch.int32)
        lp = torch.empty(20, device="cuda")
        ls = torch.empty(20, device="cuda")
        P.rlvla_logprob_fwd_bwd(x, t, logp=lp, lse=ls)
        P.rlvla_logprob_fwd_bwd(x, t, lse=ls, grad_logp=torch.ones(20, device="cuda"),
                                dlogits=torch.empty_like(x))
    torch.cuda.synchronize()
    print("SANITIZE DRIVE OK")


if __name__ == "__main__":
    main()
