"""Out-of-bounds write detection without compute-sanitizer (closed on the GPU pool): every
output of every entry point is carved from a larger allocation whose 4 KB before and after
are filled with a canary pattern, on shapes with ragged tails; after the calls the canaries
must be intact. Covers the scatter buffer, advantages, the three log-prob kernel paths (all
modes), rlvla_ppo_loss (token and chunk ratio), rlvla_value_loss, the batcher (both
observation layouts) and the flow kernels (tile and scalar paths)."""
import numpy as np
import pytest
import torch

import synth
from tests import harness as H

pytestmark = pytest.mark.gpu
GUARD = 4096
CANARY = 0xA5


class Guarded:
    def __init__(self):
        self.blocks = []

    def __call__(self, shape, dtype, fill=0):
        n = int(np.prod(shape)) * torch.tensor([], dtype=dtype).element_size()
        raw = torch.full((GUARD + n + GUARD,), CANARY, dtype=torch.uint8, device="cuda")
        self.blocks.append((raw, n))
        t = raw[GUARD:GUARD + n].view(dtype).view(*shape)
        if fill is not None:
            t.fill_(fill)
        return t

    def check(self, what=""):
        torch.cuda.synchronize()
        for raw, n in self.blocks:
            lo, hi = raw[:GUARD], raw[GUARD + n:]
            assert bool((lo == CANARY).all()) and bool((hi == CANARY).all()), f"canary overwritten ({what})"


def _P():
    import paper_2602_05765_b200 as P
    return P


def test_guards_core_path():
    P = _P()
    gd = Guarded()
    for cfg in (synth.CONFIGS["tiny"], synth.scaled(synth.CONFIGS["libero_spatial_oft"], n_env=3)):
        case = H.build_case(cfg, device="cuda", behav_sample=8)
        E, T, A, V = case.n_env, cfg.t_steps, cfg.a_tok, cfg.vocab
        buf = P.TrajectoryBuffer(E, T, A, gd((E, T), torch.int64), gd((E, T), torch.float32),
                                 gd((E, T), torch.uint8), gd((E, T), torch.float32), gd((E, T), torch.int32),
                                 gd((E, T, A), torch.int32), gd((E, T, A), torch.float32))
        rec = H.to_dev_batch(case)
        cnt = gd((4,), torch.int64)
        seq = 1
        for sl in synth.arrival_chunks(rec.n, 64):
            P.rlvla_scatter_steps(buf, rec.slice(sl), synth.CUR_VERSION, seq, cnt)
            seq += sl.stop - sl.start
        P.rlvla_scatter_steps(buf, rec, synth.CUR_VERSION, seq, cnt)       # multi-CTA path
        ws = P.workspace(E)
        st = gd((24,), torch.float64)
        adv, ret = gd((E, T), torch.float32), gd((E, T), torch.float32)
        lv = torch.from_numpy(case.traj.last_value).cuda()
        P.rlvla_advantages(buf, lv, P.adv_params("gae", whiten=True, n_env_global=E, cur_version=100),
                           adv, ret, st, ws)
        P.rlvla_advantages(buf, lv, P.adv_params("grpo", group_id=torch.from_numpy(case.traj.group_id).cuda(),
                                                 group_size=cfg.group_size, n_env_global=E, cur_version=100),
                           adv, ret, st, ws)
        R = E * T * A
        x = case.logits
        tgt = buf.tokens.view(-1)
        logp, lse, g, lt = (gd((R,), torch.float32) for _ in range(4))
        dx = gd(tuple(x.shape), x.dtype)
        P.rlvla_logprob_fwd_bwd(x, tgt, logp=logp, lse=lse, stats=st, ws=ws)
        for var in (dict(), dict(dual_clip=3.0, logp_ref=buf.logp_behav.view(-1), kl_coef=0.1, ent_coef=0.01)):
            fa = P.ppo_args(logp_behav=buf.logp_behav.view(-1), adv=adv.view(-1), version=buf.version.view(-1),
                            slot_key=buf.slot_key.view(-1), a_tok=A, cur_version=100, adv_stats=st,
                            out_grad_logp=g, out_loss_tok=lt, **var)
            P.rlvla_logprob_fwd_bwd(x, tgt, logp=logp, lse=lse, fused=fa, dlogits=dx, stats=st, ws=ws)
        P.rlvla_logprob_fwd_bwd(x, tgt, lse=lse, grad_logp=g, dlogits=dx)
        fa = P.ppo_args(logp_behav=buf.logp_behav.view(-1), adv=adv.view(-1), version=buf.version.view(-1),
                        slot_key=buf.slot_key.view(-1), a_tok=A, cur_version=100, adv_stats=st)
        P.rlvla_ppo_loss(logp, tgt, fa, g, lt, st, ws)
        fa.ratio_level = 1
        P.rlvla_ppo_loss(logp, tgt, fa, g, lt, st, ws)
        gv, ls_ = gd((E * T,), torch.float32), gd((E * T,), torch.float32)
        P.rlvla_value_loss(buf.value.view(-1), buf.value.view(-1), ret.view(-1), buf.slot_key.view(-1),
                           buf.version.view(-1), 100, gv, loss_step=ls_, stats=st, ws=ws)
        gd.check(cfg.name)
    # generic path: ragged V, fp32
    x = torch.randn(19, 1003, device="cuda")
    t = torch.randint(-1, 1003, (19,), device="cuda", dtype=torch.int32)
    lp, ls2 = gd((19,), torch.float32), gd((19,), torch.float32)
    dx = gd((19, 1003), torch.float32)
    P.rlvla_logprob_fwd_bwd(x, t, logp=lp, lse=ls2)
    P.rlvla_logprob_fwd_bwd(x, t, lse=ls2, grad_logp=torch.ones(19, device="cuda"), dlogits=dx)
    gd.check("generic")
    # row path: aligned fp32 beyond the warp kernel, fused with PPO statistics
    x = torch.randn(21, 8192, device="cuda")
    t = torch.randint(-1, 8192, (21,), device="cuda", dtype=torch.int32)
    lp, ls2 = gd((21,), torch.float32), gd((21,), torch.float32)
    dx = gd((21, 8192), torch.float32)
    P.rlvla_logprob_fwd_bwd(x, t, logp=lp, lse=ls2)
    P.rlvla_logprob_fwd_bwd(x, t, lse=ls2, grad_logp=torch.ones(21, device="cuda"), dlogits=dx)
    gd.check("row")


@pytest.mark.parametrize("fifo", [False, True])
def test_guards_batcher(fifo):
    P = _P()
    gd = Guarded()
    E, ob, B = 41, 3 * 16 + 16 * 1000, 7
    rows = E + (B if fifo else 0)
    q = P.BatchQueue(E, ob, gd((rows, ob), torch.uint8), gd((E,), torch.int32), gd((E,), torch.int64),
                     gd((E,), torch.uint8), gd((8,), torch.int64), int(fifo), B if fifo else 0)
    ws = P.workspace(1)
    cnt = gd((4,), torch.int64)
    oe, ot, on = gd((B,), torch.int32), gd((B,), torch.int64), gd((1,), torch.int32)
    oo = gd((B, ob), torch.uint8)
    src = torch.randint(0, 256, (13, ob), dtype=torch.uint8, device="cuda")
    for k in range(40):
        env = torch.tensor([(5 * k + j) % 47 for j in range(13)], dtype=torch.int32, device="cuda")
        P.rlvla_batch_offer(q, env, torch.full((13,), k, dtype=torch.int64, device="cuda"), k, cnt,
                            obs_src=src, ws=ws)
        P.rlvla_batch_poll(q, k, B, 3, oe, ot, on, out_obs=oo, ws=ws)
    gd.check(f"batcher fifo={fifo}")


@pytest.mark.parametrize("K,D", [(4, 70), (4, 35), (3, 7)])
def test_guards_flow(K, D):
    P = _P()
    gd = Guarded()
    R = 45
    mu = torch.randn(R, K, D, device="cuda").to(torch.bfloat16)
    x = torch.randn(R, K, D, device="cuda")
    lsd = torch.randn(R, K, D, device="cuda") * 0.3 - 1.0
    sig = torch.linspace(0.8, 0.2, K, device="cuda")
    g, lt, logp = gd((R,), torch.float32), gd((R,), torch.float32), gd((R,), torch.float32)
    fa = P.ppo_args(logp_behav=torch.full((R,), -100.0, device="cuda"), adv=torch.randn(R, device="cuda"),
                    version=torch.full((R,), 100, dtype=torch.int32, device="cuda"),
                    slot_key=torch.ones(R, dtype=torch.int64, device="cuda"), a_tok=1, cur_version=100,
                    tok_denominator=float(R), out_grad_logp=g, out_loss_tok=lt, ent_coef=0.01)
    st = gd((24,), torch.float64)
    ws = P.workspace(1)
    for learned in (None, lsd):
        dmu = gd((R, K, D), torch.bfloat16)
        dls = gd((R, K, D), torch.float32) if learned is not None else None
        P.rlvla_flow_logprob(P.GaussChain(mu, x, sig, learned), logp=logp, fused=fa, dmu=dmu, dlog_std=dls,
                             stats=st, ws=ws)
        P.rlvla_flow_logprob(P.GaussChain(mu, x, sig, learned), logp=logp, stats=st, ws=ws)
    P.rlvla_flow_logprob(P.GaussChain(mu, x, None, lsd), grad_logp=torch.ones(R, device="cuda"),
                         dmu=gd((R, K, D), torch.bfloat16), dlog_std=gd((R, K, D), torch.float32))
    gd.check(f"flow {K}x{D}")
