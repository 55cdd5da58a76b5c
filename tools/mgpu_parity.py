"""Multi-GPU parity of the CUDA path (run under torchrun, one rank per GPU, NCCL):
each rank scatters the records it owns, computes GRPO (groups spanning ranks: C2
allgather + C1 allreduce) and GAE+global whitening advantages, and the fused loss with the
C3 allreduce, all through the C ABI with the library's NCCL communicator; the result is
compared with the oracle on the same shard using the same sharding helpers. Then the value
loss (slots 19..21) and the flow-policy chain loss (C3) with a global denominator, and rank
invariance: the same global problem on one rank vs sharded gives bit-identical GRPO advantages
and per-row logp / grad / dlogits, and loss statistics within 1e-12.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_parity.py

RLVLA_MGPU_MODE=p2p-only: no NCCL anywhere — a gloo process group, the library's P2P-only
communicator (CUDA IPC mailbox handles exchanged over gloo) and ranks placed round-robin on
the visible GPUs, so 8 ranks run on 4 GPUs (2 per GPU) and the in-kernel C1/C2/C3 exchange
runs at its full 8-rank capacity.

Also covered: the chunk-ratio path with its default normaliser (the global step count, and
N_LOSS_STEPS from rlvla_advantages), the value loss with its own global count, and a rank
whose share of a fused call is empty (it still takes part in C3).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
import paper_2602_05765_b200 as P  # noqa: E402
from paper_2602_05765_b200 import sharding  # noqa: E402
from oracle import advantages as O_adv  # noqa: E402
from oracle import logprob as O_lp  # noqa: E402
from oracle import path as O_path  # noqa: E402
from oracle import scatter as O_sc  # noqa: E402
from tests import harness as H  # noqa: E402

CUR = synth.CUR_VERSION


MODE = os.environ.get("RLVLA_MGPU_MODE", "nccl")


def _host_coll(fn, t, *a):
    """Run a torch collective; with gloo on host copies (results copied back)."""
    if MODE == "nccl":
        return fn(t, *a)
    if isinstance(t, list):
        h = [x.cpu() for x in t]
        fn(h, *(x.cpu() for x in a))
        for x, y in zip(t, h):
            x.copy_(y)
        return
    h = t.cpu()
    fn(h, *a)
    t.copy_(h)


def all_reduce(t):
    _host_coll(dist.all_reduce, t)


def all_gather(out, t):
    _host_coll(lambda o, x: dist.all_gather(o, x), out, t)


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    ndev = torch.cuda.device_count()
    local = local % ndev                      # p2p-only: several ranks per GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if MODE == "nccl":
        dist.init_process_group("nccl", device_id=dev)
        comm = P.Comm.from_process_group(device=dev)
    else:
        dist.init_process_group("gloo")
        comm = P.Comm.p2p_from_process_group()
        assert comm.p2p, "P2P-only communicator did not connect"
    E = 16 * world
    cfg = synth.scaled(synth.CONFIGS["tiny"], n_env=E, group_size=4, interleave_groups=True)
    traj = synth.make_trajectories(cfg)
    rec = synth.make_records(traj, 0, E)
    lo, hi = sharding.env_range(E, world, rank)
    E_r, T, A, V = hi - lo, cfg.t_steps, cfg.a_tok, cfg.vocab
    idx, local_env = sharding.route_records(rec.env_id, E, world, rank)
    x = synth.gen_logits(cfg, traj, 0, E).double().numpy()            # all rows (for lb)
    rows_g = synth.record_rows(rec, cfg, E)
    f = O_lp.log_softmax_gather(x, traj.tokens.reshape(-1))["logp"]
    lb = (np.where(rows_g >= 0, np.nan_to_num(f)[np.maximum(rows_g, 0)], 0.0) + rec.behav_noise).astype(np.float32)
    recd = dict(env_id=local_env, step=rec.step[idx], version=rec.version[idx],
                reward=rec.reward[idx], done=rec.done[idx], value=rec.value[idx],
                tokens=rec.tokens[idx], logp_behav=lb[idx])
    # ---- oracle on this shard (host) ----------------------------------------------------
    obuf = O_sc.new_buffer(E_r, T, A)
    ocnt = O_sc.scatter_steps(obuf, recd, CUR, 1)
    # ---- CUDA path ----------------------------------------------------------------------
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    batch = P.StepBatch(*(t(recd[k]) for k in ("env_id", "step", "version", "reward", "done",
                                                 "value", "tokens", "logp_behav")))
    buf = P.TrajectoryBuffer.allocate(E_r, T, A, device=dev)
    cnt = torch.zeros(4, dtype=torch.int64, device=dev)
    P.rlvla_scatter_steps(buf, batch, CUR, 1, cnt)
    gb = H.buf_to_np(buf)
    for k in obuf:
        assert np.array_equal(gb[k].view(np.uint8), obuf[k].view(np.uint8)), k
    assert cnt.cpu().numpy().tolist() == ocnt.tolist()
    ws = P.workspace(E, device=dev)
    gid = t(traj.group_id)
    lv = t(traj.last_value[lo:hi])
    valid = obuf["slot_key"] != 0
    # GRPO with groups spanning ranks (C2 + C1)
    adv = torch.zeros(E_r, T, device=dev)
    ret = torch.zeros(E_r, T, device=dev)
    st = torch.zeros(24, dtype=torch.float64, device=dev)
    P.rlvla_advantages(buf, lv, P.adv_params("grpo", group_id=gid, group_size=4, env_offset=lo,
                                             n_env_global=E, cur_version=CUR), adv, ret, st, ws,
                       comm=comm)
    R_all = [torch.zeros(E_r, dtype=torch.float64, device=dev) for _ in range(world)]
    all_gather(R_all, torch.from_numpy(O_adv.episode_return(obuf["reward"], valid)).to(dev))
    R_glob = torch.cat(R_all).cpu().numpy()
    a_ref = O_adv.grpo_step_adv(O_adv.grpo(R_glob, traj.group_id)[lo:hi], valid)
    H.assert_close_rel(adv.cpu().numpy(), a_ref, 1e-5, 1e-3, "grpo adv (spanning ranks)")
    c = O_adv.step_counts(valid, obuf["version"], obuf["tokens"], CUR, 1)
    tot = torch.tensor([c["n_valid"], c["n_tok"], c["n_stale"], c["n_bad"]], dtype=torch.float64, device=dev)
    all_reduce(tot)
    s = st.cpu().numpy()
    assert (s[0], s[3], s[4], s[5]) == tuple(tot.cpu().numpy().tolist()), (s[:6], tot)
    # GAE + global whitening (C1)
    adv2 = torch.zeros(E_r, T, device=dev)
    st2 = torch.zeros(24, dtype=torch.float64, device=dev)
    P.rlvla_advantages(buf, lv, P.adv_params("gae", whiten=True, env_offset=lo, n_env_global=E,
                                             cur_version=CUR), adv2, ret, st2, ws, comm=comm)
    a_gae, _ = O_adv.gae(obuf["reward"], obuf["value"], obuf["done"], valid, traj.last_value[lo:hi], 0.99, 0.95)
    ws_ = torch.tensor(O_adv.whiten_stats(a_gae, valid), dtype=torch.float64, device=dev)
    all_reduce(ws_)
    a_w = O_adv.whiten(a_gae, valid, 1e-8, stats=tuple(ws_.cpu().numpy()))
    H.assert_close_rel(adv2.cpu().numpy(), a_w, 1e-5, max(1e-3, float(np.sqrt(np.mean(a_w ** 2)))), "gae whitened")
    # fused loss with global N_tok (from st) and C3, on the GPU's own advantages (GRPO: the
    # fp32 rounding of the oracle's value, 6e-8 relative, far inside the 1e-5 bar)
    xr = torch.from_numpy(x[lo * T * A:hi * T * A].astype(np.float32)).to(dev)
    R = E_r * T * A
    logp = torch.empty(R, device=dev)
    g = torch.empty(R, device=dev)
    dx = torch.empty_like(xr)
    st3 = torch.zeros(24, dtype=torch.float64, device=dev)
    fa = P.ppo_args(logp_behav=buf.logp_behav.view(-1), adv=adv.view(-1), version=buf.version.view(-1),
                    slot_key=buf.slot_key.view(-1), a_tok=A, cur_version=CUR, adv_stats=st,
                    out_grad_logp=g)
    P.rlvla_logprob_fwd_bwd(xr, buf.tokens.view(-1), logp=logp, fused=fa, dlogits=dx, stats=st3,
                            ws=ws, comm=comm)
    torch.cuda.synchronize()
    tv = O_path.token_view(obuf, a_ref, A, CUR)
    ref = O_path.loss_and_grad(x[lo * T * A:hi * T * A], tv, n_tok=float(tot[1].item()))
    nt = ref["ppo"]["near_tie"]
    H.assert_close_rel(g.cpu().numpy()[~nt], ref["ppo"]["grad"][~nt], 1e-5, 1e-7, "grad (global N)")
    rs = torch.tensor([ref["stats"][k] for k in ("loss", "n_loss_tok", "entropy_sum")],
                      dtype=torch.float64, device=dev)
    all_reduce(rs)
    s3 = st3.cpu().numpy()
    rs = rs.cpu().numpy()
    assert abs(s3[6] - rs[0]) <= 1e-5 * max(1e-3, abs(rs[0])), (s3[6], rs[0])
    assert s3[11] == rs[1] and abs(s3[9] - rs[2]) <= 1e-5 * abs(rs[2])
    assert s3[18] == tot[1].item()
    # ---- rank invariance: the same global problem on ONE rank vs sharded ----
    # GRPO advantages and every per-row output bit-identical; global stats within 1e-12
    full_batch = P.StepBatch(*(t(a_) for a_ in (rec.env_id, rec.step, rec.version, rec.reward, rec.done,
                                                rec.value, rec.tokens, lb)))
    buf_f = P.TrajectoryBuffer.allocate(E, T, A, device=dev)
    P.rlvla_scatter_steps(buf_f, full_batch, CUR, 1, torch.zeros(4, dtype=torch.int64, device=dev))
    adv_f = torch.zeros(E, T, device=dev)
    st_f = torch.zeros(24, dtype=torch.float64, device=dev)
    ws_f = P.workspace(E, device=dev)
    P.rlvla_advantages(buf_f, t(traj.last_value), P.adv_params("grpo", group_id=gid, group_size=4,
                       n_env_global=E, cur_version=CUR), adv_f, torch.zeros(E, T, device=dev), st_f, ws_f)
    adv_d = torch.zeros(E_r, T, device=dev)
    st_d = torch.zeros(24, dtype=torch.float64, device=dev)
    P.rlvla_advantages(buf, lv, P.adv_params("grpo", group_id=gid, group_size=4, env_offset=lo,
                                             n_env_global=E, cur_version=CUR), adv_d, ret, st_d, ws,
                       comm=comm)
    assert torch.equal(adv_d.view(torch.int32), adv_f[lo:hi].view(torch.int32)), "GRPO adv not rank-invariant"
    assert torch.equal(st_d[:6], st_f[:6])
    xf = torch.from_numpy(x.astype(np.float32)).to(dev)
    outs = {}
    for name, (bb, aa, xx, ss, cm) in {"full": (buf_f, adv_f, xf, st_f, None),
                                       "shard": (buf, adv_d, xr, st_d, comm)}.items():
        n_ = xx.shape[0]
        lp_, g_ = torch.empty(n_, device=dev), torch.empty(n_, device=dev)
        dx_ = torch.empty_like(xx)
        so = torch.zeros(24, dtype=torch.float64, device=dev)
        fa_ = P.ppo_args(logp_behav=bb.logp_behav.view(-1), adv=aa.view(-1), version=bb.version.view(-1),
                         slot_key=bb.slot_key.view(-1), a_tok=A, cur_version=CUR, adv_stats=ss, out_grad_logp=g_)
        P.rlvla_logprob_fwd_bwd(xx, bb.tokens.view(-1), logp=lp_, fused=fa_, dlogits=dx_, stats=so,
                                ws=ws_f if cm is None else ws, comm=cm)
        outs[name] = (lp_, g_, dx_, so)
    r0, r1 = lo * T * A, hi * T * A
    for k_ in range(3):
        assert torch.equal(outs["full"][k_][r0:r1].view(torch.int32), outs["shard"][k_].view(torch.int32)), k_
    sf, sd = outs["full"][3].cpu().numpy(), outs["shard"][3].cpu().numpy()
    for k_ in range(6, 18):
        assert abs(sf[k_] - sd[k_]) <= 1e-12 * max(1.0, abs(sf[k_])), (k_, sf[k_], sd[k_])
    # NEXT-2 value loss: per-rank steps, explicit global N_v, slots 19..21 allreduced
    from oracle import flow as O_fl
    from oracle import ppo as O_ppo
    rng = np.random.default_rng(100 + rank)
    nv = 3000
    v, vo, Rt = (rng.normal(size=nv).astype(np.float32) for _ in range(3))
    key = np.where(rng.random(nv) < 0.9, 1, 0).astype(np.int64)
    ver = np.full(nv, CUR, np.int32)
    Nv = float(world * nv)
    gv = torch.empty(nv, device=dev)
    st4 = torch.zeros(24, dtype=torch.float64, device=dev)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    P.rlvla_value_loss(cu(v), cu(vo), cu(Rt), cu(key), cu(ver), CUR, gv, clip_eps=0.2, denominator=Nv,
                       stats=st4, ws=ws, comm=comm)
    o = O_ppo.value_loss(v, vo, Rt, key != 0, clip_eps=0.2, n_den=Nv)
    H.assert_close_rel(gv.cpu().numpy(), o["grad"], 1e-5, 1e-9, "value grad")
    rv = torch.tensor([o["stats"]["loss"], float((key != 0).sum())], dtype=torch.float64, device=dev)
    all_reduce(rv)
    s4 = st4.cpu().numpy()
    assert abs(s4[19] - rv[0].item()) <= 1e-5 * abs(rv[0].item()) and s4[21] == rv[1].item()
    # NEXT-4 flow chain + PPO: one ratio per step, C3 over the ranks
    Rf, K, Df = 200, 4, 70
    sig = np.array([0.8, 0.5, 0.3, 0.1], np.float32)
    mu = rng.normal(size=(Rf, K, Df)).astype(np.float32)
    xf = (mu + sig[None, :, None] * rng.normal(size=(Rf, K, Df))).astype(np.float32)
    lp = O_fl.chain_logprob(mu, xf, sigma_k=sig)["logp"]
    lb = (lp - rng.normal(0, 0.05, Rf)).astype(np.float32)
    advf = rng.normal(size=Rf).astype(np.float32)
    Nf = float(world * Rf)
    gf = torch.empty(Rf, device=dev)
    st5 = torch.zeros(24, dtype=torch.float64, device=dev)
    fa = P.ppo_args(logp_behav=cu(lb), adv=cu(advf), version=cu(np.full(Rf, CUR, np.int32)),
                    slot_key=cu(np.ones(Rf, np.int64)), a_tok=1, cur_version=CUR, tok_denominator=Nf,
                    out_grad_logp=gf)
    ch = P.GaussChain(cu(mu), cu(xf), cu(sig))
    P.rlvla_flow_logprob(ch, logp=torch.empty(Rf, device=dev), fused=fa, dmu=torch.empty_like(ch.mu),
                         stats=st5, ws=ws, comm=comm)
    pf = O_ppo.ppo_loss(lp, lb, advf, np.ones(Rf, bool), np.zeros(Rf, int), n_tok=Nf)
    ok = ~pf["near_tie"]
    H.assert_close_rel(gf.cpu().numpy()[ok], pf["grad"][ok], 1e-4, 1e-6, "flow grad")
    rf = torch.tensor([pf["stats"]["loss"], float(Rf)], dtype=torch.float64, device=dev)
    all_reduce(rf)
    s5 = st5.cpu().numpy()
    assert abs(s5[6] - rf[0].item()) <= 1e-4 * max(1e-3, abs(rf[0].item())), (s5[6], rf[0].item())
    assert s5[11] == rf[1].item() and s5[18] == Nf
    # NEXT-2 chunk-level ratio through rlvla_ppo_loss (explicit denominator), C3 over the ranks
    S, A2 = 200, 56
    Rc = S * A2
    lpc = rng.normal(-4, 1, Rc).astype(np.float32)
    lbc = (lpc - rng.normal(0, 0.004, Rc)).astype(np.float32)
    advc = rng.normal(size=S).astype(np.float32)
    gc = torch.empty(Rc, device=dev)
    st6 = torch.zeros(24, dtype=torch.float64, device=dev)
    fa = P.ppo_args(logp_behav=cu(lbc), adv=cu(advc), version=cu(np.full(S, CUR, np.int32)),
                    slot_key=cu(np.ones(S, np.int64)), a_tok=A2, cur_version=CUR, ratio_level=1,
                    tok_denominator=1000.0)
    P.rlvla_ppo_loss(cu(lpc), None, fa, gc, None, st6, ws, comm=comm)
    oc = O_ppo.ppo_loss_chunk(lpc, lbc, advc, np.ones(Rc, bool), np.arange(Rc) // A2, S, n_den=1000.0)
    H.assert_close_rel(gc.cpu().numpy(), oc["grad"], 1e-4, 1e-9, "chunk grad")
    rc = torch.tensor([oc["stats"]["loss"]], dtype=torch.float64, device=dev)
    all_reduce(rc)
    s6 = st6.cpu().numpy()
    assert abs(s6[6] - rc[0].item()) <= 1e-4 * max(1e-3, abs(rc[0].item())), (s6[6], rc[0].item())
    # NEXT-2 chunk ratio with its DEFAULT normaliser: the call's own masked steps over all
    # ranks (it was this rank's count only), then N_LOSS_STEPS of rlvla_advantages
    tc = np.where(rng.random(Rc) < 0.05, -1, 3).astype(np.int32)
    tc[:A2] = -1                                                      # a step without tokens
    gc2 = torch.empty(Rc, device=dev)
    st7 = torch.zeros(24, dtype=torch.float64, device=dev)
    fa = P.ppo_args(logp_behav=cu(lbc), adv=cu(advc), version=cu(np.full(S, CUR, np.int32)),
                    slot_key=cu(np.ones(S, np.int64)), a_tok=A2, cur_version=CUR, ratio_level=1)
    P.rlvla_ppo_loss(cu(lpc), cu(tc), fa, gc2, None, st7, ws, comm=comm)
    mc = tc >= 0
    n_loc = O_ppo.ppo_loss_chunk(lpc, lbc, advc, mc, np.arange(Rc) // A2, S)["stats"]["n_steps"]
    ng = torch.tensor([n_loc], dtype=torch.float64, device=dev)
    all_reduce(ng)
    Ng = float(ng.item())
    oc2 = O_ppo.ppo_loss_chunk(lpc, lbc, advc, mc, np.arange(Rc) // A2, S, n_den=Ng)
    H.assert_close_rel(gc2.cpu().numpy(), oc2["grad"], 1e-4, 1e-9, "chunk grad (global own count)")
    rc2 = torch.tensor([oc2["stats"]["loss"]], dtype=torch.float64, device=dev)
    all_reduce(rc2)
    s7 = st7.cpu().numpy()
    assert s7[18] == Ng, (s7[18], Ng)
    assert abs(s7[6] - rc2.item()) <= 1e-4 * max(1e-3, abs(rc2.item())), (s7[6], rc2.item())
    # ... and N_steps = N_LOSS_STEPS of the buffer's advantages call (global over ranks)
    c_all = torch.tensor([c["n_loss_steps"]], dtype=torch.float64, device=dev)
    all_reduce(c_all)
    assert st[23].item() == c_all.item(), (st[23].item(), c_all.item())
    # NEXT-2 value loss with its own count over all ranks (no explicit N_v)
    gv2 = torch.empty(nv, device=dev)
    st8 = torch.zeros(24, dtype=torch.float64, device=dev)
    P.rlvla_value_loss(cu(v), cu(vo), cu(Rt), cu(key), cu(ver), CUR, gv2, clip_eps=0.2,
                       stats=st8, ws=ws, comm=comm)
    Nv2 = torch.tensor([float((key != 0).sum())], dtype=torch.float64, device=dev)
    all_reduce(Nv2)
    o2 = O_ppo.value_loss(v, vo, Rt, key != 0, clip_eps=0.2, n_den=float(Nv2.item()))
    H.assert_close_rel(gv2.cpu().numpy(), o2["grad"], 1e-5, 1e-9, "value grad (global own count)")
    rv2 = torch.tensor([o2["stats"]["loss"]], dtype=torch.float64, device=dev)
    all_reduce(rv2)
    s8 = st8.cpu().numpy()
    assert s8[22] == Nv2.item() and abs(s8[19] - rv2.item()) <= 1e-5 * abs(rv2.item())
    # a rank with NO rows in a fused call still takes part in C3: rank 0 empty
    xs = xr if rank != 0 else xr[:0]
    n_ = xs.shape[0]
    so = torch.zeros(24, dtype=torch.float64, device=dev)
    fa_ = P.ppo_args(logp_behav=buf.logp_behav.view(-1)[:n_], adv=adv.view(-1), version=buf.version.view(-1),
                     slot_key=buf.slot_key.view(-1), a_tok=A, cur_version=CUR, adv_stats=st,
                     out_grad_logp=torch.empty(n_, device=dev))
    P.rlvla_logprob_fwd_bwd(xs, buf.tokens.view(-1)[:n_], logp=torch.empty(n_, device=dev), fused=fa_,
                            dlogits=torch.empty_like(xs), stats=so, ws=ws, comm=comm)
    tv0 = O_path.token_view(obuf, a_ref, A, CUR)
    mine = O_path.loss_and_grad(x[lo * T * A:hi * T * A], tv0, n_tok=float(tot[1].item()))["stats"]
    re = torch.tensor([0.0 if rank == 0 else mine["loss"], 0.0 if rank == 0 else mine["n_loss_tok"]],
                      dtype=torch.float64, device=dev)
    all_reduce(re)
    so_ = so.cpu().numpy()
    assert abs(so_[6] - re[0].item()) <= 1e-5 * max(1e-3, abs(re[0].item())), (so_[6], re[0].item())
    assert so_[11] == re[1].item()
    dist.barrier()
    if rank == 0:
        nccl = P.rlvla_nccl_version() if MODE == "nccl" else "none"
        print(f"MGPU PARITY OK world={world} mode={MODE} gpus={ndev} nccl={nccl} "
              f"in-kernel-p2p={comm.p2p}", flush=True)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
