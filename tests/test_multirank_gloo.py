"""World-size 2 and 8 (gloo, CPU) tests of the data-parallel sharding the C ABI implements
over NVLink / NCCL: contiguous env shards, records routed to their owner rank, C1
(advantage-statistics allreduce), C2 (GRPO returns allgather, groups spanning ranks), C3
(loss-statistics allreduce). The sharded computation (oracle arithmetic + host sharding
helpers + the collectives) must equal the unsharded one. Cases: tiny at world 2, and the
shapes of BASELINE configs 4 (ManiSkill PPO+GAE with whitening, 8 ranks) and 5 (GRPO groups
of 8 interleaved so every group has one member on each of the 8 ranks) with a small
vocabulary so the oracle finishes in seconds."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import advantages as O_adv
from oracle import path as O_path
from oracle import scatter as O_sc
from paper_2602_05765_b200 import sharding

CASES = {
    "tiny_w2": (2, lambda: synth.scaled(synth.CONFIGS["tiny"], n_env=16, group_size=4,
                                        interleave_groups=True, faults=False)),
    # config 4 shape: 1024 envs x 80 steps, chunk 8 -> 8 envs per rank x 10 steps x 56 tokens
    "maniskill_w8": (8, lambda: synth.scaled(synth.CONFIGS["maniskill_ppo_gae"], n_env=64,
                                             vocab=64, dtype="f32")),
    # config 5 shape: GRPO groups of 8 spanning all 8 ranks (g(e) = e mod E/G)
    "grpo_span_w8": (8, lambda: synth.scaled(synth.CONFIGS["grpo_span"], n_env=64, n_es=32,
                                             vocab=64, dtype="f32")),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(name):
    cfg = CASES[name][1]()
    traj = synth.make_trajectories(cfg)
    rec = synth.make_records(traj, 0, cfg.n_env)         # global env ids, arrival order
    x = synth.gen_logits(cfg, traj, 0, cfg.n_env).double().numpy()
    return cfg, traj, rec, x


def _recs(rec, idx, local_env, lb):
    return dict(env_id=local_env, step=rec.step[idx], version=rec.version[idx],
                reward=rec.reward[idx], done=rec.done[idx], value=rec.value[idx],
                tokens=rec.tokens[idx], logp_behav=lb[idx])


def _pipeline(cfg, traj, rec, x, lo, hi, idx, local_env, allreduce, allgather):
    """One rank's path: scatter own records, advantages with C1/C2, loss with C3."""
    T, A = cfg.t_steps, cfg.a_tok
    E_r = hi - lo
    lb = (rec.behav_noise - 2.0).astype(np.float32)
    buf = O_sc.new_buffer(E_r, T, A)
    r = _recs(rec, idx, local_env, lb)
    O_sc.scatter_steps(buf, r, synth.CUR_VERSION, 1)
    valid = buf["slot_key"] != 0
    # S2 GRPO with groups spanning ranks: local returns -> allgather (C2)
    R_loc = O_adv.episode_return(buf["reward"], valid)
    R_glob = allgather(R_loc)
    A_grpo = O_adv.grpo_step_adv(O_adv.grpo(R_glob, traj.group_id)[lo:hi], valid)
    adv_loss = A_grpo if cfg.adv_mode == "grpo" else None
    # S2 GAE + global whitening: (n, sum A, sum A^2) allreduce (C1)
    a_gae, _ = O_adv.gae(buf["reward"], buf["value"], buf["done"], valid,
                         traj.last_value[lo:hi], 0.99, 0.95)
    st = allreduce(np.array(O_adv.whiten_stats(a_gae, valid)))
    a_w = O_adv.whiten(a_gae, valid, 1e-8, stats=tuple(st))
    c = O_adv.step_counts(valid, buf["version"], buf["tokens"], synth.CUR_VERSION, 1)
    n_tok = allreduce(np.array([c["n_tok"]], np.float64))[0]
    # S3+S4 on own rows with the global N_tok (the config's advantages); loss stats (C3)
    tv = O_path.token_view(buf, a_w if adv_loss is None else adv_loss, A, synth.CUR_VERSION)
    rows = np.arange(E_r * T * A)
    out = O_path.loss_and_grad(x[lo * T * A:hi * T * A], tv, n_tok=n_tok, rows=rows)
    keys = ["loss", "n_clipped", "kl_k3_sum", "entropy_sum", "ratio_sum", "n_loss_tok"]
    loss = allreduce(np.array([out["stats"][k] for k in keys]))
    return dict(grpo=A_grpo, gae_w=a_w, n_tok=n_tok, loss=loss, dx=out["dx"], buf=buf)


def _worker(rank, port, q, name):
    WORLD = CASES[name][0]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        cfg, traj, rec, x = _case(name)
        lo, hi = sharding.env_range(cfg.n_env, WORLD, rank)
        idx, local_env = sharding.route_records(rec.env_id, cfg.n_env, WORLD, rank)

        def allreduce(v):
            t = torch.from_numpy(np.asarray(v, np.float64).copy())
            dist.all_reduce(t)
            return t.numpy()

        def allgather(v):
            t = torch.from_numpy(np.asarray(v, np.float64).copy())
            parts = [torch.zeros_like(t) for _ in range(WORLD)]
            dist.all_gather(parts, t)
            return torch.cat(parts).numpy()

        out = _pipeline(cfg, traj, rec, x, lo, hi, idx, local_env, allreduce, allgather)
        q.put((rank, {k: out[k] for k in ("grpo", "gae_w", "n_tok", "loss", "dx")}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", list(CASES))
def test_sharded_equals_unsharded(name):
    WORLD = CASES[name][0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, name)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, traj, rec, x = _case(name)
    ident = lambda v: np.asarray(v, np.float64)  # noqa: E731
    full = _pipeline(cfg, traj, rec, x, 0, cfg.n_env, np.arange(rec.n), rec.env_id, ident, ident)
    E_r = cfg.n_env // WORLD
    T, A = cfg.t_steps, cfg.a_tok
    for r in range(WORLD):
        sl = slice(r * E_r, (r + 1) * E_r)
        np.testing.assert_allclose(res[r]["grpo"], full["grpo"][sl], rtol=0, atol=1e-12)
        np.testing.assert_allclose(res[r]["gae_w"], full["gae_w"][sl], rtol=1e-12, atol=1e-12)
        assert res[r]["n_tok"] == full["n_tok"]
        np.testing.assert_allclose(res[r]["loss"], full["loss"], rtol=1e-12, atol=1e-15)
        dx_full = full["dx"][r * E_r * T * A:(r + 1) * E_r * T * A]
        if cfg.adv_mode == "grpo":      # rank-invariant advantages => bit-identical rows
            np.testing.assert_array_equal(res[r]["dx"], dx_full)
        else:                           # whitened: (mu, sigma) differ by the sum order
            np.testing.assert_allclose(res[r]["dx"], dx_full, rtol=1e-12, atol=1e-300)
    # groups really span the ranks (GRPO configs)
    if cfg.group_size:
        g = traj.group_id
        assert all(len({e // E_r for e in np.nonzero(g == k)[0]}) == min(WORLD, cfg.group_size)
                   for k in np.unique(g))


def test_route_records_partitions_stream():
    E, P = 12, 3
    env = np.array([0, 5, 11, -1, 4, 12, 7, 8, 3])
    seen = []
    for r in range(P):
        idx, loc = sharding.route_records(env, E, P, r)
        lo, hi = sharding.env_range(E, P, r)
        for i, l in zip(idx, loc):
            if 0 <= env[i] < E:
                assert lo <= env[i] < hi and l == env[i] - lo
        seen += list(idx)
    assert sorted(seen) == list(range(len(env)))   # every record exactly once (OOB on rank 0)
    with pytest.raises(ValueError):
        sharding.env_range(10, 3, 0)
