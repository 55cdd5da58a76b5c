"""Full-size parity at BASELINE.json config 1 (LIBERO-Spatial OFT: 64 envs x 512 steps,
8x7 chunk, V = 32000 bf16 -> 229,376 rows, 14.7 GB of logits) in the launch configuration
bench.py times (one fused TMA launch over all rows after 64 arrival-chunk scatters and GRPO).

Checked against the oracle on sampled rows the oracle computes one by one, and through
properties that hold at any size: bit-exact scatter (4,096 records, full oracle replay),
advantages (full oracle), every row's dlogits summing to ~0, logp <= 0, statistics equal
to the fp64 sum of the per-row outputs, bit-identical reruns."""
import numpy as np
import pytest
import torch

import synth
from oracle import logprob as O_lp
from oracle import path as O_path
from tests import harness as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def full():
    import paper_2602_05765_b200 as P
    cfg = synth.CONFIGS["libero_spatial_oft"]
    case = H.build_case(cfg, device="cuda", behav_sample=128)
    gbuf, gcnt = H.gpu_scatter(case)
    obuf, ocnt = H.oracle_scatter(case)
    E, T, A, V = cfg.n_env, cfg.t_steps, cfg.a_tok, cfg.vocab
    ws = P.workspace(E)
    stats = torch.zeros(24, dtype=torch.float64, device="cuda")
    adv = torch.zeros(E, T, device="cuda")
    ret = torch.zeros(E, T, device="cuda")
    prm = P.adv_params("grpo", group_id=torch.from_numpy(case.traj.group_id).cuda(), group_size=8,
                       n_env_global=E, cur_version=synth.CUR_VERSION)
    P.rlvla_advantages(gbuf, None, prm, adv, ret, stats, ws)
    R = E * T * A
    logp = torch.empty(R, device="cuda")
    lse = torch.empty(R, device="cuda")
    g = torch.empty(R, device="cuda")
    lt = torch.empty(R, device="cuda")
    dx = torch.empty_like(case.logits)
    st2 = torch.zeros(24, dtype=torch.float64, device="cuda")
    fa = P.ppo_args(logp_behav=gbuf.logp_behav.view(-1), adv=adv.view(-1), version=gbuf.version.view(-1),
                    slot_key=gbuf.slot_key.view(-1), a_tok=A, cur_version=synth.CUR_VERSION,
                    adv_stats=stats, out_grad_logp=g, out_loss_tok=lt)
    P.rlvla_logprob_fwd_bwd(case.logits, gbuf.tokens.view(-1), logp=logp, lse=lse, fused=fa,
                            dlogits=dx, stats=st2, ws=ws)
    torch.cuda.synchronize()
    return dict(case=case, gbuf=gbuf, gcnt=gcnt, obuf=obuf, ocnt=ocnt, adv=adv, stats=stats,
                st2=st2, logp=logp, lse=lse, g=g, lt=lt, dx=dx, P=P, fa=fa, ws=ws)


def test_fullsize_scatter_and_advantages(full):
    gb = H.buf_to_np(full["gbuf"])
    for k, v in full["obuf"].items():
        assert np.array_equal(gb[k].view(np.uint8), v.view(np.uint8)), k
    assert full["gcnt"].cpu().numpy().tolist() == full["ocnt"].tolist()
    oadv = H.oracle_advantages(full["case"], full["obuf"], "grpo")
    H.assert_close_rel(full["adv"].cpu().numpy(), oadv["adv"], 1e-5, 1e-3, "adv")
    assert full["stats"][3].item() == oadv["counts"]["n_tok"]


def test_fullsize_sampled_rows_match_oracle(full):
    """Sampled rows of the bench's launch vs the oracle chain: the GPU ran on its own
    advantages and N_tok, the oracle on its own (S2's tolerance propagated into S3/S4 as in
    tests/test_parity_path.py; nothing crosses between the chains)."""
    from tests.test_parity_path import _compare_rows
    case = full["case"]
    cfg = case.cfg
    A = cfg.a_tok
    rng = np.random.default_rng(0)
    crafted = np.concatenate([np.asarray(v) for v in case.traj.crafted.values()])
    rows = np.unique(np.concatenate([rng.choice(full["dx"].shape[0], 1024, replace=False), crafted,
                                     np.asarray(case.extra["behav_rows"][:256])]))
    oadv = H.oracle_advantages(case, full["obuf"], "grpo")
    floor = max(1e-3, float(np.sqrt(np.mean(oadv["adv"] ** 2))))
    tol_tok = np.repeat((1e-5 * np.maximum(np.abs(oadv["adv"]), floor)).reshape(-1), A)
    tv = O_path.token_view(full["obuf"], oadv["adv"], A, synth.CUR_VERSION)
    out = {k: full[k].cpu().numpy() for k in ("logp", "lse", "g", "lt")}
    out["dx"] = full["dx"]
    n_tok = float(oadv["counts"]["n_tok"])
    assert full["stats"][3].item() == n_tok
    for s in range(0, len(rows), 512):
        rr = rows[s:s + 512]
        _compare_rows(case, out, tv, rr, n_tok, tol_tok[rr])


def test_fullsize_properties(full):
    dx = full["dx"]
    R = dx.shape[0]
    # every row's gradient sums to ~0 (sum_j (1[j=a] - p_j) = 0): each element carries at
    # most half a bf16 ulp (2^-9 relative) of rounding
    s = torch.zeros(R, dtype=torch.float64, device="cuda")
    sa = torch.zeros(R, dtype=torch.float64, device="cuda")
    for r0 in range(0, R, 16384):
        blk = dx[r0:r0 + 16384].double()
        s[r0:r0 + 16384] = blk.sum(dim=1)
        sa[r0:r0 + 16384] = blk.abs().sum(dim=1)
    assert torch.all(s.abs() <= 2.0 ** -8 * sa + 1e-30).item()
    logp = full["logp"]
    assert torch.all(logp <= 1e-6).item()
    # statistics = fp64 sums of the per-row outputs
    st = full["st2"].cpu().numpy()
    N = full["stats"][3].item()
    lt = full["lt"].double().sum().item()
    assert abs(st[6] - lt / N) <= 1e-9 * max(1.0, abs(lt / N)) + 1e-12
    assert st[18] == N
    mask = full["g"] != 0
    assert st[11] >= mask.sum().item()


def test_fullsize_rerun_bit_identical(full):
    P = full["P"]
    case = full["case"]
    dx2 = torch.empty_like(full["dx"])
    logp2 = torch.empty_like(full["logp"])
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    P.rlvla_logprob_fwd_bwd(case.logits, full["gbuf"].tokens.view(-1), logp=logp2, fused=full["fa"],
                            dlogits=dx2, stats=st, ws=full["ws"])
    torch.cuda.synchronize()
    assert torch.equal(dx2, full["dx"]) and torch.equal(logp2, full["logp"])
    assert torch.equal(st, full["st2"])


def test_fullsize_flow_sampled_rows():
    """NEXT-4 at the prof_flow.py launch size (196,608 pi_0 decision steps, K 4 x D 70,
    bf16 means, fused PPO + backward): sampled steps against the oracle, every step's
    gradient row consistent with its own g (dmu * sigma^2 / (x - mu) == g), stats = fp64 sum
    of the per-step outputs."""
    import paper_2602_05765_b200 as P
    from oracle import flow as O_fl
    from oracle import ppo as O_ppo
    R, K, D = 196608, 4, 70
    g0 = torch.Generator(device="cuda").manual_seed(5)
    sig = torch.tensor([0.8, 0.5, 0.3, 0.1], device="cuda")
    mu = torch.randn(R, K, D, generator=g0, device="cuda").to(torch.bfloat16)
    x = (mu.float() + sig.view(1, K, 1) * torch.randn(R, K, D, generator=g0, device="cuda")).contiguous()
    ch = P.GaussChain(mu, x, sig)
    lp0 = torch.empty(R, device="cuda")
    P.rlvla_flow_logprob(ch, logp=lp0)
    lb = (lp0 + 0.05 * torch.randn(R, generator=g0, device="cuda")).contiguous()
    adv = torch.randn(R, generator=g0, device="cuda")
    ver = torch.full((R,), 100, dtype=torch.int32, device="cuda")
    key = torch.ones(R, dtype=torch.int64, device="cuda")
    g = torch.empty(R, device="cuda")
    fa = P.ppo_args(logp_behav=lb, adv=adv, version=ver, slot_key=key, a_tok=1, cur_version=100,
                    tok_denominator=float(R), out_grad_logp=g)
    logp = torch.empty(R, device="cuda")
    dmu = torch.empty_like(mu)
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    P.rlvla_flow_logprob(ch, logp=logp, fused=fa, dmu=dmu, stats=st, ws=P.workspace(1))
    torch.cuda.synchronize()
    assert torch.equal(logp, lp0)                                   # same sums in both modes
    rows = np.random.default_rng(0).choice(R, 256, replace=False)
    rt = torch.from_numpy(rows).cuda()
    mu64 = mu[rt].double().cpu().numpy()
    x64 = x[rt].double().cpu().numpy()
    o = O_fl.chain_logprob(mu64, x64, sigma_k=sig.cpu().numpy())
    es = (0.5 * o["z"] ** 2 + np.abs(np.log(sig.cpu().numpy().astype(np.float64)))[None, :, None] + 1.0).sum(axis=(1, 2))
    H.assert_close_rel(logp[rt].cpu().numpy(), o["logp"], 2e-7, es, "logp (sampled)")
    p = O_ppo.ppo_loss(o["logp"], lb[rt].double().cpu().numpy(), adv[rt].double().cpu().numpy(),
                       np.ones(256, bool), np.zeros(256, int), n_tok=float(R))
    ok = ~p["near_tie"]
    sens = np.abs(adv[rt].double().cpu().numpy()) * p["ratio"]
    H.assert_close_rel(g[rt].cpu().numpy()[ok], p["grad"][ok], 1e-5, (sens * 2e-7 * es / R / 1e-5)[ok] + 1e-12, "g")
    gr = O_fl.chain_grads(mu64, x64, g[rt].double().cpu().numpy(), sigma_k=sig.cpu().numpy())
    bits = dmu[rt].view(torch.int16).cpu().numpy().astype(np.int32) & 0xFFFF
    H.assert_bf16_ulp(bits, gr["dmu"], 1)
    # statistics = fp64 sums of the per-step outputs
    s = st.cpu().numpy()
    assert s[11] == R and s[18] == R
    assert abs(s[14] - logp.double().sum().item()) <= 1e-6 * logp.double().abs().sum().item()


def test_fullsize_batcher_oft_gather():
    """NEXT-3 at OFT observation size with 1,024 envs: 16 rounds of 64-request offers in a
    random order and firing polls; every batch is the FIFO block and its bytes the slots'."""
    import paper_2602_05765_b200 as P
    from oracle import batcher as O_b
    E, ob, B = 1024, synth.OBS_BYTES_OFT, 64
    q = P.BatchQueue.allocate(E, ob)
    g0 = torch.Generator(device="cuda").manual_seed(8)
    q.obs.copy_(torch.randint(0, 256, (E, ob), generator=g0, device="cuda", dtype=torch.uint8))
    ws = P.workspace(1)
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    out_env = torch.empty(B, dtype=torch.int32, device="cuda")
    out_time = torch.empty(B, dtype=torch.int64, device="cuda")
    out_n = torch.empty(1, dtype=torch.int32, device="cuda")
    out_obs = torch.empty(B, ob, dtype=torch.uint8, device="cuda")
    bt = O_b.Batcher(E)
    order = np.random.default_rng(9).permutation(E)
    for k in range(16):
        env = order[k * B:(k + 1) * B].astype(np.int32)
        now = 10 * k
        P.rlvla_batch_offer(q, torch.from_numpy(env).cuda(), torch.full((B,), now, dtype=torch.int64, device="cuda"),
                            now, cnt, ws=ws)
        bt.offer(env, [now] * B, now)
        P.rlvla_batch_poll(q, now, B, 5, out_env, out_time, out_n, out_obs=out_obs, ws=ws)
        exp = bt.poll(now, B, 5)
        assert int(out_n.item()) == len(exp) == B
        assert out_env.cpu().tolist() == [e for e, _ in exp]
        assert torch.equal(out_obs, q.obs[out_env.long()])
    assert cnt.cpu().tolist() == bt.counters.tolist()


@pytest.mark.parametrize("name", ["libero10_long", "maniskill_ppo_gae", "grpo_span"])
def test_fullsize_microbatched_configs(name):
    """BASELINE.json configs 2-4 at full size in the launch configuration bench.py times on
    one GPU (e.g. LIBERO-10: 256 envs x 128 decision steps, 1.8 M logit rows): every
    arrival-chunk scatter, the advantages over the full buffer (GAE + global whitening, or
    GRPO with interleaved groups; compared with the oracle in full), then the fused S3+S4
    call on micro-batches of <= 131,072 rows — the first and the ragged last one — with
    logits generated per micro-batch, sampled rows against the oracle."""
    import paper_2602_05765_b200 as P
    cfg = synth.CONFIGS[name]
    E, T, A, V = cfg.n_env, cfg.t_steps, cfg.a_tok, cfg.vocab
    traj = synth.make_trajectories(cfg)
    rec = synth.make_records(traj, 0, E)
    rows_of = synth.record_rows(rec, cfg, E)                       # [M, A] logit rows
    env_rows = T * A
    mb_envs = 131072 // env_rows
    mbs = [(e0, min(E, e0 + mb_envs)) for e0 in range(0, E, mb_envs)]
    tested = [mbs[0], mbs[-1]]
    rng = np.random.default_rng(11)
    # behaviour log-probs: oracle logp + noise for the sampled rows' records, synthetic elsewhere
    lb = (-3.0 + 0.5 * rng.standard_normal(rec.behav_noise.shape)).astype(np.float32)
    samples = {}
    for e0, e1 in tested:
        lo, hi = e0 * env_rows, e1 * env_rows
        pick = rng.choice(np.arange(lo, hi), 96, replace=False)
        samples[(e0, e1)] = np.sort(pick)
        x = synth.gen_logits(cfg, traj, e0, e1, device="cuda")[torch.from_numpy(pick - lo).cuda()].double().cpu().numpy()
        for k, r in enumerate(pick):
            m, a = np.argwhere(rows_of == r)[0] if (rows_of == r).any() else (None, None)
            if m is None:
                continue
            f = O_lp.log_softmax_gather(x[k:k + 1], rec.tokens[m, a:a + 1])
            if np.isfinite(f["logp"][0]):
                lb[m, a] = np.float32(f["logp"][0] + rec.behav_noise[m, a])
    case = H.Case(cfg, traj, 0, E, rec, lb, None)
    gbuf, gcnt = H.gpu_scatter(case)
    obuf, ocnt = H.oracle_scatter(case)
    assert gcnt.cpu().numpy().tolist() == ocnt.tolist()
    ws = P.workspace(E)
    stats = torch.zeros(24, dtype=torch.float64, device="cuda")
    adv = torch.zeros(E, T, device="cuda")
    ret = torch.zeros(E, T, device="cuda")
    if cfg.adv_mode == "grpo":
        prm = P.adv_params("grpo", group_id=torch.from_numpy(traj.group_id).cuda(),
                           group_size=cfg.group_size, n_env_global=E, cur_version=synth.CUR_VERSION)
        P.rlvla_advantages(gbuf, None, prm, adv, ret, stats, ws)
        oadv = H.oracle_advantages(case, obuf, "grpo")
        H.assert_close_rel(adv.cpu().numpy(), oadv["adv"], 1e-5, 1e-3, "adv (grpo)")
    else:
        prm = P.adv_params("gae", gamma=0.99, lam=0.95, whiten=cfg.whiten, n_env_global=E,
                           cur_version=synth.CUR_VERSION)
        P.rlvla_advantages(gbuf, torch.from_numpy(traj.last_value).cuda(), prm, adv, ret, stats, ws)
        oadv = H.oracle_advantages(case, obuf, "gae", whiten=cfg.whiten)
        H.assert_close_rel(adv.cpu().numpy(), oadv["adv"], 1e-5, 1.0, "adv (gae)")
    assert stats[3].item() == oadv["counts"]["n_tok"]
    # the GPU chain runs on its own advantages and N_tok, the oracle chain on its own (S2's
    # tolerance propagated as in tests/test_parity_path.py)
    from tests.test_parity_path import check_rows
    floor = max(1e-3, float(np.sqrt(np.mean(oadv["adv"] ** 2))))
    tol_tok = np.repeat((1e-5 * np.maximum(np.abs(oadv["adv"]), floor)).reshape(-1), A)
    tv = O_path.token_view(obuf, oadv["adv"], A, synth.CUR_VERSION)
    N = float(oadv["counts"]["n_tok"])
    for e0, e1 in tested:
        lo, hi = e0 * env_rows, e1 * env_rows
        xmb = synth.gen_logits(cfg, traj, e0, e1, device="cuda")
        n = hi - lo
        logp = torch.empty(n, device="cuda")
        g = torch.empty(n, device="cuda")
        dx = torch.empty_like(xmb)
        st = torch.zeros(24, dtype=torch.float64, device="cuda")
        s0, s1 = lo // A, hi // A
        fa = P.ppo_args(logp_behav=gbuf.logp_behav.view(-1)[lo:hi], adv=adv.view(-1)[s0:s1],
                        version=gbuf.version.view(-1)[s0:s1], slot_key=gbuf.slot_key.view(-1)[s0:s1],
                        a_tok=A, cur_version=synth.CUR_VERSION, adv_stats=stats, out_grad_logp=g)
        P.rlvla_logprob_fwd_bwd(xmb, gbuf.tokens.view(-1)[lo:hi], logp=logp, fused=fa, dlogits=dx,
                                stats=st, ws=ws)
        torch.cuda.synchronize()
        rows = samples[(e0, e1)]
        li = torch.from_numpy(rows - lo).cuda()
        x = xmb[li].double().cpu().numpy()
        check_rows(x, dict(logp=logp.cpu().numpy()[rows - lo], g=g.cpu().numpy()[rows - lo], dx=dx[li]),
                   tv, rows, N, tol_tok[rows], xmb.dtype)
        # the call's token count = the oracle's masked tokens of this micro-batch
        allr = np.arange(lo, hi)
        base = tv["valid"][allr] & (tv["target"][allr] >= 0) & (tv["lag"][allr] >= 0) & (tv["lag"][allr] <= 1)
        assert st.cpu().numpy()[11] == base.sum() - 0  # no non-finite logits in these envs
        assert st.cpu().numpy()[18] == N
        del xmb, dx
        torch.cuda.empty_cache()
