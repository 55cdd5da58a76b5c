"""GPU parity for S1 (bit-exact buffer + counters) and S2 (GAE / GRPO) beyond the tiny
path test: multi-CTA scatter (M > 1024), chunk sizes, resends, long horizons (T=1024,
chunk 1), ragged T, done patterns, whitening, population std, contiguous groups."""
import numpy as np
import pytest
import torch

import synth
from oracle import advantages as O_adv
from oracle import path as O_path
from tests import harness as H

pytestmark = pytest.mark.gpu


def _P():
    import paper_2602_05765_b200 as P
    return P


@pytest.mark.parametrize("chunk", [1, 64, 1000, 5000])
def test_scatter_bit_exact_chunks(chunk):
    cfg = synth.scaled(synth.CONFIGS["tiny"], n_env=40, n_es=96, faults=True)
    case = H.build_case(cfg, device="cpu")
    # heavy resend traffic: append a shuffled copy of a third of the stream with new payloads
    rng = np.random.default_rng(0)
    idx = rng.choice(case.rec.n, size=case.rec.n // 3, replace=False)
    extra = case.rec.take(idx)
    extra.reward = extra.reward + np.float32(1.5)
    extra.version = extra.version - rng.integers(0, 2, size=len(idx)).astype(np.int32)
    case.rec = synth.Records(*(np.concatenate([getattr(case.rec, f), getattr(extra, f)])
                               for f in ("env_id", "step", "version", "reward", "done", "value",
                                         "tokens", "behav_noise", "fault")))
    case.logp_behav = np.concatenate([case.logp_behav, case.logp_behav[idx] + np.float32(0.5)])
    gbuf, gcnt = H.gpu_scatter(case, chunk=chunk)
    obuf, ocnt = H.oracle_scatter(case, chunk=chunk)
    gb = H.buf_to_np(gbuf)
    for k in obuf:
        assert np.array_equal(gb[k].view(np.uint8), obuf[k].view(np.uint8)), k
    assert gcnt.cpu().numpy().tolist() == ocnt.tolist()
    assert ocnt[2] > 0 and ocnt[0] > 0 and ocnt[1] > 0


def _gae_case(T, E, seed, done_p, valid_p):
    rng = np.random.default_rng(seed)
    reward = rng.normal(size=(E, T)).astype(np.float32)
    value = rng.normal(size=(E, T)).astype(np.float32)
    done = (rng.random((E, T)) < done_p).astype(np.uint8)
    valid = rng.random((E, T)) < valid_p
    ver = (100 - rng.integers(0, 3, size=(E, T))).astype(np.int32)
    tokens = rng.integers(-1, 50, size=(E, T, 3)).astype(np.int32)
    lv = rng.normal(size=E).astype(np.float32)
    tokens[rng.random((E, T)) < 0.03] = -1       # steps without a usable token (N_LOSS_STEPS)
    return reward, value, done, valid, ver, tokens, lv


def _gpu_buffer(reward, value, done, valid, ver, tokens):
    P = _P()
    E, T = reward.shape
    buf = P.TrajectoryBuffer.allocate(E, T, tokens.shape[2])
    buf.reward.copy_(torch.from_numpy(reward))
    buf.value.copy_(torch.from_numpy(value))
    buf.done.copy_(torch.from_numpy(done))
    buf.version.copy_(torch.from_numpy(ver))
    buf.tokens.copy_(torch.from_numpy(tokens))
    buf.slot_key.copy_(torch.from_numpy(np.where(valid, 5, 0).astype(np.int64)))
    return buf


@pytest.mark.parametrize("T,E,done_p,valid_p,whiten", [
    (1, 5, 0.3, 1.0, False), (31, 9, 0.1, 0.9, False), (64, 64, 0.02, 1.0, True),
    (80, 128, 0.05, 0.97, True), (1024, 16, 0.004, 0.999, True), (1000, 7, 0.5, 0.5, False)])
@pytest.mark.parametrize("gamma,lam", [(0.99, 0.95), (1.0, 1.0), (0.9, 0.0)])
def test_gae_matches_oracle(T, E, done_p, valid_p, whiten, gamma, lam):
    P = _P()
    reward, value, done, valid, ver, tokens, lv = _gae_case(T, E, T * 7 + E, done_p, valid_p)
    buf = _gpu_buffer(reward, value, done, valid, ver, tokens)
    adv = torch.zeros(E, T, device="cuda")
    ret = torch.zeros(E, T, device="cuda")
    stats = torch.zeros(24, dtype=torch.float64, device="cuda")
    prm = P.adv_params("gae", gamma=gamma, lam=lam, whiten=whiten, n_env_global=E,
                       cur_version=100, max_staleness=1)
    P.rlvla_advantages(buf, torch.from_numpy(lv).cuda(), prm, adv, ret, stats, P.workspace(E))
    a, r = O_adv.gae(reward, value, done, valid, lv, gamma, lam)
    n, s1, s2 = O_adv.whiten_stats(a, valid)
    st = stats.cpu().numpy()
    assert st[0] == n
    assert abs(st[1] - s1) <= 1e-5 * max(1.0, np.abs(a).sum())
    assert abs(st[2] - s2) <= 1e-5 * max(1.0, s2)
    c = O_adv.step_counts(valid, ver, tokens, 100, 1)
    assert (st[3], st[4], st[5], st[23]) == (c["n_tok"], c["n_stale"], c["n_bad"], c["n_loss_steps"])
    if whiten:
        a = O_adv.whiten(a, valid, 1e-8)
    floor = max(1e-3, float(np.sqrt(np.mean(a ** 2))))
    H.assert_close_rel(adv.cpu().numpy(), a, 1e-5, floor, "adv")
    H.assert_close_rel(ret.cpu().numpy(), r, 1e-5, max(1e-3, float(np.sqrt(np.mean(r ** 2)))), "ret")


@pytest.mark.parametrize("E,G,explicit,unbiased", [(8, 4, True, True), (8, 4, False, False),
                                                   (2048, 8, True, True), (96, 3, False, True),
                                                   (33, 33, False, True)])
def test_grpo_matches_oracle(E, G, explicit, unbiased):
    P = _P()
    T = 40
    rng = np.random.default_rng(E + G)
    reward = (rng.random((E, T)) < 0.02).astype(np.float32)
    reward[: E // 4] = 0.0                     # some all-zero envs -> equal groups
    valid = rng.random((E, T)) < 0.97
    value = np.zeros((E, T), np.float32)
    done = np.zeros((E, T), np.uint8)
    ver = np.full((E, T), 100, np.int32)
    tokens = np.zeros((E, T, 2), np.int32)
    buf = _gpu_buffer(reward, value, done, valid, ver, tokens)
    gid = (np.arange(E) % (E // G)) if explicit else (np.arange(E) // G)
    adv = torch.zeros(E, T, device="cuda")
    ret = torch.zeros(E, T, device="cuda")
    stats = torch.zeros(24, dtype=torch.float64, device="cuda")
    prm = P.adv_params("grpo", group_id=torch.from_numpy(gid.astype(np.int32)).cuda() if explicit else None,
                       group_size=G, std_unbiased=unbiased, n_env_global=E, cur_version=100)
    P.rlvla_advantages(buf, None, prm, adv, ret, stats, P.workspace(E))
    c = O_adv.step_counts(valid, ver, tokens, 100, 1)
    st = stats.cpu().numpy()
    assert (st[0], st[3], st[23]) == (c["n_valid"], c["n_tok"], c["n_loss_steps"])
    R = O_adv.episode_return(reward, valid)
    A = O_adv.grpo_step_adv(O_adv.grpo(R, gid, 1e-6, unbiased), valid)
    H.assert_close_rel(adv.cpu().numpy(), A, 1e-5, 1e-3, "grpo adv")
    H.assert_close_rel(ret.cpu().numpy(), O_adv.grpo_step_adv(R, valid), 1e-6, 1e-3, "grpo R")
    # all-equal groups give exactly 0
    Rg = R.reshape(-1)
    for g in np.unique(gid):
        m = gid == g
        if np.all(Rg[m] == Rg[m][0]):
            assert np.all(adv.cpu().numpy()[m] == 0.0)


def test_advantages_deterministic():
    P = _P()
    reward, value, done, valid, ver, tokens, lv = _gae_case(512, 256, 3, 0.01, 0.99)
    buf = _gpu_buffer(reward, value, done, valid, ver, tokens)
    outs = []
    ws = P.workspace(256)
    for _ in range(3):
        adv = torch.zeros(256, 512, device="cuda")
        ret = torch.zeros(256, 512, device="cuda")
        st = torch.zeros(24, dtype=torch.float64, device="cuda")
        P.rlvla_advantages(buf, torch.from_numpy(lv).cuda(),
                           P.adv_params("gae", whiten=True, n_env_global=256, cur_version=100),
                           adv, ret, st, ws)
        outs.append((adv, ret, st))
    for o in outs[1:]:
        assert all(torch.equal(a, b) for a, b in zip(o, outs[0]))


def test_gae_token_count_multipass():
    """Loss-token count when the token sweep needs several grid passes and ends ragged:
    512 x 300 x 9 = 1,382,400 tokens > 8 CTAs/SM x 256 threads x 4 tokens per pass,
    negative targets and stale/bad versions mixed in (oracle step_counts)."""
    P = _P()
    reward, value, done, valid, ver, _, lv = _gae_case(300, 512, 11, 0.01, 0.95)
    rng = np.random.default_rng(12)
    tokens = rng.integers(-2, 40, size=(512, 300, 9)).astype(np.int32)
    tokens[rng.random((512, 300)) < 0.05] = -1             # steps without a usable token
    tokens[rng.random((512, 300)) < 0.05, :5] = -1         # ... or whose first 5 are ignored
    ver = (100 - rng.integers(-1, 4, size=(512, 300))).astype(np.int32)
    buf = _gpu_buffer(reward, value, done, valid, ver, tokens)
    adv = torch.zeros(512, 300, device="cuda")
    ret = torch.zeros(512, 300, device="cuda")
    stats = torch.zeros(24, dtype=torch.float64, device="cuda")
    prm = P.adv_params("gae", n_env_global=512, cur_version=100, max_staleness=1)
    P.rlvla_advantages(buf, torch.from_numpy(lv).cuda(), prm, adv, ret, stats, P.workspace(512))
    st = stats.cpu().numpy()
    c = O_adv.step_counts(valid, ver, tokens, 100, 1)
    assert (st[3], st[4], st[5], st[23]) == (c["n_tok"], c["n_stale"], c["n_bad"], c["n_loss_steps"])
    a, _ = O_adv.gae(reward, value, done, valid, lv, 0.99, 0.95)
    H.assert_close_rel(adv.cpu().numpy(), a, 1e-5, max(1e-3, float(np.sqrt(np.mean(a ** 2)))), "adv")
