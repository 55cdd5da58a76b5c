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
    case = full["case"]
    cfg = case.cfg
    A = cfg.a_tok
    rng = np.random.default_rng(0)
    crafted = np.concatenate([np.asarray(v) for v in case.traj.crafted.values()])
    rows = np.unique(np.concatenate([rng.choice(full["dx"].shape[0], 1024, replace=False), crafted,
                                     np.asarray(case.extra["behav_rows"][:256])]))
    oadv = H.oracle_advantages(case, full["obuf"], "grpo")
    a32 = full["adv"].cpu().numpy().astype(np.float64)   # S4 compared on the GPU's own adv,
    H.assert_close_rel(a32, oadv["adv"], 1e-5, 1e-3, "adv")  # which matched the oracle above
    tv = O_path.token_view(full["obuf"], a32, A, synth.CUR_VERSION)
    x = case.logits[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    ref = O_path.loss_and_grad(x, tv, n_tok=full["stats"][3].item(), rows=rows)
    H.assert_close_rel(full["logp"].cpu().numpy()[rows], ref["fwd"]["logp"], 1e-5, 1.0, "logp")
    nt = ref["ppo"]["near_tie"]
    H.assert_close_rel(full["g"].cpu().numpy()[rows][~nt], ref["ppo"]["grad"][~nt], 1e-5, 1e-9, "grad")
    bits = full["dx"][torch.from_numpy(rows).cuda()].view(torch.int16).cpu().numpy().astype(np.int32) & 0xFFFF
    H.assert_bf16_ulp(bits[~nt], ref["dx"][~nt], 1)


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
