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
    adv = torch.from_numpy(oadv["adv"].astype(np.float32)).cuda()
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
    tv = O_path.token_view(obuf, oadv["adv"].astype(np.float32).astype(np.float64), A, synth.CUR_VERSION)
    tot = {}
    for s in range(0, R, 2048):
        rr = np.arange(s, min(R, s + 2048))
        ref = O_path.loss_and_grad(x[torch.from_numpy(rr).cuda()].double().cpu().numpy(), tv,
                                   n_tok=N, rows=rr)["stats"]
        for k, v in ref.items():
            tot[k] = tot.get(k, 0.0) + v
    assert abs(b[6] - tot["loss"]) <= 1e-5 * max(1e-3, abs(tot["loss"]))
    assert b[11] == tot["n_loss_tok"]
