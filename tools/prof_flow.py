"""Time the NEXT-4 flow-policy chain log-likelihood fused with PPO (rlvla_flow_logprob) at
pi_0 LIBERO shape (Table 2 setup A: 4 denoising steps, chunk 10 x 7-DoF = 70 dims; 128 envs
x 48 decision steps x 4 rollout epochs = 24,576 decision steps per update).

  python tools/prof_flow.py [--rows R] [--K 4] [--D 70] [--iters N] [--learned] [--f32]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_05765_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=24576)
    ap.add_argument("--K", type=int, default=4)
    ap.add_argument("--D", type=int, default=70)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--learned", action="store_true", help="learned ln sigma (+ its gradient)")
    ap.add_argument("--f32", action="store_true", help="fp32 means (default bf16)")
    ap.add_argument("--no-stats", action="store_true", help="no loss statistics (no last-CTA reduction)")
    ap.add_argument("--fwd", action="store_true", help="chain log-likelihood only (no PPO, no backward)")
    a = ap.parse_args()
    R, K, D = a.rows, a.K, a.D
    g = torch.Generator(device="cuda").manual_seed(0)
    mdt = torch.float32 if a.f32 else torch.bfloat16
    mu = torch.randn(R, K, D, generator=g, device="cuda").to(mdt)
    sig = torch.tensor([0.8, 0.5, 0.3, 0.1][:K], device="cuda")
    ls = (torch.randn(R, K, D, generator=g, device="cuda") * 0.3 - 1.2) if a.learned else None
    s = ls.exp() if a.learned else sig.view(1, K, 1)
    x = (mu.float() + s * torch.randn(R, K, D, generator=g, device="cuda")).contiguous()
    ch = P.GaussChain(mu, x, sig, ls)
    logp = torch.empty(R, device="cuda")
    P.rlvla_flow_logprob(ch, logp=logp)
    lb = (logp + 0.05 * torch.randn(R, generator=g, device="cuda")).contiguous()
    adv = torch.randn(R, generator=g, device="cuda")
    ver = torch.full((R,), 100, dtype=torch.int32, device="cuda")
    key = torch.ones(R, dtype=torch.int64, device="cuda")
    fa = P.ppo_args(logp_behav=lb, adv=adv, version=ver, slot_key=key, a_tok=1, cur_version=100,
                    tok_denominator=float(R))
    dmu = torch.empty_like(mu)
    dls = torch.empty(R, K, D, device="cuda") if a.learned else None
    st = torch.zeros(24, dtype=torch.float64, device="cuda")
    ws = P.workspace(1)
    flush = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")

    def call():
        if a.fwd:
            P.rlvla_flow_logprob(ch, logp=logp)
        else:
            P.rlvla_flow_logprob(ch, logp=logp, fused=fa, dmu=dmu, dlog_std=dls,
                                 stats=None if a.no_stats else st, ws=ws)

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    torch.cuda._sleep(100_000_000)
    evs = []
    for _ in range(a.iters):
        flush.sum()                      # read flush: inputs come from HBM
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        call()
        e[1].record()
        evs.append(e)
    torch.cuda.synchronize()
    ms = sorted(e[0].elapsed_time(e[1]) for e in evs)
    # the same timing around a one-element torch kernel: the event + launch floor
    one = torch.zeros(1, device="cuda")
    torch.cuda._sleep(100_000_000)
    fe = []
    for _ in range(a.iters):
        flush.sum()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        one.add_(1.0)
        e[1].record()
        fe.append(e)
    torch.cuda.synchronize()
    floor = sorted(e[0].elapsed_time(e[1]) for e in fe)
    n = R * K * D
    eb = mu.element_size()
    byts = n * (eb + 4 + (4 if a.learned else 0)) + n * (eb + (4 if a.learned else 0)) + R * (4 + 4 + 4 + 4 + 8 + 4)
    med = ms[len(ms) // 2]
    if a.fwd:
        byts = n * (eb + 4 + (4 if a.learned else 0)) + R * 4
    print(json.dumps({"what": "rlvla_flow_logprob " + ("forward only" if a.fwd else "fused PPO + backward")
                      + (", no stats" if a.no_stats else ""), "rows": R, "K": K, "D": D,
                      "mu_dtype": str(mdt).replace("torch.", ""), "learned_log_std": a.learned,
                      "alg_bytes": byts, "us_median": med * 1e3, "us_min": ms[0] * 1e3,
                      "GBps_median": byts / med / 1e6, "GBps_best": byts / ms[0] / 1e6,
                      "loss": float(st[6].item()), "ms_all": [round(v * 1e3, 2) for v in ms],
                      "floor_us_median": floor[len(floor) // 2] * 1e3}))


if __name__ == "__main__":
    main()
