"""Time (and serve as the ncu target for) one rlvla_logprob_fwd_bwd mode at the
LIBERO-Spatial OFT shape: 229,376 rows x 32000 bf16 (14.7 GB) on one GPU.

  python tools/prof_fused.py [--mode fused|fwd|bwd] [--iters N] [--rows R]

The first launch is a warm-up (ncu: -s 1 -c 1 captures the second)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_05765_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="fused", choices=["fused", "fwd", "bwd", "copy"],
                    help="copy: torch's dx.copy_(x) of the same bytes (the copy ceiling at this size)")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rows", type=int, default=229376)
    ap.add_argument("--vocab", type=int, default=32000)
    ap.add_argument("--A", type=int, default=56)
    ap.add_argument("--f32", action="store_true", help="fp32 logits (the row kernel at V > 2048)")
    ap.add_argument("--variant", default="none", choices=["none", "dual", "kl", "ent", "all"],
                    help="NEXT-2 loss knobs on the fused call (readings R19-R20)")
    a = ap.parse_args()
    R, V, A = a.rows - a.rows % a.A, a.vocab, a.A  # whole decision steps
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    dt = torch.float32 if a.f32 else torch.bfloat16
    esz = 4 if a.f32 else 2
    x = torch.empty(R, V, dtype=dt, device=dev)
    for s in range(0, R, 16384):
        n = min(16384, R - s)
        x[s:s + n] = (torch.randn(n, V, generator=g, device=dev) * 1.5).to(dt)
    t = torch.randint(V - 256, V, (R,), generator=g, device=dev, dtype=torch.int32)
    dx = torch.empty_like(x)
    logp = torch.empty(R, device=dev)
    lse = torch.empty(R, device=dev)
    S = R // A
    # behaviour log-probs near the current policy (rollout/trainer drift N(0, 0.05^2)) so that
    # ~all rows take the unclipped path like the bench workload (clipped rows skip pass C)
    P.rlvla_logprob_fwd_bwd(x, t, logp=logp)
    lb = (logp + 0.05 * torch.randn(R, generator=g, device=dev)).contiguous()
    adv = torch.randn(S, generator=g, device=dev)
    ver = torch.full((S,), 100, dtype=torch.int32, device=dev)
    key = torch.ones(S, dtype=torch.int64, device=dev)
    stats = torch.zeros(24, dtype=torch.float64, device=dev)
    ws = P.workspace(1)
    vk = {}
    if a.variant in ("dual", "all"):
        vk["dual_clip"] = 3.0
    if a.variant in ("kl", "all"):
        vk["logp_ref"] = (logp + 0.1 * torch.randn(R, generator=g, device=dev)).contiguous()
        vk["kl_coef"] = 0.05
    if a.variant in ("ent", "all"):
        vk["ent_coef"] = 0.01
    fa = P.ppo_args(logp_behav=lb, adv=adv, version=ver, slot_key=key, a_tok=A, cur_version=100,
                    tok_denominator=float(R), **vk)
    gl = torch.randn(R, generator=g, device=dev) * 1e-4

    def call():
        if a.mode == "fused":
            P.rlvla_logprob_fwd_bwd(x, t, logp=logp, fused=fa, dlogits=dx, stats=stats, ws=ws)
        elif a.mode == "copy":
            dx.copy_(x)
        elif a.mode == "fwd":
            P.rlvla_logprob_fwd_bwd(x, t, logp=logp, lse=lse)
        else:
            P.rlvla_logprob_fwd_bwd(x, t, lse=lse, grad_logp=gl, dlogits=dx)

    if a.mode == "bwd":
        P.rlvla_logprob_fwd_bwd(x, t, logp=logp, lse=lse)
    call()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.iters + 1)]
    ev[0].record()
    for i in range(a.iters):
        call()
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.iters)]
    rw = {"copy": 2 * V * esz, "fused": 2 * V * esz + 12, "fwd": V * esz + 12, "bwd": 2 * V * esz + 12}[a.mode]
    if a.mode == "fused" and "logp_ref" in vk:
        rw += 4
    byt = R * rw
    avg = sum(ms) / len(ms)
    if a.mode == "fused":
        torch.cuda.synchronize()
        st = stats.cpu().tolist()
        clip = st[7] / max(1.0, st[11])
    else:
        clip = None
    print(json.dumps({"mode": a.mode, "variant": a.variant, "rows": R, "vocab": V, "dtype": str(dt), "ms_avg": avg, "ms_min": min(ms),
                      "clip_frac": clip,
                      "GBps_avg": byt / avg / 1e6, "GBps_best": byt / min(ms) / 1e6,
                      "ms_all": [round(v, 3) for v in ms]}))


if __name__ == "__main__":
    main()
