"""CUDA-event timing of S2 (rlvla_advantages): GAE (+ whitening) and GRPO at the per-GPU
shapes of the BASELINE.json configs (SURVEY §8 sizes table) and one large shape.

Usage (GPU box): python tools/prof_adv.py [--iters 200] > gpurun_out/prof_adv.jsonl
Each line: mode, E_r, T, A, us per call (median / min over `iters` events on the launching
stream), ns per env step. S2 is latency-bound at the BJ sizes (a few thousand steps).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_05765_b200 as P  # noqa: E402

SHAPES = [("libero_spatial_oft", 64, 64, 56), ("libero10_long/2", 128, 128, 56),
          ("maniskill_ppo_gae/8", 128, 10, 56), ("grpo_span/8", 256, 64, 56),
          ("large", 4096, 1024, 8)]


def buffer(E, T, A, seed):
    rng = np.random.default_rng(seed)
    buf = P.TrajectoryBuffer.allocate(E, T, A)
    buf.reward.copy_(torch.from_numpy((rng.random((E, T)) < 0.02).astype(np.float32)))
    buf.value.copy_(torch.from_numpy(rng.normal(size=(E, T)).astype(np.float32)))
    buf.done.copy_(torch.from_numpy((rng.random((E, T)) < 0.01).astype(np.uint8)))
    buf.version.fill_(100)
    buf.tokens.copy_(torch.from_numpy(rng.integers(0, 256, size=(E, T, A)).astype(np.int32)))
    buf.slot_key.fill_(5)
    return buf


def time_call(fn, iters):
    stream = torch.cuda.current_stream()
    for _ in range(10):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(iters)]
    torch.cuda.synchronize()
    for a, b in ev:
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    us = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
    return float(np.median(us)), float(us.min())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    for name, E, T, A in SHAPES:
        buf = buffer(E, T, A, E + T)
        lv = torch.zeros(E, device="cuda")
        adv = torch.empty(E, T, device="cuda")
        ret = torch.empty(E, T, device="cuda")
        stats = torch.zeros(24, dtype=torch.float64, device="cuda")
        ws = P.workspace(E)
        gid = torch.arange(E, dtype=torch.int32, device="cuda") // 8
        modes = {
            "gae": P.adv_params("gae", n_env_global=E, cur_version=100),
            "gae+whiten": P.adv_params("gae", whiten=True, n_env_global=E, cur_version=100),
            "grpo": P.adv_params("grpo", group_id=gid, group_size=8, n_env_global=E,
                                 cur_version=100),
        }
        for mode, prm in modes.items():
            def fn():
                P.rlvla_advantages(buf, lv, prm, adv, ret, stats, ws, check=False)
            med, mn = time_call(fn, args.iters)
            print(json.dumps({"shape": name, "mode": mode, "E_r": E, "T": T, "A": A,
                              "us_median": round(med, 2), "us_min": round(mn, 2),
                              "ns_per_slot": round(med * 1e3 / (E * T), 3)}), flush=True)


if __name__ == "__main__":
    main()
