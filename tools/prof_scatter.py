"""Time S1 at the LIBERO-Spatial OFT shape the bench uses: 4,096 step records (A = 56) in 64
Eq. (1) arrival chunks of 64, scattered by 64 rlvla_scatter_steps calls captured in one CUDA
graph (as in bench.py). Prints us per call.

  python tools/prof_scatter.py [--iters N] [--chunk 64]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_05765_b200 as P  # noqa: E402
import synth  # noqa: E402
from tests import harness as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--chunk", type=int, default=synth.B_MAX)
    a = ap.parse_args()
    cfg = synth.CONFIGS["libero_spatial_oft"]
    traj = synth.make_trajectories(cfg)
    rec = synth.make_records(traj, 0, cfg.n_env)
    case = H.Case(cfg, traj, 0, cfg.n_env, rec, rec.behav_noise.astype("float32"), None)
    drec = H.to_dev_batch(case)
    buf = P.TrajectoryBuffer.allocate(cfg.n_env, cfg.t_steps, cfg.a_tok)
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    chunks = synth.arrival_chunks(drec.n, a.chunk)
    batches = [drec.slice(sl) for sl in chunks]

    def once(stream):
        buf.reset()
        cnt.zero_()
        seq = 1
        for sl, b in zip(chunks, batches):
            P.rlvla_scatter_steps(buf, b, synth.CUR_VERSION, seq, cnt, stream=stream)
            seq += sl.stop - sl.start

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        once(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            once(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.iters):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    print(json.dumps({"what": "S1 scatter, one graph of the step's arrival chunks", "records": drec.n,
                      "calls": len(chunks), "us_per_step": ms * 1e3, "us_per_call": ms * 1e3 / len(chunks),
                      "counters": cnt.cpu().tolist()}))


if __name__ == "__main__":
    main()
