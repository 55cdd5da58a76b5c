"""bench.py — rollout-to-loss throughput of the B200 path (BASELINE.json metric).

One step = one pass of the whole hot path over one batch: scatter every
out-of-order step record (arrival chunks of B_max = 64, Eq. (1)) into the trajectory
buffer, advantages (GRPO for the LIBERO-Spatial OFT config), and the fused action-token
log-softmax + PPO forward/backward writing dlogits, with the loss statistics. Logits are
the (synthetic) VLA forward output and are resident in HBM before the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (weak scaling: 64 envs per GPU)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "trajectory-steps/sec (rollout-to-loss) at 1/2/4/8 B200; logprob kernel HBM GB/s vs peak"
UNIT = "env-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="libero_spatial_oft", choices=sorted(synth.CONFIGS))
    ap.add_argument("--envs-per-gpu", type=int, default=None,
                    help="weak-scaling configs (libero_spatial_oft): envs per GPU")
    ap.add_argument("--microbatch-rows", type=int, default=0,
                    help="logit rows per fused call (Streamer micro-batch, P:88); 0 = all rows "
                         "if they fit, else ~131072 rows of whole envs")
    ap.add_argument("--chunk", type=int, default=synth.B_MAX)
    ap.add_argument("--schedule", default="pipelined", choices=["pipelined", "serial"],
                    help="pipelined: S1+S2 of batch i+1 on a rollout-side stream while S3+S4 of "
                         "batch i runs (double-buffered trajectory buffer); serial: one stream")
    ap.add_argument("--reserve-sms", type=int, default=1,
                    help="pipelined: SMs the persistent log-prob kernel leaves to the other stream")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--eager", action="store_true",
                    help="launch the timed steps eagerly instead of one captured CUDA graph")
    ap.add_argument("--ref-envs", type=int, default=1, help="envs per reference-arm step")
    ap.add_argument("--trace", default=None,
                    help="write a chrome-trace JSON of the timed steps' stage events (rank 0)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --------------------------------------------------------------------------------------
# CUDA events as graph nodes: cudaEventRecordWithFlags(..., cudaEventRecordExternal) during
# stream capture records a timing event node, so kernels stay timed inside a graph replay
# --------------------------------------------------------------------------------------
class Cudart:
    def __init__(self):
        import ctypes
        self.c = ctypes
        self.L = ctypes.CDLL("libcudart.so.12")

    def event(self):
        e = self.c.c_void_p()
        assert self.L.cudaEventCreate(self.c.byref(e)) == 0
        return e

    def record(self, ev, stream_handle, external):
        fn = self.L.cudaEventRecordWithFlags
        r = fn(ev, self.c.c_void_p(stream_handle), self.c.c_uint(1 if external else 0))
        assert r == 0, f"cudaEventRecordWithFlags -> {r}"

    def elapsed(self, a, b):
        ms = self.c.c_float()
        assert self.L.cudaEventElapsedTime(self.c.byref(ms), a, b) == 0
        return ms.value

    def destroy(self, e):
        self.L.cudaEventDestroy(e)


# --------------------------------------------------------------------------------------
# clocks sampled during the timed region
# --------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
            return
        t = time.time()     # do not start timing before the sampler is producing lines
        while time.time() - t < 5.0 and os.path.getsize(self.f.name) == 0:
            time.sleep(0.02)

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [[c.strip() for c in l.split(",")] for l in open(self.f.name).read().splitlines()
                if l.strip()]
        os.unlink(self.f.name)
        if not rows:
            return None
        num = lambda v: float(v) if v.replace(".", "", 1).isdigit() else 0.0  # noqa: E731
        sm = [num(r[1]) for r in rows]
        mx = max(num(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].strip() == "Active"})
        load = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(num(r[3]) for r in rows)}


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2602_05765_b200 as P
    from paper_2602_05765_b200 import sharding

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    base = synth.CONFIGS[args.config]
    weak = base.gpus == (1,)
    if weak:      # LIBERO-Spatial OFT: 64 envs per GPU, E grows with N (weak scaling)
        E_r = args.envs_per_gpu or base.n_env
        E = E_r * world
    else:         # BJ configs quoted at a GPU count: fixed global E split over N (strong)
        E = base.n_env
        if E % world:
            raise SystemExit(f"{E} envs do not split over {world} GPUs")
        E_r = E // world
    groups_span = world > 1 and base.adv_mode == "grpo"
    cfg = synth.scaled(base, n_env=E, interleave_groups=groups_span or base.interleave_groups)
    T, A, V = cfg.t_steps, cfg.a_tok, cfg.vocab
    lo, hi = sharding.env_range(E, world, rank)
    R = E_r * T * A
    env_rows = T * A
    if args.microbatch_rows:
        mb_envs = max(1, args.microbatch_rows // env_rows)
    elif R * V * 2 * 2 <= 40e9:
        mb_envs = E_r
    else:
        mb_envs = max(1, 131072 // env_rows)
    mb_envs = min(mb_envs, E_r)
    MB = mb_envs * env_rows                       # rows per fused call
    mbs = [(m, min(R, m + MB)) for m in range(0, R, MB)]
    comm = P.Comm.from_process_group(device=dev) if world > 1 else None

    # ---- inputs (outside the timed region) -------------------------------------------
    traj = synth.make_trajectories(cfg)
    rec = synth.make_records(traj, lo, hi)
    # the VLA forward output of one micro-batch (whole envs); with several micro-batches the
    # buffer is reused: every fused call still reads and writes all of its rows
    logits = synth.gen_logits(cfg, traj, lo, lo + mb_envs, device=dev)   # [MB, V] bf16 in HBM
    dlogits = torch.empty_like(logits)
    # behaviour log-probs: the rollout's forward over the same rows (our fwd kernel),
    # plus the synthetic rollout/trainer drift
    tok_rows = torch.from_numpy(traj.tokens[lo:hi].reshape(-1)).to(dev)
    lp_roll = torch.empty(R, device=dev)
    for m0, m1 in mbs:
        P.rlvla_logprob_fwd_bwd(logits[:m1 - m0], tok_rows[m0:m1], logp=lp_roll[m0:m1])
    rows = synth.record_rows(rec, cfg, E_r)
    rows_t = torch.from_numpy(np.where(rows >= 0, rows, 0)).to(dev)
    lb = lp_roll[rows_t] * torch.from_numpy((rows >= 0).astype(np.float32)).to(dev)
    lb = (lb + torch.from_numpy(rec.behav_noise).to(dev)).contiguous()
    host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in dict(
        env_id=rec.env_id, step=rec.step, version=rec.version, reward=rec.reward, done=rec.done,
        value=rec.value, tokens=rec.tokens).items()}
    host["logp_behav"] = lb.cpu().pin_memory()
    drec = P.StepBatch(**{k: v.to(dev) for k, v in host.items()})
    h2d_bytes = sum(v.numel() * v.element_size() for v in host.values())

    # two trajectory buffers (with their advantages / statistics): in the pipelined schedule
    # batch i+1 streams into one (S1) and gets its advantages (S2) on the rollout-side stream
    # while the actor's S3+S4 reads batch i from the other (§3.1 rollout keeps running on
    # the pre-update policy; §3.3 the Streamer masks data preparation time)
    # (the pipelined schedule needs the in-kernel exchanges when N > 1: two streams must not
    # interleave NCCL collectives of one communicator)
    nbuf = 2 if args.schedule == "pipelined" and (comm is None or comm.p2p) else 1
    bufs = [P.TrajectoryBuffer.allocate(E_r, T, A, device=dev) for _ in range(nbuf)]
    cnts = [torch.zeros(4, dtype=torch.int64, device=dev) for _ in range(nbuf)]
    advs = [torch.zeros(E_r, T, device=dev) for _ in range(nbuf)]
    rets = [torch.zeros(E_r, T, device=dev) for _ in range(nbuf)]
    statss = [torch.zeros(24, dtype=torch.float64, device=dev) for _ in range(nbuf)]
    wss = [P.workspace(E, device=dev) for _ in range(nbuf)]   # S2 (rollout-side stream)
    ws_act = P.workspace(E, device=dev)                       # S3+S4 (actor stream)
    lstats = torch.zeros(24, dtype=torch.float64, device=dev)
    logp = torch.empty(R, device=dev)
    lv = torch.from_numpy(traj.last_value[lo:hi]).to(dev)
    gid = torch.from_numpy(traj.group_id).to(dev)
    prm = P.adv_params(cfg.adv_mode, whiten=cfg.whiten,
                       group_id=gid if cfg.adv_mode == "grpo" else None,
                       group_size=cfg.group_size, env_offset=lo, n_env_global=E,
                       cur_version=synth.CUR_VERSION, max_staleness=1)
    fass = []
    for k in range(nbuf):
        b, a_, st_ = bufs[k], advs[k], statss[k]
        fas = []
        for i, (m0, m1) in enumerate(mbs):
            s0, s1 = m0 // A, m1 // A
            fas.append(P.ppo_args(logp_behav=b.logp_behav.view(-1)[m0:m1], adv=a_.view(-1)[s0:s1],
                                  version=b.version.view(-1)[s0:s1],
                                  slot_key=b.slot_key.view(-1)[s0:s1], a_tok=A,
                                  cur_version=synth.CUR_VERSION, max_staleness=1, adv_stats=st_,
                                  accumulate=i > 0))
        fass.append(fas)
    chunks = synth.arrival_chunks(rec.n, args.chunk)
    chunk_batches = [drec.slice(sl) for sl in chunks]
    nmb = len(mbs)
    cr = Cudart()
    ev_k0 = [cr.event() for _ in range(args.steps * nmb)]
    ev_k1 = [cr.event() for _ in range(args.steps * nmb)]
    ev_t0, ev_t1 = cr.event(), cr.event()
    # per-stage events (S1/S2 are latency-bound, reported in us per call)
    ev_sa = [cr.event() for _ in range(args.steps)]   # before the scatter calls
    ev_sb = [cr.event() for _ in range(args.steps)]   # after the scatter calls
    ev_ad = [cr.event() for _ in range(args.steps)]   # before rlvla_advantages
    ev_sc = [cr.event() for _ in range(args.steps)]   # after rlvla_advantages
    s_roll = torch.cuda.Stream(device=dev) if nbuf == 2 else None
    if nbuf == 2:
        P.rlvla_set_reserved_sms(args.reserve_sms)
    st_pinned = torch.empty(lstats.numel(), dtype=torch.float64).pin_memory()
    dst = {k: getattr(drec, k) for k in host}

    def prepare(i, k, stream, timed, capturing, e2e):
        """S1 + S2 of batch i into buffer k on `stream` (records H2D first for e2e)."""
        sh = stream.cuda_stream
        with torch.cuda.stream(stream):
            if e2e:
                for key, v in host.items():
                    dst[key].copy_(v, non_blocking=True)
            bufs[k].reset()
            cnts[k].zero_()
            if timed:
                cr.record(ev_sa[i], sh, capturing)
            seq = 1
            for sl, cb in zip(chunks, chunk_batches):
                P.rlvla_scatter_steps(bufs[k], cb, synth.CUR_VERSION, seq, cnts[k], stream=stream)
                seq += sl.stop - sl.start
            if timed:
                cr.record(ev_sb[i], sh, capturing)
                cr.record(ev_ad[i], sh, capturing)
            P.rlvla_advantages(bufs[k], lv, prm, advs[k], rets[k], statss[k], wss[k], comm=comm,
                               stream=stream)
            if timed:
                cr.record(ev_sc[i], sh, capturing)

    def actor(i, k, stream, timed, capturing, e2e):
        """S3 + S4 (fused log-prob + PPO fwd/bwd, dlogits, loss statistics) on buffer k."""
        sh = stream.cuda_stream
        for j, ((m0, m1), fa) in enumerate(zip(mbs, fass[k])):
            if timed:
                cr.record(ev_k0[i * nmb + j], sh, capturing)
            P.rlvla_logprob_fwd_bwd(logits[:m1 - m0], bufs[k].tokens.view(-1)[m0:m1], logp=logp[m0:m1],
                                    fused=fa, dlogits=dlogits[:m1 - m0], stats=lstats, ws=ws_act,
                                    comm=comm if j == nmb - 1 else None, stream=stream)
            if timed:
                cr.record(ev_k1[i * nmb + j], sh, capturing)
        if e2e:
            st_pinned.copy_(lstats, non_blocking=True)

    def run_steps(n, timed=False, capturing=False, e2e=False):
        """n whole steps (batches). serial: S1, S2, S3+S4 of batch i back to back on one
        stream. pipelined: S1+S2 of batch i+1 on the rollout-side stream while the actor's
        S3+S4 of batch i runs (double-buffered); the first batch's preparation is exposed."""
        main = torch.cuda.current_stream()
        if nbuf == 1:
            for i in range(n):
                prepare(i, 0, main, timed, capturing, e2e)
                actor(i, 0, main, timed, capturing, e2e)
            return
        ready = [torch.cuda.Event() for _ in range(n)]
        done = [torch.cuda.Event() for _ in range(n)]
        s_roll.wait_stream(main)                               # fork
        prepare(0, 0, s_roll, timed, capturing, e2e)
        ready[0].record(s_roll)
        for i in range(n):
            if i + 1 < n:
                if i >= 1:                   # buffer (i+1) % 2 was read by batch i-1's actor
                    s_roll.wait_event(done[i - 1])
                prepare(i + 1, (i + 1) % 2, s_roll, timed, capturing, e2e)
                ready[i + 1].record(s_roll)
            main.wait_event(ready[i])
            actor(i, i % 2, main, timed, capturing, e2e)
            done[i].record(main)
        main.wait_stream(s_roll)                               # join

    n_adv_kernels = 2 if (cfg.adv_mode == "grpo" or cfg.whiten) else 1
    launches_per_step = len(chunks) + n_adv_kernels + nmb   # scatter chunks + advantages + fused

    def barrier():
        if world > 1:
            dist.barrier()

    run_steps(args.warmup)
    torch.cuda.synchronize()
    graph = None
    if not args.eager:
        # the K timed steps as ONE captured graph (event nodes around every stage)
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                cs = torch.cuda.current_stream().cuda_stream
                cr.record(ev_t0, cs, True)
                run_steps(args.steps, timed=True, capturing=True)
                cr.record(ev_t1, cs, True)
            graph.replay()                      # one untimed replay (graph upload / warm-up)
            torch.cuda.synchronize()
        except Exception as ex:                 # pragma: no cover - fall back to eager
            print(f"[bench] graph capture failed ({ex}); timing eagerly", file=sys.stderr)
            graph = None
    barrier()
    clk = ClockSampler(local)
    clk.start()
    torch.cuda.synchronize()
    barrier()
    stream = torch.cuda.current_stream()
    if graph is not None:
        graph.replay()
    else:
        cr.record(ev_t0, stream.cuda_stream, False)
        run_steps(args.steps, timed=True)
        cr.record(ev_t1, stream.cuda_stream, False)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    ms = cr.elapsed(ev_t0, ev_t1)
    k_ms = [cr.elapsed(a, b) for a, b in zip(ev_k0, ev_k1)]   # one per fused launch
    sc_ms = sorted(cr.elapsed(a, b) for a, b in zip(ev_sa, ev_sb))
    ad_ms = sorted(cr.elapsed(a, b) for a, b in zip(ev_ad, ev_sc))
    if args.trace and rank == 0:
        # chrome://tracing / Perfetto: one complete event per stage of every timed step,
        # timestamps relative to the start of the timed region (CUDA events, microseconds)
        evs = []
        for i in range(args.steps):
            t_s = cr.elapsed(ev_t0, ev_sa[i]) * 1e3
            evs.append(dict(name="S1 scatter (64 chunks)", ph="X", pid=0, tid=1 if nbuf == 2 else 0, ts=t_s,
                            dur=cr.elapsed(ev_sa[i], ev_sb[i]) * 1e3))
            evs.append(dict(name="S2 advantages", ph="X", pid=0, tid=1 if nbuf == 2 else 0, ts=cr.elapsed(ev_t0, ev_ad[i]) * 1e3,
                            dur=cr.elapsed(ev_ad[i], ev_sc[i]) * 1e3))
            for j in range(nmb):
                a_, b_ = ev_k0[i * nmb + j], ev_k1[i * nmb + j]
                evs.append(dict(name=f"S3+S4 fused (micro-batch {j})", ph="X", pid=0, tid=0,
                                ts=cr.elapsed(ev_t0, a_) * 1e3, dur=cr.elapsed(a_, b_) * 1e3))
        with open(args.trace, "w") as f:
            json.dump({"traceEvents": evs, "displayTimeUnit": "ms"}, f)
    st_host = lstats.cpu().numpy()
    cnt = cnts[(args.steps - 1) % nbuf].cpu().numpy()

    # ---- e2e: records from pinned host memory, stats back to host, every step -------
    e2e_ms = None
    if not args.no_e2e:
        run_steps(min(2, args.warmup), e2e=True)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.current_stream()
        e0.record(stream)
        run_steps(args.steps, e2e=True)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        e2e_ms = e0.elapsed_time(e1)

    # ---- max over ranks ------------------------------------------------------------------
    vals = torch.tensor([ms, float(np.mean(k_ms)), e2e_ms or 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, k_avg, e2e_ms = vals.tolist()
    if args.no_e2e:
        e2e_ms = None
    units_per_step = E * cfg.n_es        # env steps of all ranks (Eq. (2) unit)
    value = units_per_step * args.steps / (ms / 1e3)
    # algorithmic bytes of one fused launch: logits read + dlogits write + target, logp_behav,
    # logp (4 B each) per row + adv, version, slot_key (16 B) per decision step
    alg_bytes_step = R * (2 * V * 2 + 4 + 4 + 4) + (R // A) * (4 + 4 + 8)
    alg_bytes = alg_bytes_step / nmb
    achieved = alg_bytes / (k_avg / 1e3) / 1e9
    peak, peak_src = peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_fused.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            if tj.get("rows_per_launch") == MB and tj.get("vocab") == V:
                traffic = tj.get("bytes_per_launch")
        except Exception:
            traffic = None
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": cfg.name if (world == 1 or not weak) else f"{base.name} x{world} (weak)",
                   "envs_per_gpu": E_r, "envs_total": E, "episode_steps": cfg.n_es,
                   "chunk": cfg.chunk, "decision_steps": T, "tokens_per_step": A, "vocab": V,
                   "rows_per_gpu": R, "records_per_gpu": rec.n, "arrival_chunk": args.chunk,
                   "fused_calls_per_step": nmb, "rows_per_fused_call": MB,
                   "launch": "one CUDA graph of the K timed steps" if graph is not None else "eager",
                   "schedule": ("pipelined: S1+S2 of batch i+1 on a second stream during S3+S4 "
                                f"of batch i (double-buffered trajectory buffer, {args.reserve_sms} SM "
                                "left free by the persistent kernel)") if nbuf == 2 else "serial",
                   "advantages": cfg.adv_mode, "group_size": cfg.group_size,
                   "groups_span_ranks": bool(groups_span),
                   "l2": f"inputs larger than L2: {R * V * 2 / 1e9:.1f} GB logits read + same "
                         "written per step per GPU, no flush needed",
                   "parallelism": f"dp{world}",
                   "nranks": world,
                   "collectives": ("none (1 rank)" if comm is None else
                                   "C1/C2/C3 in-kernel over NVLink peer memory (CUDA IPC mailboxes)"
                                   if comm.p2p else "C1/C2/C3 NCCL collectives on the step stream")},
        "clocks": clocks,
        "e2e": None if e2e_ms is None else {
            "value": units_per_step * args.steps / (e2e_ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(st_pinned.numel() * 8),
            "note": "step records H2D from pinned memory + loss stats D2H inside the timed "
                    "region; logits are the VLA forward output produced on the device"},
        "gpu_launches": launches_per_step * args.steps,
        "gpu_launches_per_step": {"scatter": len(chunks), "advantages": n_adv_kernels,
                                  "fused_logprob_ppo": nmb},
        "stages": {"scatter_us_per_step_median": 1e3 * sc_ms[len(sc_ms) // 2],
                   "scatter_calls_per_step": len(chunks),
                   "scatter_us_per_call_median": 1e3 * sc_ms[len(sc_ms) // 2] / max(1, len(chunks)),
                   "advantages_us_median": 1e3 * ad_ms[len(ad_ms) // 2],
                   "advantages_ns_per_env_step": 1e6 * ad_ms[len(ad_ms) // 2] / (units_per_step / world),
                   "fused_ms_per_step_median": sorted(k_ms)[len(k_ms) // 2] * nmb,
                   "note": "CUDA event nodes inside the timed graph; S1/S2 latency-bound (us per call)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_nominal": 8000.0, "frac_nominal": achieved / 8000.0,
                     "kernel": "lp_tma_kernel<FUSED> (rlvla_logprob_fwd_bwd fused)",
                     "kernel_ms": k_avg, "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                     "kernel_share_of_step": k_avg * nmb / (ms / args.steps)},
        "stats_last_step": {"loss": float(st_host[6]), "clip_frac": float(st_host[7] / max(1, st_host[11])),
                            "n_loss_tok": float(st_host[11]), "n_stale_tok": float(st_host[12]),
                            "counters": cnt.tolist()},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, traj, logits, lb_fn=None,
                                           n_env_sample=min(4, mb_envs))
    if rank == 0:
        print(json.dumps(out), flush=True)
    # the captured graph holds NCCL's persistent plans for the C1/C2/C3 collectives: release
    # it before the communicator, or ncclCommDestroy waits for them forever
    graph = None
    import gc
    gc.collect()
    torch.cuda.synchronize()
    if comm is not None:
        comm.destroy()
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------------------------------
# oracle timing (cpu_baseline leg and --impl reference)
# --------------------------------------------------------------------------------------
_ORACLE_X = None      # fork-shared logits of the all-cores oracle leg (set before the fork)


def _oracle_rows(job):
    """One worker's share of the oracle's S3+S4 (rows are independent): the loss
    statistics of rows [r0, r1) (dlogits computed, not shipped back)."""
    from oracle import path as O_path
    r0, r1, n_tok, tv = job
    out = O_path.loss_and_grad(_ORACLE_X[r0:r1], tv, n_tok=n_tok, rows=np.arange(r0, r1))
    return out["stats"]


def oracle_sample_step(cfg, traj, logits_rows_fn, n_env_sample, pool=None, nproc=1):
    """The oracle's whole path over `n_env_sample` envs of the workload (their records in
    arrival order, their logit rows), stage by stage as oracle.path.rollout_to_loss composes
    it: S1 scatter of every arrival chunk, S2 advantages, S3+S4 loss and dlogits. With a
    process pool, S3+S4 is split into `nproc` row blocks whose statistics are combined in
    block order (S1/S2 stay serial: they are < 1 % of the work). Returns per-stage seconds."""
    from oracle import logprob as O_lp
    from oracle import path as O_path
    from oracle import scatter as O_sc
    rec = synth.make_records(traj, 0, n_env_sample)
    x = logits_rows_fn(n_env_sample)                         # float64 [rows, V]
    rows = synth.record_rows(rec, cfg, n_env_sample)
    # behaviour log-probs (rollout side, not timed)
    fl = O_lp.log_softmax_gather(x, traj.tokens[:n_env_sample].reshape(-1))["logp"]
    lb = np.where(rows >= 0, fl[np.maximum(rows, 0)], 0.0) + rec.behav_noise
    recd = dict(env_id=rec.env_id, step=rec.step, version=rec.version, reward=rec.reward,
                done=rec.done, value=rec.value, tokens=rec.tokens, logp_behav=lb.astype(np.float32))
    chunks = [{k: v[sl] for k, v in recd.items()} for sl in synth.arrival_chunks(rec.n)]
    t0 = time.perf_counter()
    buf = O_sc.new_buffer(n_env_sample, cfg.t_steps, cfg.a_tok)
    seq = 1
    for ch in chunks:
        O_sc.scatter_steps(buf, ch, synth.CUR_VERSION, seq)
        seq += len(ch["env_id"])
    t1 = time.perf_counter()
    adv = O_path.advantages(buf, traj.last_value[:n_env_sample], mode=cfg.adv_mode, whiten=cfg.whiten,
                            group_of_env=traj.group_id[:n_env_sample], cur_version=synth.CUR_VERSION,
                            max_staleness=1)
    t2 = time.perf_counter()
    tv = O_path.token_view(buf, adv["adv"], cfg.a_tok, synth.CUR_VERSION)
    n_tok = float(adv["counts"]["n_tok"])
    if pool is None:
        O_path.loss_and_grad(x, tv, n_tok=n_tok)
    else:
        assert _ORACLE_X.shape == x.shape and np.shares_memory(_ORACLE_X, x), \
            "the pool must be forked after _ORACLE_X is set"
        R = x.shape[0]
        cuts = np.linspace(0, R, nproc + 1).astype(int)
        parts = pool.map(_oracle_rows, [(int(a), int(b), n_tok, tv) for a, b in zip(cuts, cuts[1:])])
        _ = {k: sum(p[k] for p in parts) for k in parts[0] if k != "denom"}   # fixed order
    t3 = time.perf_counter()
    return {"s1": t1 - t0, "s2": t2 - t1, "s3s4": t3 - t2, "total": t3 - t0}


def host_cpu() -> str:
    """The GPU box's host CPU (model name, logical cores) for the oracle baseline."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{model}, {os.cpu_count()} logical cores"


def cpu_baseline(cfg, traj, logits, lb_fn=None, n_env_sample=2):
    """The oracle (as it stands) on the GPU box's host cores: one thread, then all logical
    cores (S3+S4 row blocks over a fork pool, fixed-order combine), per stage."""
    import multiprocessing as mp
    global _ORACLE_X
    x64 = logits[: n_env_sample * cfg.t_steps * cfg.a_tok].double().cpu().numpy()

    def rows_fn(n):
        return x64[: n * cfg.t_steps * cfg.a_tok]
    oracle_sample_step(cfg, traj, rows_fn, 1)          # warm-up (imports, first-call costs)
    one = oracle_sample_step(cfg, traj, rows_fn, n_env_sample)
    nproc = os.cpu_count() or 1
    _ORACLE_X = rows_fn(n_env_sample)    # inherited by the forked workers
    with mp.get_context("fork").Pool(nproc) as pool:
        allc = oracle_sample_step(cfg, traj, rows_fn, n_env_sample, pool=pool, nproc=nproc)
    _ORACLE_X = None
    units = n_env_sample * cfg.n_es
    stages = lambda d: {k: round(v, 4) for k, v in d.items()}  # noqa: E731
    return {"value": units / one["total"], "unit": UNIT, "cores": 1, "kind": "oracle", "host": host_cpu(),
            "sample": f"{n_env_sample} of {cfg.n_env} envs x {cfg.n_es} env steps "
                      f"({n_env_sample * cfg.t_steps * cfg.a_tok} logit rows x {cfg.vocab}), "
                      f"whole path S1-S4, numpy fp64 single thread, {one['total']:.1f} s",
            "stage_seconds": stages(one),
            "all_cores": {"value": units / allc["total"], "unit": UNIT, "cores": nproc,
                          "stage_seconds": stages(allc),
                          "how": "same sample; S3+S4 split into row blocks over a fork pool of "
                                 "every logical core, statistics combined in block order; S1/S2 serial"}}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import torch
    cfg = synth.CONFIGS[args.config]
    traj = synth.make_trajectories(cfg)
    n = args.ref_envs

    def rows_fn(k):
        return synth.gen_logits(cfg, traj, 0, k, device="cpu").double().numpy()

    for _ in range(args.warmup):
        oracle_sample_step(cfg, traj, rows_fn, n)
    runs = [oracle_sample_step(cfg, traj, rows_fn, n) for _ in range(args.steps)]
    secs = [r["total"] for r in runs]
    tot = float(sum(secs))
    value = n * cfg.n_es * args.steps / tot
    sample = (f"{n} of {cfg.n_env} envs x {cfg.n_es} env steps per step "
              f"({n * cfg.t_steps * cfg.a_tok} logit rows x {cfg.vocab}), whole path S1-S4")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": cfg.name, "envs_per_step": n, "vocab": cfg.vocab,
                      "parallelism": "cpu oracle (rank 0 only)"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "host": host_cpu(),
                            "sample": sample,
                            "stage_seconds": {k: round(float(np.mean([r[k] for r in runs])), 4)
                                              for k in ("s1", "s2", "s3s4", "total")}},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)
    del torch


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
