"""Test harness: builds one seeded case, runs it through the CUDA path (via the C-ABI
binding) and through the oracle, and provides the comparators. Inputs come from synth/
only; oracle outputs never feed the CUDA side except as *inputs* the rollout would have
produced (behaviour log-probs), which the real system gets from the rollout's forward."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

import synth
from oracle import advantages as O_adv
from oracle import logprob as O_lp
from oracle import path as O_path
from oracle import scatter as O_sc

# --------------------------------------------------------------------------------------
# comparators
# --------------------------------------------------------------------------------------

def bf16_ord(bits: np.ndarray) -> np.ndarray:
    b = bits.astype(np.int32) & 0xFFFF
    return np.where(b & 0x8000, -(b & 0x7FFF), b)


def bf16_rne_bits(x64: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(x64, dtype=np.float64)).to(torch.float32)
    return t.to(torch.bfloat16).view(torch.int16).numpy().astype(np.int32) & 0xFFFF


def bf16_value(bits: np.ndarray) -> np.ndarray:
    b = torch.from_numpy((np.asarray(bits).astype(np.int32) & 0xFFFF).astype(np.uint16).view(np.int16))
    return b.view(torch.bfloat16).to(torch.float64).numpy()


def assert_bf16_ulp(gpu_bits: np.ndarray, ref64: np.ndarray, max_ulp: int = 1, ftz=1.2e-38,
                    abs_floor=None):
    """|ord(gpu) - ord(RNE_bf16(ref))| <= max_ulp, ±0 equal; refs below FLT_MIN may flush.
    `abs_floor` (array or scalar): an element also passes when |gpu - ref| <= abs_floor —
    for values that are a cancelling sum, whose fp32 error bound is relative to the sum of
    the terms' magnitudes rather than to the value."""
    rb = bf16_rne_bits(ref64)
    d = np.abs(bf16_ord(gpu_bits) - bf16_ord(rb))
    tiny = np.abs(ref64) < ftz
    bad = (d > max_ulp) & ~tiny
    if abs_floor is not None and bad.any():
        bad &= ~(np.abs(bf16_value(gpu_bits) - ref64) <= abs_floor)
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{int(bad.sum())} bf16 elements off by > {max_ulp} ulp; first at "
                             f"{tuple(i)}: gpu bits {gpu_bits[tuple(i)]:#06x} ref {ref64[tuple(i)]!r}")
    return int(d[~tiny].max()) if (~tiny).any() else 0


def assert_close_rel(gpu, ref, rel=1e-5, floor=1.0, what=""):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    tol = rel * np.maximum(np.abs(ref), floor)
    err = np.abs(gpu - ref)
    same_nan = np.isnan(gpu) & np.isnan(ref)
    bad = ~(err <= tol) & ~same_nan
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {int(bad.sum())} mismatches; first at {tuple(i)} "
                             f"gpu={gpu[tuple(i)]!r} ref={ref[tuple(i)]!r} tol={tol[tuple(i)]!r}")
    return float(np.nanmax(err)) if err.size else 0.0


# --------------------------------------------------------------------------------------
# case construction
# --------------------------------------------------------------------------------------

@dataclass
class Case:
    cfg: synth.WorkloadConfig
    traj: synth.Trajectories
    env_lo: int
    env_hi: int
    rec: synth.Records
    logp_behav: np.ndarray          # f32 [M, A] (records' payload)
    logits: torch.Tensor            # [R, V] on `device`
    extra: dict = field(default_factory=dict)

    @property
    def n_env(self):
        return self.env_hi - self.env_lo


def oracle_rows_logp(x: torch.Tensor, rows: np.ndarray, targets: np.ndarray) -> np.ndarray:
    """Oracle log-probs of the given logit rows (decoded exactly to float64)."""
    out = np.zeros(len(rows))
    for s in range(0, len(rows), 4096):
        r = rows[s:s + 4096]
        xr = x[torch.from_numpy(r).to(x.device)].double().cpu().numpy()
        out[s:s + 4096] = O_lp.log_softmax_gather(xr, targets[s:s + 4096])["logp"]
    return out


def build_case(cfg, env_lo=0, env_hi=None, device="cpu", behav_sample=None, seed=None) -> Case:
    """behav_sample: None => behaviour log-probs from the oracle for every record row;
    int k => only for the records of a fixed sample of k slots (others: synthetic N(-3, .5))."""
    traj = synth.make_trajectories(cfg, seed=seed)
    env_hi = cfg.n_env if env_hi is None else env_hi
    rec = synth.make_records(traj, env_lo, env_hi)
    E = env_hi - env_lo
    logits = synth.gen_logits(cfg, traj, env_lo, env_hi, device=device)
    rows = synth.record_rows(rec, cfg, E)                     # [M, A], -1 for OOB
    lb = rec.behav_noise.astype(np.float64).copy()
    ok = rows >= 0
    if behav_sample is not None:
        rng = np.random.default_rng(7)
        lb[:] = -3.0 + 0.5 * rng.standard_normal(lb.shape)
        pick = np.zeros(rows.shape[0], bool)
        pick[rng.choice(rows.shape[0], size=min(behav_sample, rows.shape[0]), replace=False)] = True
        ok = ok & pick[:, None]
    r_ok = rows[ok]
    if len(r_ok):
        lp = oracle_rows_logp(logits, r_ok, rec.tokens[ok])
        lb[ok] = np.nan_to_num(lp, nan=0.0, posinf=0.0, neginf=0.0) + rec.behav_noise[ok]
    return Case(cfg, traj, env_lo, env_hi, rec, lb.astype(np.float32), logits,
                extra=dict(behav_rows=np.unique(r_ok)))


def records_np(case: Case) -> dict:
    r = case.rec
    return dict(env_id=r.env_id, step=r.step, version=r.version, reward=r.reward, done=r.done,
                value=r.value, tokens=r.tokens, logp_behav=case.logp_behav)


# --------------------------------------------------------------------------------------
# CUDA path through the binding
# --------------------------------------------------------------------------------------

def to_dev_batch(case: Case, device="cuda"):
    from paper_2602_05765_b200 import StepBatch
    r = records_np(case)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
    return StepBatch(t(r["env_id"]), t(r["step"]), t(r["version"]), t(r["reward"]),
                     t(r["done"]), t(r["value"]), t(r["tokens"]), t(r["logp_behav"]))


def gpu_scatter(case: Case, chunk=synth.B_MAX, seq_base=1, cur_version=synth.CUR_VERSION):
    import paper_2602_05765_b200 as P
    cfg = case.cfg
    buf = P.TrajectoryBuffer.allocate(case.n_env, cfg.t_steps, cfg.a_tok)
    rec = to_dev_batch(case)
    counters = torch.zeros(4, dtype=torch.int64, device="cuda")
    seq = seq_base
    for sl in synth.arrival_chunks(rec.n, chunk):
        P.rlvla_scatter_steps(buf, rec.slice(sl), cur_version, seq, counters)
        seq += sl.stop - sl.start
    return buf, counters


def oracle_scatter(case: Case, chunk=synth.B_MAX, seq_base=1, cur_version=synth.CUR_VERSION):
    cfg = case.cfg
    buf = O_sc.new_buffer(case.n_env, cfg.t_steps, cfg.a_tok)
    r = records_np(case)
    cnt = np.zeros(4, np.int64)
    seq = seq_base
    for sl in synth.arrival_chunks(len(r["env_id"]), chunk):
        cnt += O_sc.scatter_steps(buf, {k: v[sl] for k, v in r.items()}, cur_version, seq)
        seq += sl.stop - sl.start
    return buf, cnt


def buf_to_np(buf) -> dict:
    return dict(slot_key=buf.slot_key.cpu().numpy().view(np.uint64),
                reward=buf.reward.cpu().numpy(), done=buf.done.cpu().numpy(),
                value=buf.value.cpu().numpy(), version=buf.version.cpu().numpy(),
                tokens=buf.tokens.cpu().numpy(), logp_behav=buf.logp_behav.cpu().numpy())


def oracle_advantages(case: Case, obuf: dict, mode, **kw):
    cfg = case.cfg
    lv = case.traj.last_value[case.env_lo:case.env_hi]
    gid = case.traj.group_id
    return O_path.advantages(obuf, lv, mode=mode, group_of_env=gid,
                             cur_version=synth.CUR_VERSION, max_staleness=1,
                             env_offset=case.env_lo, **kw)


# --------------------------------------------------------------------------------------
# NEXT-3: closed-loop request traffic for the Eq. (1) batcher, driven by the ORACLE
# --------------------------------------------------------------------------------------
@dataclass
class BatcherCase:
    n_env: int
    obs_bytes: int
    b_max: int
    t_max: int
    ticks: list = field(default_factory=list)   # per tick: dict(now, env, time, cycle, expect)
    counters: np.ndarray | None = None


def batcher_case(n_env, ticks, b_max, t_max, obs_bytes=0, fault_rate=0.05, seed=7):
    """Envs offer when their step finishes, wait for their batch, then step again after the
    batch's inference latency; ~fault_rate of ticks carry bad offers (out-of-range env,
    future enqueue time, a repeat of a pending env or of an env offered in the same tick).
    The ORACLE batcher decides who is batched when; the event list (offers per tick, with
    the payload cycle of each) and its expected batches are what the GPU replays."""
    from oracle import batcher as O_b
    tr = synth.batcher_traffic(n_env, 64, ticks, seed)
    bt = O_b.Batcher(n_env)
    nxt = tr.step_ticks[:, 0].copy()          # first offers after the first env step
    cyc = np.zeros(n_env, np.int64)
    nb = 0
    case = BatcherCase(n_env, obs_bytes, b_max, t_max)
    for now in range(ticks):
        envs = [int(e) for e in np.nonzero(nxt == now)[0]]
        times = [now - int(tr.enq_lag[e, cyc[e] % 64]) for e in envs]
        cycles = [int(cyc[e]) for e in envs]
        u, fe = tr.fault_u[now], tr.fault_env[now]
        if u[0] < fault_rate:                                   # out of range
            envs.append(n_env + int(fe[0] % 5)); times.append(now); cycles.append(-1)
        if u[1] < fault_rate:                                   # enqueue time in the future
            envs.append(int(fe[1] % n_env)); times.append(now + 1 + int(fe[1] % 3)); cycles.append(-1)
        if u[2] < fault_rate and bt.pending.any():              # repeat of a pending env
            pend = np.nonzero(bt.pending)[0]
            envs.append(int(pend[fe[2] % len(pend)])); times.append(now); cycles.append(-1)
        if u[3] < fault_rate and cycles and cycles[0] >= 0:     # same env twice in one tick
            envs.append(envs[0]); times.append(now); cycles.append(-1)
        bt.offer(envs, times, now)
        batch = bt.poll(now, b_max, t_max)
        case.ticks.append(dict(now=now, env=envs, time=times, cycle=cycles, expect=batch))
        if batch:
            back = now + int(tr.infer_ticks[nb])
            nb += 1
            for e, _ in batch:
                cyc[e] += 1
                nxt[e] = back + int(tr.step_ticks[e, cyc[e] % 64])
    case.counters = bt.counters.copy()
    return case


def payload(case: BatcherCase, env: int, cycle: int) -> np.ndarray:
    if cycle < 0:  # bad offers carry a recognisable filler payload
        return np.full(case.obs_bytes, 0xEE, np.uint8)
    return synth.payload_bytes(1234, env, cycle, case.obs_bytes)
