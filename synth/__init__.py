"""Seeded synthetic workload generators — the ONE module both sides share.

This module draws random numbers and does index bookkeeping only. It holds none
of the method's arithmetic: no log-softmax, no advantage, no ratio, no loss, no
scatter rule. Both the CUDA path's tests/bench and the oracle consume what it
returns; neither side's arithmetic lives here (DESIGN.md §3 "Input recipe").

Shapes follow the paper's workloads:
  * env counts, episode lengths, chunk sizes: PAPER.md Table 2 (App. A);
    "Total Env/Node", "Max Episode Steps", "Chunk Size".
  * action tokens: OpenVLA "discretizes the action space into tokens" (§2);
    7-DoF x 256 bins, 32000-token vocabulary (BASELINE.json configs).
  * out-of-order arrival: requests from subsets of envs enter early (§3.2);
    arrival chunks of B_max records (Eq. (1)).
  * policy-version lag <= 1 under the paper's schedule (§3.1).
Latencies use SPEC's LogNormalShifted model purely as an arrival-order
generator.

Behaviour log-probs are NOT produced here (that would be method arithmetic):
the generator returns `behav_noise` and the caller forms
logp_behav = logp(current logits) + behav_noise with its own implementation
(the oracle in tests, the GPU forward in bench — the rollout worker's stand-in).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 2602_05765
CUR_VERSION = 100
ACTION_BINS = 256          # OpenVLA 256-bin action tokenisation (BASELINE.json)
DOF = 7                    # 7-DoF action (BASELINE.json)
B_MAX = 64                 # arrival chunk = Eq. (1)'s maximum inference batch


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    index: int               # position in BASELINE.json "configs"
    n_env: int               # E (global)
    n_es: int                # N = env steps per episode window
    chunk: int               # c (action chunk)
    vocab: int               # V
    dtype: str               # "f32" | "bf16"
    adv_mode: str            # "grpo" | "gae"
    group_size: int = 0      # GRPO group size G
    interleave_groups: bool = False
    whiten: bool = False
    gpus: tuple = (1,)
    reward_kind: str = "sparse_once"
    lag_probs: tuple = (0.5, 0.5)       # P(lag = 0), P(lag = 1), P(lag = 2) ...
    faults: bool = False
    dof: int = DOF

    @property
    def t_steps(self) -> int:           # T = N / c decision steps (reading R1)
        return self.n_es // self.chunk

    @property
    def a_tok(self) -> int:             # A = c * d tokens per decision step
        return self.chunk * self.dof

    @property
    def rows(self) -> int:              # R = E * T * A logit rows
        return self.n_env * self.t_steps * self.a_tok

    @property
    def env_steps(self) -> int:         # Eq. (2) numerator for one window: N_env * N_es
        return self.n_env * self.n_es


CONFIGS = {
    "tiny": WorkloadConfig("tiny", 0, 8, 32, 1, 256, "f32", "grpo", group_size=4,
                           reward_kind="sparse_once", lag_probs=(0.6, 0.3, 0.1),
                           faults=True),
    "libero_spatial_oft": WorkloadConfig("libero_spatial_oft", 1, 64, 512, 8, 32000, "bf16",
                                         "grpo", group_size=8, reward_kind="sparse_once",
                                         lag_probs=(0.5, 0.5)),
    "libero10_long": WorkloadConfig("libero10_long", 2, 256, 1024, 8, 32000, "bf16", "gae",
                                    whiten=True, gpus=(2, 4), reward_kind="autoreset",
                                    lag_probs=(0.495, 0.495, 0.01)),
    "maniskill_ppo_gae": WorkloadConfig("maniskill_ppo_gae", 3, 1024, 80, 8, 32000, "bf16",
                                        "gae", whiten=True, gpus=(8,), reward_kind="dense",
                                        lag_probs=(1.0,)),
    "grpo_span": WorkloadConfig("grpo_span", 4, 2048, 512, 8, 32000, "bf16", "grpo",
                                group_size=8, interleave_groups=True, gpus=(8,),
                                reward_kind="outcome", lag_probs=(0.5, 0.5)),
}


def scaled(cfg: WorkloadConfig, **kw) -> WorkloadConfig:
    """Same recipe, different sizes (e.g. a reduced LIBERO shape the oracle finishes)."""
    d = dict(cfg.__dict__)
    d.update(kw)
    return WorkloadConfig(**d)


def seed_for(cfg: WorkloadConfig, salt: int = 0) -> int:
    return SEED_BASE + 100 * cfg.index + salt


# --------------------------------------------------------------------------------------
# Trajectories (per decision step), global over all envs so that any sharding sees the
# same values for the same env.
# --------------------------------------------------------------------------------------

@dataclass
class Trajectories:
    cfg: WorkloadConfig
    reward: np.ndarray        # f32 [E, T]  (chunk's env-step rewards, reading R1)
    done: np.ndarray          # u8  [E, T]
    value: np.ndarray         # f32 [E, T]  value-head output of the rollout
    version: np.ndarray       # i32 [E, T]  policy version that produced the step
    tokens: np.ndarray        # i32 [E, T, A] sampled action tokens (targets)
    peak_bin: np.ndarray      # i32 [E, T, A] the row's high-probability bin
    behav_noise: np.ndarray   # f32 [E, T, A] rollout-vs-trainer numeric drift
    last_value: np.ndarray    # f32 [E] bootstrap value at window end
    group_id: np.ndarray      # i32 [E] GRPO group of each env
    present: np.ndarray       # bool [E, T] step is delivered at all (False => never arrives)
    crafted: dict = field(default_factory=dict)   # kind -> list of global row ids


def _episode_layout(cfg, rng, E, T):
    """done flags, reward, value per step following the config's reward recipe."""
    reward = np.zeros((E, T), np.float32)
    done = np.zeros((E, T), np.uint8)
    seg_start = np.zeros((E, T), bool)       # first step of an episode segment
    seg_start[:, 0] = True
    if cfg.reward_kind == "sparse_once":
        # LIBERO: success w.p. 0.6 at a uniform step in [0.3T, T): reward 1, done there;
        # the env autoresets and the rest of the window is a new (timed-out) episode.
        succ = rng.random(E) < 0.6
        lo = int(0.3 * T)
        ts = rng.integers(lo, T, size=E)
        for e in range(E):
            if succ[e]:
                reward[e, ts[e]] = 1.0
                done[e, ts[e]] = 1
                if ts[e] + 1 < T:
                    seg_start[e, ts[e] + 1] = True
        value = rng.random((E, T), dtype=np.float32)
    elif cfg.reward_kind == "autoreset":
        # LIBERO-10 long horizon: episodes back to back, lengths ~ U[T/8, T/2].
        for e in range(E):
            t = 0
            while t < T:
                L = int(rng.integers(max(1, T // 8), max(2, T // 2) + 1))
                end = min(T, t + L) - 1
                if t + L <= T:
                    done[e, end] = 1
                    if rng.random() < 0.5:
                        reward[e, end] = 1.0
                    if end + 1 < T:
                        seg_start[e, end + 1] = True
                t = end + 1
        value = rng.random((E, T), dtype=np.float32)
    elif cfg.reward_kind == "dense":
        # ManiSkill: dense r ~ U(0, 0.1) + 1 on success (w.p. 0.7 at a uniform step => done).
        reward = (rng.random((E, T)) * 0.1).astype(np.float32)
        succ = rng.random(E) < 0.7
        ts = rng.integers(0, T, size=E)
        for e in range(E):
            if succ[e]:
                reward[e, ts[e]] += np.float32(1.0)
                done[e, ts[e]] = 1
                if ts[e] + 1 < T:
                    seg_start[e, ts[e] + 1] = True
        value = (0.5 + 0.2 * rng.standard_normal((E, T))).astype(np.float32)
    elif cfg.reward_kind == "outcome":
        # GRPO: binary outcome reward at the last step, per-group success prob ~ U(0.2, 0.9).
        G = max(1, cfg.group_size)
        n_groups = max(1, E // G)
        p_group = rng.uniform(0.2, 0.9, size=n_groups)
        gid = _group_ids(cfg, E)
        succ = rng.random(E) < p_group[gid % n_groups]
        reward[:, T - 1] = succ.astype(np.float32)
        done[:, T - 1] = 1
        value = rng.random((E, T), dtype=np.float32)
    else:
        raise ValueError(cfg.reward_kind)
    return reward, done, value.astype(np.float32), seg_start


def _group_ids(cfg, E):
    G = max(1, cfg.group_size)
    if cfg.interleave_groups:
        # every group spans all ranks: g(e) = e mod (E/G)
        return (np.arange(E) % max(1, E // G)).astype(np.int32)
    return (np.arange(E) // G).astype(np.int32)


def make_trajectories(cfg: WorkloadConfig, seed: int | None = None) -> Trajectories:
    rng = np.random.default_rng(seed_for(cfg) if seed is None else seed)
    E, T, A, V = cfg.n_env, cfg.t_steps, cfg.a_tok, cfg.vocab
    reward, done, value, seg_start = _episode_layout(cfg, rng, E, T)

    # policy version per episode segment (trajectory-level version pinning)
    lag_p = np.asarray(cfg.lag_probs, dtype=np.float64)
    lag_p = lag_p / lag_p.sum()
    version = np.zeros((E, T), np.int32)
    for e in range(E):
        lag = 0
        for t in range(T):
            if seg_start[e, t]:
                lag = int(rng.choice(len(lag_p), p=lag_p))
            version[e, t] = CUR_VERSION - lag

    W = min(ACTION_BINS, V)
    peak_bin = (V - W + rng.integers(0, W, size=(E, T, A))).astype(np.int32)
    hit = rng.random((E, T, A)) < 0.6
    other = (V - W + rng.integers(0, W, size=(E, T, A))).astype(np.int32)
    tokens = np.where(hit, peak_bin, other).astype(np.int32)

    lag_tok = (CUR_VERSION - version)[:, :, None]
    sd = np.where(lag_tok == 0, 0.01, 0.1)
    behav_noise = (rng.standard_normal((E, T, A)) * sd).astype(np.float32)

    last_value = rng.random(E, dtype=np.float32)
    present = np.ones((E, T), bool)
    crafted = {}
    if cfg.faults:
        # a few steps never arrive (R8: unfilled slots)
        for _ in range(3):
            present[rng.integers(0, E), rng.integers(1, T)] = False
    traj = Trajectories(cfg, reward, done, value, version, tokens, peak_bin, behav_noise,
                        last_value, _group_ids(cfg, E), present, crafted)
    _craft_rows(traj, rng)
    return traj


CRAFT_KINDS = ("uniform", "saturated", "tied_max", "neg_inf_cols", "ignore")


def _craft_rows(traj: Trajectories, rng):
    """Crafted rows at fixed, delivered positions (edge cases of S3)."""
    cfg = traj.cfg
    E, T, A = cfg.n_env, cfg.t_steps, cfg.a_tok
    if E * T * A < 64:
        return
    pos = 0
    for kind in CRAFT_KINDS:
        rows = []
        for k in range(2):
            # spread crafted rows over different envs/steps; skip undelivered steps
            while True:
                r = (pos * 7919 + 13) % (E * T * A)
                pos += 1
                e, t = r // (T * A), (r // A) % T
                if traj.present[e, t]:
                    break
            rows.append(r)
            if kind == "ignore":
                traj.tokens.reshape(-1)[r] = -1
        traj.crafted[kind] = rows


# --------------------------------------------------------------------------------------
# Records: one per delivered decision step, in out-of-order arrival order.
# --------------------------------------------------------------------------------------

@dataclass
class Records:
    env_id: np.ndarray        # i32 [M]
    step: np.ndarray          # i32 [M]
    version: np.ndarray       # i32 [M]
    reward: np.ndarray        # f32 [M]
    done: np.ndarray          # u8  [M]
    value: np.ndarray         # f32 [M]
    tokens: np.ndarray        # i32 [M, A]
    behav_noise: np.ndarray   # f32 [M, A]
    fault: np.ndarray         # i8 [M] 0 ok, 1 dup-resend, 2 oob, 3 future version

    @property
    def n(self) -> int:
        return int(self.env_id.shape[0])

    def take(self, idx) -> "Records":
        return Records(*(getattr(self, f)[idx] for f in
                         ("env_id", "step", "version", "reward", "done", "value",
                          "tokens", "behav_noise", "fault")))


def make_records(traj: Trajectories, env_lo: int = 0, env_hi: int | None = None,
                 seed: int | None = None) -> Records:
    """Records for envs [env_lo, env_hi) with LOCAL env ids, in arrival order.

    Arrival: per-env decision-step completion times are cumulative sums of
    LogNormalShifted(mu=3.0, sigma=0.5, shift=20 ms) latencies; records are sorted
    by (time, env, step) — out of order across envs.
    """
    cfg = traj.cfg
    env_hi = cfg.n_env if env_hi is None else env_hi
    rng = np.random.default_rng((seed_for(cfg, 1) if seed is None else seed) + env_lo)
    E, T = env_hi - env_lo, cfg.t_steps
    lat = 20.0 + rng.lognormal(3.0, 0.5, size=(E, T))
    done_at = np.cumsum(lat, axis=1)
    ee, tt = np.meshgrid(np.arange(E), np.arange(T), indexing="ij")
    keep = traj.present[env_lo:env_hi]
    order = np.lexsort((tt[keep], ee[keep], done_at[keep]))
    e_sel, t_sel = ee[keep][order], tt[keep][order]
    g = e_sel + env_lo
    rec = Records(
        env_id=e_sel.astype(np.int32), step=t_sel.astype(np.int32),
        version=traj.version[g, t_sel].copy(), reward=traj.reward[g, t_sel].copy(),
        done=traj.done[g, t_sel].copy(), value=traj.value[g, t_sel].copy(),
        tokens=traj.tokens[g, t_sel].copy(), behav_noise=traj.behav_noise[g, t_sel].copy(),
        fault=np.zeros(len(g), np.int8))
    if cfg.faults and rec.n > 16:
        rec = _inject_faults(rec, cfg, rng)
    return rec


def _inject_faults(rec: Records, cfg, rng) -> Records:
    """3 duplicates (2 same-version resends with changed payload, 1 stale resend),
    2 out-of-range ids, 1 future version (SURVEY §8(d) tiny)."""
    M = rec.n
    extra = []
    for kind, src in (("resend", 3), ("resend", M // 2), ("stale", M // 3),
                      ("oob_env", 5), ("oob_step", 7), ("future", 11)):
        r = rec.take(np.array([src]))
        if kind == "resend":
            r.reward = r.reward + np.float32(0.25)
            r.behav_noise = r.behav_noise + np.float32(0.001)
            r.fault[:] = 1
        elif kind == "stale":
            r.version = r.version - 1
            r.reward = r.reward - np.float32(0.5)
            r.fault[:] = 1
        elif kind == "oob_env":
            r.env_id[:] = cfg.n_env + 3
            r.fault[:] = 2
        elif kind == "oob_step":
            r.step[:] = -1
            r.fault[:] = 2
        elif kind == "future":
            r.version[:] = CUR_VERSION + 1
            r.fault[:] = 3
        extra.append(r)
    parts = [rec] + extra
    cat = Records(*(np.concatenate([getattr(p, f) for p in parts]) for f in
                    ("env_id", "step", "version", "reward", "done", "value", "tokens",
                     "behav_noise", "fault")))
    # faults arrive late but interleaved with the tail of the normal stream
    order = np.arange(cat.n)
    tail = order[M - 24:]
    rng.shuffle(tail)
    order[M - 24:] = tail
    return cat.take(order)


def record_rows(rec: Records, cfg: WorkloadConfig, n_env_local: int) -> np.ndarray:
    """Global-in-shard logit row ids [M, A] of each record's tokens; -1 for out-of-range."""
    T, A = cfg.t_steps, cfg.a_tok
    ok = (rec.env_id >= 0) & (rec.env_id < n_env_local) & (rec.step >= 0) & (rec.step < T)
    base = (rec.env_id.astype(np.int64) * T + rec.step) * A
    rows = base[:, None] + np.arange(A)[None, :]
    return np.where(ok[:, None], rows, -1)


def arrival_chunks(n: int, b_max: int = B_MAX):
    """Slices of the arrival stream as delivered by the Eq. (1) trigger (size B_max)."""
    return [slice(i, min(n, i + b_max)) for i in range(0, n, b_max)]


# --------------------------------------------------------------------------------------
# Logits (the VLA forward's output; synthetic). Generated per env so any sharding sees
# identical rows for the same env.
# --------------------------------------------------------------------------------------

def gen_logits(cfg: WorkloadConfig, traj: Trajectories, env_lo: int, env_hi: int,
               device="cpu", out=None, torch_dtype=None):
    """Logits [ (env_hi-env_lo)*T*A, V ] in cfg.dtype on `device`.

    Recipe: x ~ N(0, s^2) over the vocabulary with s = 1.5 (bf16 configs)
    or 2.0 (tiny); the action window [V-256, V) is shifted by +2.5 (bf16 configs), and
    the row's peak bin gets +4. Crafted rows overwrite whole rows.
    """
    import torch
    T, A, V = cfg.t_steps, cfg.a_tok, cfg.vocab
    dt = torch_dtype or (torch.bfloat16 if cfg.dtype == "bf16" else torch.float32)
    R_env = T * A
    n = (env_hi - env_lo) * R_env
    if out is None:
        out = torch.empty((n, V), dtype=dt, device=device)
    W = min(ACTION_BINS, V)
    s = 2.0 if cfg.dtype == "f32" else 1.5
    shift = 0.0 if cfg.dtype == "f32" else 2.5
    gen = torch.Generator(device=device)
    for k, e in enumerate(range(env_lo, env_hi)):
        gen.manual_seed(seed_for(cfg, 1000 + e))
        x = torch.randn((R_env, V), generator=gen, device=device, dtype=torch.float32)
        x.mul_(s)
        if shift:
            x[:, V - W:] += shift
        pk = torch.from_numpy(traj.peak_bin[e].reshape(-1).astype(np.int64)).to(device)
        x[torch.arange(R_env, device=device), pk] += 4.0
        out[k * R_env:(k + 1) * R_env].copy_(x)
    _apply_crafted(cfg, traj, env_lo, env_hi, out)
    return out


def _apply_crafted(cfg, traj, env_lo, env_hi, out):
    import torch
    T, A, V = cfg.t_steps, cfg.a_tok, cfg.vocab
    lo, hi = env_lo * T * A, env_hi * T * A
    flat_tok = traj.tokens.reshape(-1)
    for kind, rows in traj.crafted.items():
        for r in rows:
            if not (lo <= r < hi):
                continue
            rl = r - lo
            a = int(flat_tok[r])
            if kind == "uniform":
                out[rl].fill_(0.0)
            elif kind == "saturated":
                out[rl].fill_(-30.0)
                out[rl, a] = 30.0
            elif kind == "tied_max":
                out[rl].fill_(-1.0)
                out[rl, a] = 5.0
                out[rl, (a + 17) % V] = 5.0
                out[rl, (a + 101) % V] = 5.0
            elif kind == "neg_inf_cols":
                cols = torch.tensor([(a + 1) % V, (a + 2) % V, (a + 50) % V, (a + 3 * V // 4) % V])
                out[rl, cols.to(out.device)] = float("-inf")
            # "ignore": target -1 (in tokens); logits left as drawn
    return out


# --------------------------------------------------------------------------------------
# NEXT-3: request traffic for the Eq. (1) dynamic batching scheduler (§3.2).
# Random draws only; the closed loop (who is batched when) is run by the caller's batcher.
# --------------------------------------------------------------------------------------
# OpenVLA-OFT on LIBERO: third-person + wrist 224x224 RGB uint8 images and an 8-float
# proprio state per observation (P:99 OFT; 16-byte multiple)
OBS_BYTES_OFT = 2 * 224 * 224 * 3 + 8 * 4


@dataclass
class BatcherTraffic:
    n_env: int
    step_ticks: np.ndarray    # i64 [n_env, n_cycles] env step durations in ticks (1 tick = 1 ms)
    infer_ticks: np.ndarray   # i64 [n_batches_max] inference latency of the k-th batch
    enq_lag: np.ndarray       # i64 [n_env, n_cycles] enqueue_time = offer tick - lag (0..2)
    fault_u: np.ndarray       # f64 [ticks, 4] uniforms deciding injected bad offers per tick
    fault_env: np.ndarray     # i64 [ticks, 4] raw env draws for those offers
    seed: int


def batcher_traffic(n_env: int, n_cycles: int, ticks: int, seed: int,
                    mu: float = 3.0, sigma: float = 0.5, shift: int = 20,
                    infer_lo: int = 5, infer_hi: int = 15) -> BatcherTraffic:
    """Env step latencies ~ LogNormalShifted(mu, sigma, shift) ms rounded to ticks;
    inference latency per batch ~ U[infer_lo, infer_hi] ticks; per tick four uniforms and
    env draws that the caller turns into bad offers (out-of-range env, future time,
    repeated env) at its chosen rate."""
    rng = np.random.default_rng(seed)
    step = np.rint(shift + rng.lognormal(mu, sigma, (n_env, n_cycles))).astype(np.int64)
    infer = rng.integers(infer_lo, infer_hi + 1, n_env * n_cycles + 1).astype(np.int64)
    lag = rng.choice([0, 0, 0, 1, 2], size=(n_env, n_cycles)).astype(np.int64)
    return BatcherTraffic(n_env, step, infer, lag, rng.random((ticks, 4)),
                          rng.integers(0, 1 << 30, (ticks, 4)).astype(np.int64), seed)


def payload_bytes(seed: int, env: int, cycle: int, obs_bytes: int) -> np.ndarray:
    """The observation an env offers in a given cycle: seeded random bytes."""
    r = np.random.default_rng([seed, env, cycle])
    return r.integers(0, 256, obs_bytes, dtype=np.uint8)
