"""Thin Python binding of the C ABI (include/rlvla.h), same names as the C entry points.

Argument marshalling only: torch tensors (device memory the caller owns) are turned into
raw pointers, the current CUDA stream is passed through, and a non-OK status raises.
Every step of the path runs in librlvla.so's kernels; nothing here computes.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _abi as A
from ._abi import lib


class RlvlaError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().rlvla_status_string(status).decode()
        super().__init__(f"{where}: status {status} ({msg})")
        self.status = status


def _ptr(t) -> int | None:
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"expected a torch.Tensor, got {type(t)}")
    return t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        if not torch.cuda.is_available():
            return None
        stream = torch.cuda.current_stream()
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _check(st: int, where: str, check: bool) -> int:
    if check and st != A.OK:
        raise RlvlaError(st, where)
    return st


# --------------------------------------------------------------------------------------
# containers (device memory owned by the caller; allocation is plumbing)
# --------------------------------------------------------------------------------------
@dataclass
class TrajectoryBuffer:
    """rlvla_traj_buffer: one rank's shard, [n_env, t_steps] steps x a_tok tokens."""
    n_env: int
    t_steps: int
    a_tok: int
    slot_key: torch.Tensor     # int64 view of uint64 [E, T]
    reward: torch.Tensor       # f32 [E, T]
    done: torch.Tensor         # u8 [E, T]
    value: torch.Tensor        # f32 [E, T]
    version: torch.Tensor      # i32 [E, T]
    tokens: torch.Tensor       # i32 [E, T, A]
    logp_behav: torch.Tensor   # f32 [E, T, A]

    @classmethod
    def allocate(cls, n_env, t_steps, a_tok, device="cuda"):
        z = lambda *s, dt: torch.zeros(*s, dtype=dt, device=device)  # noqa: E731
        return cls(n_env, t_steps, a_tok, z(n_env, t_steps, dt=torch.int64),
                   z(n_env, t_steps, dt=torch.float32), z(n_env, t_steps, dt=torch.uint8),
                   z(n_env, t_steps, dt=torch.float32), z(n_env, t_steps, dt=torch.int32),
                   z(n_env, t_steps, a_tok, dt=torch.int32),
                   z(n_env, t_steps, a_tok, dt=torch.float32))

    def reset(self):
        self.slot_key.zero_()

    def c(self) -> A.c_traj_buffer:
        return A.c_traj_buffer(self.n_env, self.t_steps, self.a_tok, _ptr(self.slot_key),
                               _ptr(self.reward), _ptr(self.done), _ptr(self.value),
                               _ptr(self.version), _ptr(self.tokens), _ptr(self.logp_behav))


@dataclass
class StepBatch:
    """rlvla_step_batch: M records in arrival order (device tensors)."""
    env_id: torch.Tensor      # i32 [M]
    step: torch.Tensor        # i32 [M]
    version: torch.Tensor     # i32 [M]
    reward: torch.Tensor      # f32 [M]
    done: torch.Tensor        # u8 [M]
    value: torch.Tensor       # f32 [M]
    tokens: torch.Tensor      # i32 [M, A]
    logp_behav: torch.Tensor  # f32 [M, A]

    @property
    def n(self) -> int:
        return int(self.env_id.shape[0])

    def slice(self, sl: slice) -> "StepBatch":
        return StepBatch(*(getattr(self, f)[sl] for f in
                           ("env_id", "step", "version", "reward", "done", "value", "tokens",
                            "logp_behav")))

    def c(self) -> A.c_step_batch:
        return A.c_step_batch(self.n, _ptr(self.env_id), _ptr(self.step), _ptr(self.version),
                              _ptr(self.reward), _ptr(self.done), _ptr(self.value),
                              _ptr(self.tokens), _ptr(self.logp_behav))


def workspace(n_env_global: int = 1, rows: int = 0, t_steps: int = 0, device="cuda"):
    """Zero-filled, 256-byte aligned workspace of rlvla_workspace_bytes(...) bytes."""
    nb = int(lib().rlvla_workspace_bytes(rows, n_env_global, t_steps))
    return torch.zeros(nb + 256, dtype=torch.uint8, device=device)


def _ws_ptr(ws):
    if ws is None:
        return None, 0
    p = ws.data_ptr()
    off = (-p) % 256
    return p + off, ws.numel() - off


# --------------------------------------------------------------------------------------
# entry points
# --------------------------------------------------------------------------------------
def rlvla_scatter_steps(buf: TrajectoryBuffer, rec: StepBatch, cur_version: int,
                        seq_base: int, counters: torch.Tensor, stream=None, check=True) -> int:
    b, r = buf.c(), rec.c()
    st = lib().rlvla_scatter_steps(ctypes.byref(b), ctypes.byref(r), cur_version, seq_base,
                                   _ptr(counters), _stream(stream))
    return _check(st, "rlvla_scatter_steps", check)


def adv_params(mode, *, gamma=0.99, lam=0.95, whiten=False, whiten_eps=1e-8, group_id=None,
               group_size=0, std_unbiased=True, grpo_eps=1e-6, env_offset=0, n_env_global=0,
               cur_version=0, max_staleness=1, boot_value=None) -> A.c_adv_params:
    p = A.c_adv_params(A.ADV_GAE if mode == "gae" else A.ADV_GRPO, gamma, lam, int(whiten),
                       whiten_eps, _ptr(group_id), group_size, int(std_unbiased), grpo_eps,
                       env_offset, n_env_global, cur_version, max_staleness, _ptr(boot_value))
    p._keep = (group_id, boot_value)  # the struct holds raw pointers: keep the tensors alive
    return p


def rlvla_advantages(buf: TrajectoryBuffer, last_value, params: A.c_adv_params, adv, ret,
                     stats, ws, comm=None, stream=None, check=True) -> int:
    b = buf.c()
    wp, wn = _ws_ptr(ws)
    st = lib().rlvla_advantages(ctypes.byref(b), _ptr(last_value), ctypes.byref(params),
                                _ptr(adv), _ptr(ret), _ptr(stats), wp, wn,
                                comm.handle if comm is not None else None, _stream(stream))
    return _check(st, "rlvla_advantages", check)


def logits_desc(x: torch.Tensor, vocab: int | None = None) -> A.c_logits:
    if x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("logits must be a 2-D row-major tensor")
    dt = {torch.float32: A.F32, torch.bfloat16: A.BF16}[x.dtype]
    return A.c_logits(_ptr(x), dt, x.shape[0], vocab or x.shape[1], x.stride(0))


def ppo_args(*, logp_behav, adv, version, slot_key, a_tok, cur_version, max_staleness=1,
             eps_low=0.2, eps_high=0.2, is_cap=0.0, logp_prox=None, tok_denominator=0.0,
             adv_stats=None, out_grad_logp=None, out_loss_tok=None,
             accumulate=False, dual_clip=0.0, logp_ref=None, kl_coef=0.0, ent_coef=0.0,
             ratio_level=0) -> A.c_ppo_args:
    a = A.c_ppo_args(_ptr(logp_behav), _ptr(logp_prox), _ptr(adv), _ptr(version),
                     _ptr(slot_key), a_tok, cur_version, max_staleness, eps_low, eps_high,
                     is_cap, tok_denominator, _ptr(adv_stats), _ptr(out_grad_logp),
                     _ptr(out_loss_tok), int(accumulate), dual_clip, _ptr(logp_ref), kl_coef,
                     ent_coef, ratio_level)
    # the struct holds raw pointers: keep the tensors alive as long as the struct
    a._keep = (logp_behav, logp_prox, adv, version, slot_key, adv_stats, out_grad_logp,
               out_loss_tok, logp_ref)
    return a


def rlvla_logprob_fwd_bwd(x: torch.Tensor, target, logp=None, lse=None, grad_logp=None,
                          fused: A.c_ppo_args | None = None, dlogits=None, stats=None, ws=None,
                          comm=None, stream=None, vocab=None, check=True) -> int:
    xd = logits_desc(x, vocab)
    wp, wn = _ws_ptr(ws)
    st = lib().rlvla_logprob_fwd_bwd(ctypes.byref(xd), _ptr(target), _ptr(logp), _ptr(lse),
                                     _ptr(grad_logp),
                                     ctypes.byref(fused) if fused is not None else None,
                                     _ptr(dlogits), _ptr(stats), wp, wn,
                                     comm.handle if comm is not None else None, _stream(stream))
    return _check(st, "rlvla_logprob_fwd_bwd", check)


def rlvla_ppo_loss(logp, target, args: A.c_ppo_args, grad_logp, loss_tok=None, stats=None,
                   ws=None, comm=None, stream=None, check=True) -> int:
    wp, wn = _ws_ptr(ws)
    st = lib().rlvla_ppo_loss(_ptr(logp), logp.numel(), _ptr(target), ctypes.byref(args),
                              _ptr(grad_logp), _ptr(loss_tok), _ptr(stats), wp, wn,
                              comm.handle if comm is not None else None, _stream(stream))
    return _check(st, "rlvla_ppo_loss", check)


def rlvla_value_loss(v_new, v_old, ret, slot_key, version, cur_version, grad_v, *,
                     max_staleness=1, clip_eps=0.2, denominator=0.0, loss_step=None,
                     stats=None, ws=None, comm=None, stream=None, check=True) -> int:
    wp, wn = _ws_ptr(ws)
    st = lib().rlvla_value_loss(_ptr(v_new), _ptr(v_old), _ptr(ret), _ptr(slot_key),
                                _ptr(version), v_new.numel(), cur_version, max_staleness,
                                clip_eps, denominator, _ptr(grad_v), _ptr(loss_step),
                                _ptr(stats), wp, wn,
                                comm.handle if comm is not None else None, _stream(stream))
    return _check(st, "rlvla_value_loss", check)


@dataclass
class BatchQueue:
    """rlvla_batch_queue: one rollout worker's Eq. (1) request queue (NEXT-3)."""
    n_env: int
    obs_bytes: int
    obs: torch.Tensor | None   # u8 [n_env (+ max_batch), obs_bytes] observation rows
    ring_env: torch.Tensor     # i32 [n_env]
    ring_time: torch.Tensor    # i64 [n_env]
    pending: torch.Tensor      # u8 [n_env]
    state: torch.Tensor        # i64 [8] head, tail, anchor, batches, batch row, reserved
    obs_fifo: int = 0
    max_batch: int = 0

    @classmethod
    def allocate(cls, n_env, obs_bytes=0, device="cuda", obs_fifo=False, max_batch=0):
        z = lambda *s, dt: torch.zeros(*s, dtype=dt, device=device)  # noqa: E731
        rows = n_env + (max_batch if obs_fifo else 0)
        obs = z(rows, obs_bytes, dt=torch.uint8) if obs_bytes > 0 else None
        return cls(n_env, obs_bytes, obs, z(n_env, dt=torch.int32), z(n_env, dt=torch.int64),
                   z(n_env, dt=torch.uint8), z(8, dt=torch.int64), int(obs_fifo), int(max_batch))

    def batch_rows(self, b: int) -> torch.Tensor:
        """obs_fifo: the last emitted batch (b rows), a view into obs (no copy)."""
        r0 = int(self.state[4].item())
        return self.obs[r0:r0 + b]

    def c(self) -> A.c_batch_queue:
        return A.c_batch_queue(self.n_env, self.obs_bytes, _ptr(self.obs), _ptr(self.ring_env),
                               _ptr(self.ring_time), _ptr(self.pending), _ptr(self.state),
                               self.obs_fifo, self.max_batch)


def rlvla_batch_offer(q: BatchQueue, env_id, enqueue_time, now: int, counters, *, obs_src=None,
                      ws=None, stream=None, check=True) -> int:
    """Offers in arrival order; more than 1024 requests go as consecutive calls with the
    same `now` (identical semantics, see rlvla.h)."""
    qc = q.c()
    wp, wn = _ws_ptr(ws)
    n = int(env_id.numel())
    st = A.OK
    for i0 in range(0, max(n, 1), 1024):
        i1 = min(n, i0 + 1024)
        src = None if obs_src is None else obs_src[i0:i1]
        st = lib().rlvla_batch_offer(ctypes.byref(qc), _ptr(env_id[i0:i1]), _ptr(enqueue_time[i0:i1]),
                                     i1 - i0, now, _ptr(src), _ptr(counters), wp, wn,
                                     _stream(stream))
        _check(st, "rlvla_batch_offer", check)
    return st


def rlvla_batch_poll(q: BatchQueue, now: int, b_max: int, t_max: int, out_env, out_time, out_n, *,
                     out_obs=None, ws=None, stream=None, check=True) -> int:
    qc = q.c()
    wp, wn = _ws_ptr(ws)
    st = lib().rlvla_batch_poll(ctypes.byref(qc), now, b_max, t_max, _ptr(out_env), _ptr(out_time),
                                _ptr(out_obs), _ptr(out_n), wp, wn, _stream(stream))
    return _check(st, "rlvla_batch_poll", check)


@dataclass
class GaussChain:
    """rlvla_gauss_chain (NEXT-4): K Gaussian denoising transitions per decision step."""
    mu: torch.Tensor                    # [rows, K, D] f32 | bf16 denoiser means
    x: torch.Tensor                     # [rows, K, D] f32 sampled x_{k+1}
    sigma_k: torch.Tensor | None = None  # [K] f32 std schedule
    log_std: torch.Tensor | None = None  # [rows, K, D] f32 learned ln sigma

    def c(self) -> A.c_gauss_chain:
        R, K, D = self.mu.shape
        dt = A.BF16 if self.mu.dtype == torch.bfloat16 else A.F32
        return A.c_gauss_chain(_ptr(self.mu), dt, _ptr(self.x), _ptr(self.sigma_k),
                               _ptr(self.log_std), R, K, D)


def rlvla_flow_logprob(chain: GaussChain, logp=None, grad_logp=None, fused: A.c_ppo_args | None = None,
                       dmu=None, dlog_std=None, stats=None, ws=None, comm=None, stream=None,
                       check=True) -> int:
    cc = chain.c()
    wp, wn = _ws_ptr(ws)
    st = lib().rlvla_flow_logprob(ctypes.byref(cc), _ptr(logp), _ptr(grad_logp),
                                  ctypes.byref(fused) if fused is not None else None, _ptr(dmu),
                                  _ptr(dlog_std), _ptr(stats), wp, wn,
                                  comm.handle if comm is not None else None, _stream(stream))
    return _check(st, "rlvla_flow_logprob", check)


def rlvla_workspace_bytes(rows: int, n_env_global: int, t_steps: int) -> int:
    return int(lib().rlvla_workspace_bytes(rows, n_env_global, t_steps))


def rlvla_set_reserved_sms(n: int) -> int:
    """SMs the persistent kernels leave free for other streams; returns the previous value."""
    return int(lib().rlvla_set_reserved_sms(int(n)))


def rlvla_abi_version() -> int:
    return int(lib().rlvla_abi_version())


def rlvla_nccl_version() -> int:
    return int(lib().rlvla_nccl_version())


class Comm:
    """rlvla_comm: over NCCL (from_process_group; the 128-byte unique id travels over a torch
    ProcessGroup) or P2P-only (p2p_from_process_group; CUDA IPC mailbox handles travel over
    the ProcessGroup, no NCCL: several ranks may share a GPU)."""

    def __init__(self, handle, nranks, rank):
        self.handle, self.nranks, self.rank = handle, nranks, rank

    @staticmethod
    def _group_info(group):
        import torch.distributed as dist
        return dist.get_rank(group), dist.get_world_size(group), dist.get_backend(group)

    @classmethod
    def from_process_group(cls, group=None, device=None):
        import torch.distributed as dist
        rank, n, backend = cls._group_info(group)
        uid = (ctypes.c_ubyte * 128)()
        if rank == 0:
            _check(lib().rlvla_comm_unique_id(uid), "rlvla_comm_unique_id", True)
        dev = device if (backend == "nccl") else "cpu"
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
        # group_src: the GROUP's rank 0 (src would be a global rank)
        dist.broadcast(t, group_src=0, group=group)
        raw = bytes(t.cpu().tolist())
        uid2 = (ctypes.c_ubyte * 128).from_buffer_copy(raw)
        h = ctypes.c_void_p()
        _check(lib().rlvla_comm_init(uid2, n, rank, ctypes.byref(h)), "rlvla_comm_init", True)
        return cls(h, n, rank)

    @classmethod
    def p2p_from_process_group(cls, group=None):
        """P2P-only communicator on the current CUDA device: every rank allocates its mailbox,
        the IPC handles are allgathered over `group` (any backend, e.g. gloo), every rank maps
        its peers, and the outcome is agreed over `group` (any failure raises everywhere)."""
        import torch.distributed as dist
        rank, n, _ = cls._group_info(group)
        hb = A.P2P_HANDLE_BYTES
        mine = (ctypes.c_ubyte * hb)()
        h = ctypes.c_void_p()
        st = lib().rlvla_comm_init_p2p(n, rank, mine, ctypes.byref(h))
        recs = [None] * n
        dist.all_gather_object(recs, (int(st), bytes(mine)), group=group)
        ok = all(r[0] == A.OK for r in recs)
        if ok:
            allh = (ctypes.c_ubyte * (hb * n)).from_buffer_copy(b"".join(r[1] for r in recs))
            ok = lib().rlvla_comm_connect_p2p(h, allh) == A.OK
        votes = [None] * n
        dist.all_gather_object(votes, bool(ok), group=group)
        if not all(votes):
            if h:
                lib().rlvla_comm_destroy(h)
            raise RlvlaError(A.ERR_CUDA if st == A.OK else st,
                             f"rlvla_comm_init_p2p/connect (ranks ok: {votes})")
        return cls(h, n, rank)

    @property
    def p2p(self) -> bool:
        """Loss statistics reduced in-kernel over NVLink peer memory (else NCCL)."""
        return bool(self.handle) and bool(lib().rlvla_comm_p2p_enabled(self.handle))

    def destroy(self):
        if self.handle:
            lib().rlvla_comm_destroy(self.handle)
            self.handle = None
