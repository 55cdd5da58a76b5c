"""ctypes mirror of include/rlvla.h. Loads the in-tree librlvla.so and fails loudly if it
is missing — there is no CPU fallback."""
from __future__ import annotations

import ctypes
import os
import re
from ctypes import POINTER, c_double, c_float, c_int32, c_int64, c_size_t, c_uint64, c_void_p

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# RLVLA_LIB overrides the library path (A/B timing of variant builds in tools/)
LIB_PATH = os.environ.get("RLVLA_LIB") or os.path.join(PKG, "librlvla.so")
HEADER = os.path.join(ROOT, "include", "rlvla.h")

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_CUDA, ERR_NCCL, ERR_DATA = range(6)
F32, BF16 = 0, 1
ADV_GAE, ADV_GRPO = 0, 1
NSTATS = 24
(STAT_N_VALID_STEPS, STAT_SUM_ADV, STAT_SUM_ADV2, STAT_N_TOK, STAT_N_STALE_STEPS,
 STAT_N_BAD_STEPS, STAT_LOSS, STAT_N_CLIPPED, STAT_KL_K3_SUM, STAT_ENTROPY_SUM,
 STAT_RATIO_SUM, STAT_N_LOSS_TOK, STAT_N_STALE_TOK, STAT_N_BAD_TOK, STAT_LOGP_SUM,
 STAT_KL_REF_SUM, STAT_N_DUAL_CLIPPED, STAT_PG_LOSS, STAT_DENOM, STAT_VALUE_LOSS,
 STAT_N_VALUE_CLIPPED, STAT_N_VALUE_STEPS, STAT_VALUE_DENOM, STAT_N_LOSS_STEPS) = range(24)
CNT_OOB, CNT_BAD_VERSION, CNT_DUP, CNT_WRITTEN = range(4)
P2P_HANDLE_BYTES = 64           # RLVLA_P2P_HANDLE_BYTES (cudaIpcMemHandle_t)


class c_traj_buffer(ctypes.Structure):
    _fields_ = [("n_env", c_int32), ("t_steps", c_int32), ("a_tok", c_int32),
                ("slot_key", c_void_p), ("reward", c_void_p), ("done", c_void_p),
                ("value", c_void_p), ("version", c_void_p), ("tokens", c_void_p),
                ("logp_behav", c_void_p)]


class c_step_batch(ctypes.Structure):
    _fields_ = [("n_rec", c_int32), ("env_id", c_void_p), ("step", c_void_p),
                ("version", c_void_p), ("reward", c_void_p), ("done", c_void_p),
                ("value", c_void_p), ("tokens", c_void_p), ("logp_behav", c_void_p)]


class c_adv_params(ctypes.Structure):
    _fields_ = [("mode", c_int32), ("gamma", c_float), ("lam", c_float), ("whiten", c_int32),
                ("whiten_eps", c_float), ("group_id", c_void_p), ("group_size", c_int32),
                ("std_unbiased", c_int32), ("grpo_eps", c_float), ("env_offset", c_int32),
                ("n_env_global", c_int32), ("cur_version", c_int32), ("max_staleness", c_int32),
                ("boot_value", c_void_p)]


class c_logits(ctypes.Structure):
    _fields_ = [("ptr", c_void_p), ("dtype", c_int32), ("rows", c_int64), ("vocab", c_int32),
                ("ld", c_int64)]


class c_ppo_args(ctypes.Structure):
    _fields_ = [("logp_behav", c_void_p), ("logp_prox", c_void_p), ("adv", c_void_p),
                ("version", c_void_p), ("slot_key", c_void_p), ("a_tok", c_int32),
                ("cur_version", c_int32), ("max_staleness", c_int32), ("eps_low", c_float),
                ("eps_high", c_float), ("is_cap", c_float), ("tok_denominator", c_double),
                ("adv_stats", c_void_p), ("out_grad_logp", c_void_p),
                ("out_loss_tok", c_void_p), ("accumulate", c_int32), ("dual_clip", c_float),
                ("logp_ref", c_void_p), ("kl_coef", c_float), ("ent_coef", c_float),
                ("ratio_level", c_int32)]


BCNT_OOB, BCNT_FUTURE, BCNT_DUP, BCNT_ACCEPTED = range(4)


class c_batch_queue(ctypes.Structure):
    _fields_ = [("n_env", c_int32), ("obs_bytes", c_int64), ("obs", c_void_p),
                ("ring_env", c_void_p), ("ring_time", c_void_p), ("pending", c_void_p),
                ("state", c_void_p), ("obs_fifo", c_int32), ("max_batch", c_int32)]


class c_gauss_chain(ctypes.Structure):
    _fields_ = [("mu", c_void_p), ("mu_dtype", c_int32), ("x", c_void_p), ("sigma_k", c_void_p),
                ("log_std", c_void_p), ("rows", c_int64), ("n_steps", c_int32), ("dim", c_int32)]


_SIGS = {
    "rlvla_scatter_steps": (c_int32, [POINTER(c_traj_buffer), POINTER(c_step_batch), c_int32,
                                      c_uint64, c_void_p, c_void_p]),
    "rlvla_advantages": (c_int32, [POINTER(c_traj_buffer), c_void_p, POINTER(c_adv_params),
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p,
                                   c_void_p]),
    "rlvla_logprob_fwd_bwd": (c_int32, [POINTER(c_logits), c_void_p, c_void_p, c_void_p,
                                        c_void_p, POINTER(c_ppo_args), c_void_p, c_void_p,
                                        c_void_p, c_size_t, c_void_p, c_void_p]),
    "rlvla_ppo_loss": (c_int32, [c_void_p, c_int64, c_void_p, POINTER(c_ppo_args), c_void_p,
                                 c_void_p, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    "rlvla_value_loss": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                   c_int32, c_int32, c_float, c_double, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_size_t, c_void_p, c_void_p]),
    "rlvla_batch_offer": (c_int32, [POINTER(c_batch_queue), c_void_p, c_void_p, c_int32, c_int64,
                                    c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "rlvla_batch_poll": (c_int32, [POINTER(c_batch_queue), c_int64, c_int32, c_int64, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "rlvla_flow_logprob": (c_int32, [POINTER(c_gauss_chain), c_void_p, c_void_p, POINTER(c_ppo_args),
                                     c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p,
                                     c_void_p]),
    "rlvla_workspace_bytes": (c_size_t, [c_int64, c_int32, c_int32]),
    "rlvla_comm_unique_id": (c_int32, [c_void_p]),
    "rlvla_comm_init": (c_int32, [c_void_p, c_int32, c_int32, POINTER(c_void_p)]),
    "rlvla_comm_destroy": (c_int32, [c_void_p]),
    "rlvla_comm_p2p_enabled": (c_int32, [c_void_p]),
    "rlvla_comm_init_p2p": (c_int32, [c_int32, c_int32, c_void_p, POINTER(c_void_p)]),
    "rlvla_comm_connect_p2p": (c_int32, [c_void_p, c_void_p]),
    "rlvla_status_string": (ctypes.c_char_p, [c_int32]),
    "rlvla_abi_version": (c_int32, []),
    "rlvla_set_reserved_sms": (c_int32, [c_int32]),
    "rlvla_nccl_version": (c_int32, []),
}


def header_functions(path: str = HEADER) -> list[str]:
    """Every function the C header declares (RLVLA_API ... name(...))."""
    src = open(path).read()
    return re.findall(r"RLVLA_API\s+[\w\s\*]+?\b(rlvla_\w+)\s*\(", src)


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2602_05765_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("RLVLA_LIB") and not hasattr(L, name):
                continue  # an older revision under A/B timing (tools/ab_variants.py)
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
