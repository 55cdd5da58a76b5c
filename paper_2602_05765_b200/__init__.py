"""B200-native rollout-to-loss path of RL-VLA^3 (arXiv 2602.05765).

The C ABI (include/rlvla.h, librlvla.so — hand-written sm_100a kernels) is the product;
this package is its thin binding plus host-side sharding helpers. Importing it does not
load the library; the first call does, and raises if librlvla.so has not been built.
"""
from .api import (  # noqa: F401
    BatchQueue, Comm, GaussChain, RlvlaError, StepBatch, TrajectoryBuffer, adv_params, logits_desc,
    ppo_args, rlvla_abi_version, rlvla_advantages, rlvla_batch_offer, rlvla_batch_poll,
    rlvla_flow_logprob,
    rlvla_logprob_fwd_bwd, rlvla_nccl_version, rlvla_ppo_loss, rlvla_scatter_steps,
    rlvla_set_reserved_sms,
    rlvla_value_loss, rlvla_workspace_bytes, workspace)
from . import _abi as abi  # noqa: F401
from . import sharding  # noqa: F401
