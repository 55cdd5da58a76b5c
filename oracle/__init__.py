"""CPU oracle for the RL-VLA^3 rollout-to-loss hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl
reference` legs may import, call or execute anything under `oracle/`. The product path
(`paper_2602_05765_b200`) never imports it and fails loudly without its CUDA library.

Plain, slow, obviously correct: numpy in float64, straightforward loops in the
paper's / textbook's order, no blocking or fusion. It shares no code with the CUDA
path (no common kernels, headers, helpers, tables or constants); the only shared
module is `synth/`, which draws inputs and holds none of the method's arithmetic.

The paper fixes the data semantics but not the math of this path
("PPO", "GRPO", "GAE" never occur in PAPER.md). Every function below
therefore cites both the paper passage that fixes its data contract and the textbook
definition it writes out, and every reading where the paper is silent is listed in
DESIGN.md §2 ("Readings").

Functions and their pins (tests/test_oracle_*.py, all `-m "not gpu"`):

  scatter.scatter_steps      S1  P:62 (§3.1 version), P:75 (§3.2 out-of-order)
                                 (§3.3 trajectory buffer); reading R6 (sequential replay).
      pins: permutation invariance (all 6! orders), conservation, bitwise round trip
            incl. NaN payloads, brute-force duplicate interleavings vs max-key rule.
  advantages.gae             S2a Schulman et al. 2016 (GAE); readings R7, R8.
      pins: constant-reward closed form, gamma*lambda = 1 telescoping, lambda = 0,
            lambda = 1, done-everywhere, brute-force double sum over all 2^T done
            patterns (T <= 10).
  advantages.whiten          S2a reading R9. pins: mean 0 / unbiased std closed form.
  advantages.grpo            S2b Shao et al. 2024 (GRPO); reading R10.
      pins: printed values for {0,1} and {1,0,0,0} groups (unbiased and population),
            zero-sum, affine invariance, all-equal => 0, singleton => 0.
  advantages.episode_return, advantages.grpo_step_adv, advantages.step_counts
                             S2b / pre-loss glue. pins (tests/test_oracle_path.py): a
            hand-built 2-groups-of-4 buffer whose unfilled slots hold junk rewards and stale
            versions, answered by the printed GRPO values and a closed form (SURVEY §8(c)
            S2b (vi)); per-element broadcast table; closed-form counts with stale, future,
            ignored and unfilled steps (plus the brute-force loop in test_oracle_advantages).
  logprob.log_softmax_gather S3  P:39 (§2, action tokens); readings R3, R4, R5.
      pins: sum_j exp(logp_j) = 1, uniform row = -ln V, saturation,
            shift invariance, tied maxima, -inf columns, entropy closed forms.
  logprob.log_softmax_grad   S3 bwd. pins: uniform K=4 gradient (0.75,-0.25,...),
            sum_j dx_j = 0, central finite differences.
  ppo.ppo_loss               S4  P:62 (§3.1 staleness), P:18 (AReaL decoupled objective,
                                 cited only); readings R11-R14.
      pins: clip table, ratio == 1, decoupled(prox = behav) ==
            standard, staleness lag = eta / eta+1 / -1, finite differences of the
            composed loss, micro-batch split invariance.
  path.advantages            S2 on a buffer (valid = slot_key != 0). pins: the GRPO
            brute force above; GAE gamma = lambda = 1 segment counts with a junk-filled unfilled
            slot and whitening against numpy std (ddof = 1); P = 1 vs P = 2, 8 logical shards
            (GRPO bit-identical, whitened GAE within 1e-12: SURVEY §8(c) S2b (vii), S2a (vii)).
  path.token_view            row r <-> token r % A of step r // A, lag = cur - version:
            a hand-built 2 x 3 x 2 buffer with every expected row written out.
  path.loss_and_grad         S3 + S4 composed. pins: torch fp64 autograd of the composed
            objective (tests/test_oracle_next2.py), the clip table and finite differences.
  path.rollout_to_loss       S1..S4 composed. pins: a hand-evaluable 2-env GRPO case
            (counters, A = +-0.707105781, Loss = -A/3, g and dx in closed form) plus the
            Eq. (2) throughput unit (tests/golden/eq2_throughput.csv).

No function here is "parity unpinned".
"""
from . import scatter, advantages, logprob, ppo, path  # noqa: F401
