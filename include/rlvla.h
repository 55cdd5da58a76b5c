/*
 * rlvla.h — C ABI of the B200 rollout-to-loss library (librlvla.so).
 *
 * The data-parallel hot path that RL-VLA^3's asynchronous pipeline keeps saturated
 * (arXiv 2602.05765; "P:n" = line n of the paper text, "S:n" = line n of SPEC.md):
 *
 *   S1 rlvla_scatter_steps     out-of-order step records -> trajectory buffer
 *   S2 rlvla_advantages        GAE (reverse segmented scan, done masks, global whitening)
 *                              or GRPO group normalisation (groups may span ranks)
 *   S3 rlvla_logprob_fwd_bwd   action-token log-softmax + gather, forward and backward,
 *   S4                         optionally fused with the PPO / decoupled clipped surrogate
 *      rlvla_ppo_loss          the same surrogate over log-prob arrays
 *      rlvla_value_loss        clipped value-head loss (NEXT-2)
 *   NEXT-3 rlvla_batch_offer / rlvla_batch_poll   Eq. (1) dynamic batching on the device
 *   NEXT-4 rlvla_flow_logprob  flow/diffusion chunk log-likelihood (Gaussian denoising chain)
 *
 * Conventions (all entry points):
 *   - Pointers are DEVICE pointers unless marked (host). Structs passed by pointer are
 *     HOST structs whose members are device pointers.
 *   - Every call enqueues its work on `stream` (a cudaStream_t; NULL = legacy default
 *     stream) and returns without synchronising. Cross-rank reductions (when `comm` !=
 *     NULL) run inside the computing kernel over NVLink peer memory, or as NCCL collectives
 *     on the same stream (rlvla_comm_p2p_enabled), so a whole iteration is CUDA-graph
 *     capturable.
 *   - Ownership: the caller owns every buffer, including `workspace`. The library
 *     allocates nothing in these calls and keeps no pointer after return. Its only state
 *     is the communicator handle and a per-device property cache.
 *   - Errors: host-detectable problems (NULL required pointer, negative sizes, ld < V,
 *     misalignment, dtype mismatch, shape mismatch, key-space overflow) return a status
 *     and launch nothing. Data-dependent problems (out-of-range ids, future versions,
 *     duplicates, bad targets, non-finite logits, negative lag) are COUNTED on the device
 *     and never abort. With the environment variable RLVLA_SYNC_CHECK=1 a call
 *     synchronises its stream and returns RLVLA_ERR_DATA if one of its error counters is
 *     non-zero. CUDA failures -> RLVLA_ERR_CUDA, NCCL failures -> RLVLA_ERR_NCCL.
 *   - Workspace: `workspace` must be at least rlvla_workspace_bytes(...) bytes, 256-byte
 *     aligned, and ZERO-FILLED before its first use; every call leaves it zero-filled in
 *     its control words again. One workspace must not be used by two streams at once.
 */
#ifndef RLVLA_H_
#define RLVLA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RLVLA_ABI_VERSION 2

#if defined(__GNUC__)
#define RLVLA_API __attribute__((visibility("default")))
#else
#define RLVLA_API
#endif

typedef int32_t rlvla_status;
enum {
  RLVLA_OK = 0,
  RLVLA_ERR_INVALID_ARG = 1,
  RLVLA_ERR_UNSUPPORTED = 2,
  RLVLA_ERR_CUDA = 3,
  RLVLA_ERR_NCCL = 4,
  RLVLA_ERR_DATA = 5 /* RLVLA_SYNC_CHECK=1 only */
};

typedef enum { RLVLA_F32 = 0, RLVLA_BF16 = 1 } rlvla_dtype;

/* Statistics vector: double[RLVLA_NSTATS], device memory, slots below.
 * rlvla_advantages writes slots 0..5 and 23 (and allreduces them over `comm`);
 * rlvla_logprob_fwd_bwd / rlvla_ppo_loss write slots 6..18 (allreducing 6..17);
 * rlvla_value_loss writes slots 19..22 (allreducing 19..21).
 * Each call OVERWRITES its slots unless `accumulate` is set (Streamer micro-batches). */
enum {
  RLVLA_STAT_N_VALID_STEPS = 0, /* #filled buffer slots (slot_key != 0)               */
  RLVLA_STAT_SUM_ADV = 1,       /* GAE: sum of raw advantages over filled slots (0 GRPO)*/
  RLVLA_STAT_SUM_ADV2 = 2,      /* GAE: sum of squared raw advantages           (0 GRPO)*/
  RLVLA_STAT_N_TOK = 3,         /* #tokens with target>=0 on filled steps, 0<=lag<=eta  */
  RLVLA_STAT_N_STALE_STEPS = 4, /* #filled steps with lag > eta                        */
  RLVLA_STAT_N_BAD_STEPS = 5,   /* #filled steps with lag < 0                          */
  RLVLA_STAT_LOSS = 6,          /* total loss share: sum_r m_r L_r / N - ent_coef sum m H / N */
  RLVLA_STAT_N_CLIPPED = 7,     /* #loss tokens (steps, chunk ratio) whose surrogate was clipped */
  RLVLA_STAT_KL_K3_SUM = 8,     /* sum_r m_r (rho - 1 - ln rho)  (policy vs behaviour/prox) */
  RLVLA_STAT_ENTROPY_SUM = 9,   /* sum_r m_r H_r (logits paths only; 0 in ppo_loss)     */
  RLVLA_STAT_RATIO_SUM = 10,    /* sum_r m_r rho                                        */
  RLVLA_STAT_N_LOSS_TOK = 11,   /* sum_r m_r                                            */
  RLVLA_STAT_N_STALE_TOK = 12,  /* usable tokens masked by lag > eta                    */
  RLVLA_STAT_N_BAD_TOK = 13,    /* tokens with target outside [-1,V), non-finite logp,  */
                                /* or lag < 0 (on filled steps)                         */
  RLVLA_STAT_LOGP_SUM = 14,     /* sum_r m_r logp_r                                     */
  RLVLA_STAT_KL_REF_SUM = 15,   /* sum_r m_r k3(ref), k3 = e^{lr} - lr - 1, lr = logp_ref - logp */
  RLVLA_STAT_N_DUAL_CLIPPED = 16, /* #loss tokens on the dual-clip branch (A < 0, c A > J) */
  RLVLA_STAT_PG_LOSS = 17,      /* clipped-surrogate part alone: sum_r m_r L_pg,r / N   */
  RLVLA_STAT_DENOM = 18,        /* the N used for the 1/N normalisation                 */
  RLVLA_STAT_VALUE_LOSS = 19,   /* rlvla_value_loss: sum_s m_s L_v,s / N_v              */
  RLVLA_STAT_N_VALUE_CLIPPED = 20, /* #steps on the clipped value branch                */
  RLVLA_STAT_N_VALUE_STEPS = 21,   /* sum_s m_s                                         */
  RLVLA_STAT_VALUE_DENOM = 22,     /* the N_v used                                      */
  RLVLA_STAT_N_LOSS_STEPS = 23,    /* #filled steps with 0<=lag<=eta and >= 1 target>=0: */
                                   /* the chunk-ratio normaliser N_steps (R21), global  */
  RLVLA_NSTATS = 24
};

/* Scatter counters: int64[4], ADDED to by rlvla_scatter_steps (caller zeroes). */
enum { RLVLA_CNT_OOB = 0, RLVLA_CNT_BAD_VERSION = 1, RLVLA_CNT_DUP = 2, RLVLA_CNT_WRITTEN = 3 };

typedef struct rlvla_comm_s* rlvla_comm; /* NULL => single rank, no collectives */

/* ---------------------------------------------------------------------------------
 * Trajectory buffer (§3.3 "trajectory buffer"; fields per SPEC Trajectory S:133-138).
 * One rank's shard: n_env envs x t_steps decision steps x a_tok action tokens.
 * Row-major: per-step arrays index [e * t_steps + t]; per-token arrays
 * [(e * t_steps + t) * a_tok + a]. slot_key == 0 marks a never-filled slot; otherwise
 * slot_key = (version << 40) | seq of the record that filled it (reading R6).
 * t_steps = N / c decision steps: one record = one inference = one action chunk
 * (reading R1; c = chunk size, Table 2), a_tok = c * 7 (7-DoF tokens).
 * ------------------------------------------------------------------------------- */
typedef struct {
  int32_t n_env, t_steps, a_tok;
  uint64_t* slot_key; /* [n_env*t_steps]; 8-byte aligned                         */
  float* reward;      /* [n_env*t_steps] chunk reward (sum of its env-step rewards) */
  uint8_t* done;      /* [n_env*t_steps] 1 = episode terminated at this step (R7)   */
  float* value;       /* [n_env*t_steps] value-head output V(s_t) of the rollout    */
  int32_t* version;   /* [n_env*t_steps] policy version that produced the step*/
  int32_t* tokens;    /* [n_env*t_steps*a_tok] sampled action tokens (-1 = ignore)  */
  float* logp_behav;  /* [n_env*t_steps*a_tok] behaviour log-probs from the rollout */
} rlvla_traj_buffer;

/* A batch of step records in ARRIVAL order (§3.2: ready requests from subsets of
 * environments enter early => records arrive out of order). Record i: env_id/step are
 * LOCAL to this rank's buffer. */
typedef struct {
  int32_t n_rec;
  const int32_t* env_id;     /* [n_rec]        */
  const int32_t* step;       /* [n_rec]        */
  const int32_t* version;    /* [n_rec]        */
  const float* reward;       /* [n_rec]        */
  const uint8_t* done;       /* [n_rec]        */
  const float* value;        /* [n_rec]        */
  const int32_t* tokens;     /* [n_rec*a_tok]  */
  const float* logp_behav;   /* [n_rec*a_tok]  */
} rlvla_step_batch;

/* S1 — scatter M records into the buffer.
 * Semantics = sequential replay in submission order (reading R6), reproduced
 * bit-exactly for any thread order: record i gets key_i = (version_i << 40) |
 * (seq_base + i);
 *   env_id/step out of range        -> counters[OOB] += 1
 *   version < 0 or > cur_version     -> counters[BAD_VERSION] += 1
 *   slot already filled              -> counters[DUP] += 1, and the slot takes the whole
 *                                       record iff key_i > its key
 *   else                             -> slot written, counters[WRITTEN] += 1
 * Payloads are copied bit for bit. `seq_base` >= 1 is caller-monotone across calls
 * (seq_base + n_rec < 2^40); 0 <= cur_version < 2^23. counters: device int64[4], ADDED to.
 * Returns INVALID_ARG on a key-space overflow or NULL pointers (n_rec == 0 is a no-op). */
RLVLA_API rlvla_status rlvla_scatter_steps(const rlvla_traj_buffer* buf, const rlvla_step_batch* rec,
                                 int32_t cur_version, uint64_t seq_base, int64_t* counters,
                                 void* stream);

enum { RLVLA_ADV_GAE = 0, RLVLA_ADV_GRPO = 1 };

typedef struct {
  int32_t mode;              /* RLVLA_ADV_GAE | RLVLA_ADV_GRPO                          */
  /* GAE (Schulman et al. 2016; paper-silent): */
  float gamma, lam;          /* discount and GAE lambda                                 */
  int32_t whiten;            /* 1 => adv = (A - mu) / (sigma + whiten_eps), mu/sigma over */
  float whiten_eps;          /*      all filled steps of ALL ranks (unbiased, R9)          */
  /* GRPO (Shao et al. 2024): R_e = sum_t r_t over filled steps; A_e = (R_e - mu_g) /   */
  /* (sigma_g + grpo_eps) over the env's group g, members in ascending global env id.   */
  const int32_t* group_id;   /* device int32[n_env_global] group of each GLOBAL env, or  */
                             /* NULL => contiguous groups of group_size                 */
  int32_t group_size;
  int32_t std_unbiased;      /* 1 => sigma with n-1 (R10), 0 => population (n)          */
  float grpo_eps;
  int32_t env_offset;        /* global id of this rank's env 0 (= rank * n_env)          */
  int32_t n_env_global;      /* n_env * nranks                                           */
  /* token bookkeeping for the loss normaliser (slot RLVLA_STAT_N_TOK): */
  int32_t cur_version, max_staleness;
  /* GAE time-limit truncation (NEXT-2, reading R23): a step with done == 2 ends the episode */
  /* by truncation; the recursion is cut but delta bootstraps from boot_value[e*T + t]      */
  /* (V of the true next state). NULL => done == 2 bootstraps 0 like a termination.        */
  const float* boot_value;
} rlvla_adv_params;

/* S2 — advantages for every slot of `buf`.
 * adv, ret: device float[n_env*t_steps]. GAE: adv = A_t (whitened if p->whiten),
 * ret = A_t + V_t (raw); GRPO: adv = A_e on filled steps, ret = R_e (ret may be NULL).
 * Never-filled slots get adv = ret = 0 and cut the GAE recursion (R8).
 * GAE per env, t = T-1..0: nt_t = v_t [done_t == 0] v_{t+1} (v_T := 1), tr_t = [done_t == 2];
 * delta_t = v_t (r_t + gamma (nt_t V_{t+1} + tr_t B_t) - V_t) with V_T = last_value[e]
 * (NULL => 0), B = boot_value; A_t = delta_t + gamma lam nt_t A_{t+1}. Computed as a warp-parallel suffix scan of the
 * affine maps A -> delta_t + c_t A (fp32, fp64 statistics).
 * stats: device double[RLVLA_NSTATS]; slots 0..5 and 23 written and reduced over `comm` (C1). With
 * GRPO and comm != NULL the per-env returns are allgathered (C2) first. */
RLVLA_API rlvla_status rlvla_advantages(const rlvla_traj_buffer* buf, const float* last_value,
                              const rlvla_adv_params* p, float* adv, float* ret,
                              double* stats, void* workspace, size_t ws_bytes,
                              rlvla_comm comm, void* stream);

/* Logit rows: rows x vocab, row r at ptr + r*ld elements. ptr 16-byte aligned for the
 * vectorised paths (any alignment works on the generic path). */
typedef struct {
  const void* ptr;
  int32_t dtype;   /* rlvla_dtype */
  int64_t rows;
  int32_t vocab;   /* V: the softmax normalises over these V columns (reading R3) */
  int64_t ld;      /* >= vocab, in elements */
} rlvla_logits;

/* PPO / decoupled-PPO arguments (S4). Row r belongs to decision step s = r / a_tok;
 * for a micro-batch, offset every per-row pointer by r0 and every per-step pointer by
 * r0 / a_tok (r0 a multiple of a_tok).
 *   lag = cur_version - version[s];  m_r = [slot_key[s] != 0] [target ok, finite logp]
 *                                          [0 <= lag <= max_staleness]
 *   standard : rho = exp(logp - logp_behav), w = 1
 *   decoupled: w = min(exp(logp_prox - logp_behav), is_cap) (detached, is_cap <= 0 =>
 *              no cap), rho = exp(logp - logp_prox)            (AReaL, cited P:18)
 *   L_r = -w min(rho A_s, clip(rho, 1 - eps_low, 1 + eps_high) A_s);  Loss = sum m L / N
 *   dLoss/dlogp_r = -m_r w A_s rho [active] / N, ties at the clip bound active (R11). */
typedef struct {
  const float* logp_behav;    /* [rows]                                               */
  const float* logp_prox;     /* [rows] or NULL => standard PPO                        */
  const float* adv;           /* [rows / a_tok] per decision step                      */
  const int32_t* version;     /* [rows / a_tok]                                        */
  const uint64_t* slot_key;   /* [rows / a_tok] 0 => step never filled (masked)        */
  int32_t a_tok, cur_version, max_staleness;
  float eps_low, eps_high, is_cap;
  double tok_denominator;     /* > 0: N. <= 0: N = adv_stats[RLVLA_STAT_N_TOK] (global, */
  const double* adv_stats;    /*  device, from rlvla_advantages)                       */
  float* out_grad_logp;       /* [rows] optional: dLoss/dlogp_r                        */
  float* out_loss_tok;        /* [rows] optional: m_r L_r (unnormalised)               */
  int32_t accumulate;         /* 0: overwrite stats slots 6..18 (then C3 over `comm`).  */
                              /* 1: ADD this call's slots 6..17 to `stats` (Streamer    */
                              /*    micro-batches, §3.3; fixed call order keeps the */
                              /*    sum deterministic). Pass `comm` only with the last   */
                              /*    micro-batch: its C3 then reduces the running totals. */
  /* Loss variants (all paper-silent, readings R19-R21). 0 / NULL = off.   */
  float dual_clip;            /* c > 1: for A < 0 the objective is max(J, c A) (Ye et al. */
                              /* 2020); tokens with c A > J get no gradient             */
  const float* logp_ref;      /* [rows] reference-policy log-probs (KL penalty), or NULL */
  float kl_coef;              /* L_r += kl_coef k3, k3 = e^{lr} - lr - 1, lr = logp_ref - logp */
  float ent_coef;             /* Loss -= ent_coef sum m H / N with its gradient through  */
                              /* the logits (logits path only; 0 in rlvla_ppo_loss)     */
  int32_t ratio_level;        /* rlvla_ppo_loss only: 0 token ratio; 1 one ratio per     */
                              /* decision step = the action chunk's likelihood ratio    */
                              /* exp(sum_a m (logp - logp_behav)) (decoupled: w_s =     */
                              /* min(exp(sum m (logp_prox - logp_behav)), is_cap),      */
                              /* rho_s = exp(sum m (logp - logp_prox)); dual_clip as    */
                              /* above; kl_coef / ent_coef => RLVLA_ERR_UNSUPPORTED),    */
                              /* Loss / N_steps with N_steps = tok_denominator (> 0),   */
                              /* else adv_stats[RLVLA_STAT_N_LOSS_STEPS] (global), else  */
                              /* the call's own masked-step count over all ranks of     */
                              /* `comm` (not allowed with accumulate = 1)               */
} rlvla_ppo_args;

/* S3 (+S4) — action-token log-probs over logit rows (P:39 action tokens; P:88 actor
 * micro-batch forward/backward):
 *   lse_r = m + ln sum_j exp(x_rj - m);  logp_r = x_{r,a_r} - lse_r;
 *   H_r = lse_r - sum_j p_rj x_rj;       dx_rj = g_r (1[j = a_r] - exp(x_rj - lse_r)).
 * Modes:
 *   forward only    : fused == NULL, grad_logp == NULL, dlogits == NULL
 *   external bwd    : fused == NULL, grad_logp != NULL, lse (input!) != NULL, dlogits;
 *                     one read of x, one write of dlogits, logp not written
 *   fused PPO       : fused != NULL: one pass computing logp, the PPO epilogue g_r and
 *                     (if dlogits != NULL) dlogits; stats slots 6..18; over `comm` C3.
 * target: int32[rows]; -1 => ignore (logp = 0, zero gradient row); other targets
 * outside [0, V) are counted in N_BAD_TOK and treated as ignored (R4). Non-finite
 * results (NaN/+inf logits, all -inf row, -inf target logit) give a non-finite logp,
 * are counted and masked (R5). logp: float[rows] (written except in external bwd);
 * lse: float[rows] or NULL (output in forward/fused modes). dlogits: same dtype/ld as
 * x, may alias x->ptr (each row is read completely before it is written); masked rows
 * are written as zeros. stats: NULL or device double[RLVLA_NSTATS]. */
RLVLA_API rlvla_status rlvla_logprob_fwd_bwd(const rlvla_logits* x, const int32_t* target, float* logp,
                                   float* lse, const float* grad_logp,
                                   const rlvla_ppo_args* fused, void* dlogits, double* stats,
                                   void* workspace, size_t ws_bytes, rlvla_comm comm,
                                   void* stream);

/* S4 — the same surrogate over precomputed log-probs logp[rows] (e.g. produced by
 * another forward). target: int32[rows] or NULL (all usable); rows whose target is
 * outside [0, ...) or whose logp is non-finite are masked (no vocab bound is known
 * here, so only target < 0 / non-finite are checked). grad_logp: float[rows] output
 * (required); loss_tok: float[rows] or NULL. stats slots 6..18 (entropy slot = 0). */
RLVLA_API rlvla_status rlvla_ppo_loss(const float* logp, int64_t rows, const int32_t* target,
                            const rlvla_ppo_args* a, float* grad_logp, float* loss_tok,
                            double* stats, void* workspace, size_t ws_bytes, rlvla_comm comm,
                            void* stream);

/* S4 value head (reading R22): clipped value loss per decision step,
 *   L_s = 0.5 max((v - R)^2, (v_old + clip(v - v_old, -clip_eps, clip_eps) - R)^2)
 * (clip_eps <= 0 => 0.5 (v - R)^2), m_s = [slot_key != 0][0 <= lag <= max_staleness],
 * Loss = sum m L / N_v with N_v = denominator (> 0) or the call's sum m_s over all ranks of
 * `comm` (the gradient scale waits for the reduced count). grad_v[s] = dLoss/dv_s (required), loss_step
 * optional. v_new, v_old (= buffer value), ret: float[n_steps]. stats slots 19..22 (C over
 * comm for 19..21). */
RLVLA_API rlvla_status rlvla_value_loss(const float* v_new, const float* v_old, const float* ret,
                                        const uint64_t* slot_key, const int32_t* version,
                                        int64_t n_steps, int32_t cur_version,
                                        int32_t max_staleness, float clip_eps,
                                        double denominator, float* grad_v, float* loss_step,
                                        double* stats, void* workspace, size_t ws_bytes,
                                        rlvla_comm comm, void* stream);

/* ---------------------------------------------------------------------------------
 * NEXT-3 — the Dynamic Batching Scheduler of Eq. (1) on the device (§3.2:
 * "Trigger Inference if: (Batch Size >= B_max) or (Wait Time >= T_max)"; ready requests
 * from a subset of environments enter the inference queue early). Reading R24
 * (SPEC.md S:161-180): one rollout worker's FIFO of pending requests in
 * arrival order; the wait clock is anchored when a request finds the queue empty and
 * re-anchored at the poll time when a batch leaves requests behind; an empty queue never
 * fires; more than B_max pending => the oldest B_max leave. The step just upstream of S1:
 * it gathers the ready envs' observations into one contiguous inference batch.
 * Times are int64 ticks (any unit; the comparison with T_max is exact).
 * ------------------------------------------------------------------------------- */
typedef struct {
  int32_t n_env;        /* envs served by this queue (= ring capacity; an env waits for its */
                        /* action, so it has at most one pending request)                  */
  int64_t obs_bytes;    /* observation payload per env in bytes, multiple of 16 (0 = none) */
  uint8_t* obs;         /* observation rows (16-byte aligned), see obs_fifo               */
  int32_t* ring_env;    /* [n_env] FIFO ring: env of each pending request                  */
  int64_t* ring_time;   /* [n_env] FIFO ring: its enqueue time                             */
  uint8_t* pending;     /* [n_env] 1 while the env has a request in the ring               */
  int64_t* state;       /* int64[8]: head, tail (request counts since creation), anchor,   */
                        /* number of batches emitted, first obs row of the last batch      */
                        /* (obs_fifo), 3 reserved. Zero-filled at creation; owned by the   */
                        /* device (the library never reads it on the host)                 */
  int32_t obs_fifo;     /* 0: obs = [n_env] slots indexed by env (the env side may write   */
                        /*    its slot in place; a poll GATHERS the batch into out_obs)    */
                        /* 1: obs = [n_env + max_batch] rows indexed by FIFO position: the */
                        /*    offer copies obs_src into its request's row, so a batch is   */
                        /*    already contiguous: rows [state[4], state[4] + b) of obs     */
                        /*    (a wrap copies at most b - 1 rows past n_env). Half the      */
                        /*    bytes of mode 0 per request; offers must carry obs_src. The  */
                        /*    rows stay valid until later accepted offers reuse their ring */
                        /*    positions: consume the batch in stream order before offering */
                        /*    n_env - (requests still pending) more.                       */
  int32_t max_batch;    /* obs_fifo: the largest b_max any poll will use (<= n_env)        */
} rlvla_batch_queue;

/* Batcher counters: int64[4], ADDED to by rlvla_batch_offer (caller zeroes). */
enum { RLVLA_BCNT_OOB = 0, RLVLA_BCNT_FUTURE = 1, RLVLA_BCNT_DUP = 2, RLVLA_BCNT_ACCEPTED = 3 };

/* offer: n requests in ARRIVAL order at time `now` (>= 0), 0 <= n <= 1024 per
 * call (split larger arrivals into consecutive calls with the same `now`: same result).
 * Request i = (env_id[i], enqueue_time[i]); it is rejected and counted when env_id is out of
 * [0, n_env) (OOB), when enqueue_time > now (FUTURE), or when the env already has a pending
 * request, including an earlier accepted request of the same call (DUP); otherwise it is
 * appended to the FIFO (ACCEPTED) and, if the queue was empty, the anchor := now.
 * obs_src: NULL (the env side wrote its observation into obs[env] already) or device
 * [n * obs_bytes], row i copied into obs[env_id[i]] for every accepted request.
 * counters: device int64[4], added to. workspace: as for the other calls (>= the
 * rlvla_workspace_bytes(0, 0, 0) header), used for its control words. */
RLVLA_API rlvla_status rlvla_batch_offer(const rlvla_batch_queue* q, const int32_t* env_id,
                                         const int64_t* enqueue_time, int32_t n, int64_t now,
                                         const void* obs_src, int64_t* counters,
                                         void* workspace, size_t ws_bytes, void* stream);

/* poll (Eq. (1)) — with obs_fifo = 1 out_obs may be NULL (the batch is rows
 * [state[4], state[4] + b) of q->obs); otherwise: with p = pending count, the queue fires iff p >= b_max or
 * (p >= 1 and now - anchor >= t_max); then b = min(p, b_max) oldest requests leave in FIFO
 * order: out_env[i], out_time[i] (device [b_max]) and, if out_obs != NULL, their
 * observations gathered into out_obs[i * obs_bytes ...] (device [b_max * obs_bytes],
 * 16-byte aligned); remaining requests re-anchor the clock at now. *out_n (device int32)
 * = b, 0 when the trigger does not fire (entries >= b untouched). b_max >= 1, t_max >= 0,
 * now >= 0. The gather is one read + one write of b * obs_bytes (HBM-bound). */
RLVLA_API rlvla_status rlvla_batch_poll(const rlvla_batch_queue* q, int64_t now, int32_t b_max,
                                        int64_t t_max, int32_t* out_env, int64_t* out_time,
                                        void* out_obs, int32_t* out_n, void* workspace,
                                        size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * NEXT-4 — flow / diffusion policies (pi_0, pi_0.5 flow matching; GR00T N1.5 diffusion:
 * P:39, "multi-step denoising"; Table 2 "Model Num Step" = 4). Reading
 * R25: a decision step's action chunk is the end of a K-step stochastic denoising chain
 * with Gaussian transitions x_{k+1} ~ N(mu_theta(x_k, k), diag(sigma_{k,d}^2)); its
 * log-likelihood is the sum of the K transition log-densities
 *   logp_r = sum_{k,d} [ -(x - mu)^2 / (2 sigma^2) - ln sigma - ln(2 pi)/2 ],
 * and with g_r = dLoss/dlogp_r:  dmu = g (x - mu) / sigma^2,  dln sigma = g ((x-mu)^2/sigma^2 - 1).
 * H_r = sum_{k,d} (ln sigma + ln(2 pi e)/2) (statistics; entropy bonus through ln sigma).
 * ------------------------------------------------------------------------------- */
typedef struct {
  const void* mu;        /* [rows * n_steps * dim] denoiser means, dtype mu_dtype (row-major) */
  int32_t mu_dtype;      /* RLVLA_F32 | RLVLA_BF16                                         */
  const float* x;        /* [rows * n_steps * dim] the sampled next latents x_{k+1}        */
  const float* sigma_k;  /* [n_steps] per-step std (a schedule, no gradient), used when    */
                         /* log_std == NULL; entries must be > 0                           */
  const float* log_std;  /* [rows * n_steps * dim] learned ln sigma, or NULL               */
  int64_t rows;          /* decision steps                                                  */
  int32_t n_steps, dim;  /* K denoising steps, D = chunk size x action dim                 */
} rlvla_gauss_chain;

/* Chain log-likelihood per decision step, optionally fused with the PPO surrogate and its
 * backward (the continuous-action analogue of rlvla_logprob_fwd_bwd):
 *   forward only  : grad_logp == NULL, fused == NULL: logp[rows] (+ stats 6..18 as in the
 *                   forward-only logits path: N_LOSS_TOK, ENTROPY_SUM, LOGP_SUM, N_BAD_TOK)
 *   external bwd  : grad_logp != NULL (e.g. from rlvla_ppo_loss): dmu / dlog_std from it
 *   fused PPO     : fused != NULL, a_tok == 1 (one ratio per decision step = the chunk's
 *                   likelihood ratio), ratio_level == 0; every PPO knob of rlvla_ppo_args
 *                   applies (decoupled, staleness, dual clip, logp_ref KL, entropy bonus
 *                   through ln sigma when log_std != NULL); stats slots 6..18, C3 over comm.
 * dmu: [rows*n_steps*dim] in mu_dtype, or NULL; dlog_std: float[...] (requires log_std) or
 * NULL. Rows with a non-finite logp are counted (N_BAD_TOK) and masked. n_steps*dim <= 4096. */
RLVLA_API rlvla_status rlvla_flow_logprob(const rlvla_gauss_chain* c, float* logp,
                                          const float* grad_logp, const rlvla_ppo_args* fused,
                                          void* dmu, float* dlog_std, double* stats,
                                          void* workspace, size_t ws_bytes, rlvla_comm comm,
                                          void* stream);

/* Workspace bytes for calls on buffers/logits up to these sizes (host-only, no GPU). */
RLVLA_API size_t rlvla_workspace_bytes(int64_t rows, int32_t n_env_global, int32_t t_steps);

/* Communicator over NCCL (NVLink/NVSwitch). Rank 0 calls rlvla_comm_unique_id and the
 * 128 bytes are broadcast by the caller (e.g. torch.distributed). Host pointers. Every
 * rank takes part in the same collectives at init whatever its local result (a rank whose
 * mailbox could not be mapped makes all ranks fall back to NCCL collectives together). */
RLVLA_API rlvla_status rlvla_comm_unique_id(void* out_id_128_bytes);
RLVLA_API rlvla_status rlvla_comm_init(const void* nccl_unique_id, int32_t nranks, int32_t rank,
                             rlvla_comm* out);
RLVLA_API rlvla_status rlvla_comm_destroy(rlvla_comm c);

/* P2P-only communicator (no NCCL): the cross-rank exchanges C1/C2/C3 run only inside the
 * kernels over CUDA-IPC-mapped mailboxes, so several ranks may share one GPU (NCCL refuses
 * duplicate devices) and up to 8 ranks are supported. Two phases, the handle exchange done
 * by the caller over its own process group (e.g. a torch gloo all_gather):
 *   1. rlvla_comm_init_p2p: allocates this rank's mailbox on the current device and writes
 *      its IPC handle (RLVLA_P2P_HANDLE_BYTES host bytes) to out_handle;
 *   2. rlvla_comm_connect_p2p: all_handles = host [nranks][RLVLA_P2P_HANDLE_BYTES] in rank
 *      order; maps every peer's mailbox. A failure returns RLVLA_ERR_CUDA; the caller must
 *      agree on the outcome across ranks and destroy the communicator on any failure.
 * Calls that would need an NCCL collective with such a communicator (GRPO with
 * n_env_global > 32768) return RLVLA_ERR_UNSUPPORTED. */
#define RLVLA_P2P_HANDLE_BYTES 64
RLVLA_API rlvla_status rlvla_comm_init_p2p(int32_t nranks, int32_t rank, void* out_handle,
                                           rlvla_comm* out);
RLVLA_API rlvla_status rlvla_comm_connect_p2p(rlvla_comm c, const void* all_handles);
/* 1 when the communicator reduces statistics INSIDE the computing kernel over NVLink peer
 * memory (every rank's mailbox mapped through CUDA IPC at rlvla_comm_init; the kernel's last
 * CTA pushes its slots to all ranks and sums them in rank order): C1 and the GRPO returns
 * allgather C2 in rlvla_advantages (n_env_global <= 32768), C3 in rlvla_logprob_fwd_bwd,
 * rlvla_ppo_loss and rlvla_flow_logprob. 0 when those calls use NCCL
 * collectives after the kernel. RLVLA_P2P=0 at init forces NCCL. Calls with one communicator
 * must be stream-ordered and made in the same order on every rank (as for NCCL). The
 * value loss reduces slots 19..21 and the chunk-ratio path slots 6..17 the same way. */
RLVLA_API int32_t rlvla_comm_p2p_enabled(rlvla_comm c);

/* Launch policy (host, process-wide, thread-safe): the persistent kernels (TMA log-prob
 * kernel, TMA flow kernel: one CTA per SM holding the register file) use sm_count - n SMs
 * (at least 1), leaving n SMs free so latency-bound work on another stream (e.g. the next
 * batch's rlvla_scatter_steps / rlvla_advantages while the actor's S3+S4 runs: §3.3
 * "masking data preparation time") is not blocked until they finish. Default 0. Returns
 * the previous value. */
RLVLA_API int32_t rlvla_set_reserved_sms(int32_t n);

RLVLA_API const char* rlvla_status_string(rlvla_status s);
RLVLA_API int32_t rlvla_abi_version(void);
/* Version of the NCCL library actually loaded (e.g. 22809), 0 if unavailable. */
RLVLA_API int32_t rlvla_nccl_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RLVLA_H_ */
