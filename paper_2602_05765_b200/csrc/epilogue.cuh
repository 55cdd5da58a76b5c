// epilogue.cuh — per-row S4 epilogue shared by the log-prob kernels (fused mode) and the
// standalone rlvla_ppo_loss kernel.
//
// Paper anchors: behaviour version and staleness (§3.1: rollout keeps generating
// with the pre-update weights => lag <= 1); decoupled objective cited as AReaL.
// The surrogate itself is textbook PPO-clip (Schulman et al. 2017), readings R11-R14:
//   m   = valid * usable * [0 <= lag <= eta]
//   rho = exp(logp - logp_behav)            (standard), w = 1
//   w   = min(exp(logp_prox - logp_behav), cap), rho = exp(logp - logp_prox) (decoupled)
//   L   = -w min(rho A, clip(rho, 1-eps_lo, 1+eps_hi) A)
//   g   = dLoss/dlogp = -w A rho [active] / N,  active <=> !((A>0 & rho>hi) | (A<0 & rho<lo))
#pragma once
#include "internal.cuh"

namespace rlvla {

// per-row contributions to the loss statistics, in slot order 6..17 (see rlvla.h)
constexpr int kLossSlots = 12;
struct RowStats {
  float loss;     // m * (L_pg + kl_coef k3_ref)   (unnormalised)
  float clipped;  // m * [ratio clip active]
  float k3;       // m * (rho - 1 - ln rho)
  float ent;      // m * H
  float rho;      // m * rho
  float m;        // m
  float stale;    // usable on a filled step, lag > eta
  float bad;      // bad target / non-finite / lag < 0 on a filled step
  float logp;     // m * logp
  float kl_ref;   // m * k3_ref
  float dual;     // m * [dual-clip branch]
  float pg;       // m * L_pg
};

struct PpoRowIn {
  int tgt_status;   // 0 usable, 1 ignore (-1), 2 bad target, 3 non-finite logp
  float logp;
  float H;          // entropy (0 when unavailable)
  float lpb, lpp;   // behaviour / proximal log-prob (lpp unused when !has_prox)
  float lref;       // reference log-prob (unused when !has_ref)
  float adv;
  int ver;
  int valid;        // step filled (slot_key != 0)
};

struct PpoConst {
  int has_prox, has_ref;
  int cur_version, eta;
  float lo, hi, is_cap;
  float dual_clip, kl_coef, ent_coef;
  float invN;
};

// Intermediate values of one row: ppo_grad computes what the gradient needs (the only
// part on the fused kernel's critical path), ppo_stats the rest once g is published.
struct PpoMid {
  bool m, base, clipped, dual;
  int lag;
  float lr, rho, w, J, lq;
};

// g = dLoss/dlogp for the row (including 1/N)
__device__ __forceinline__ float ppo_grad(const PpoConst& c, const PpoRowIn& in, PpoMid& t) {
  const bool usable = in.tgt_status == 0;
  t.lag = c.cur_version - in.ver;
  t.base = in.valid && usable;
  t.m = t.base && t.lag >= 0 && t.lag <= c.eta;
  t.clipped = t.dual = false;
  t.lr = t.rho = t.J = t.lq = 0.f;
  t.w = 1.f;
  if (!t.m) return 0.f;
  if (c.has_prox) {
    t.lr = in.logp - in.lpp;
  } else {
    t.lr = in.logp - in.lpb;
  }
  // (measured and rejected: rho = p_a e^{-lp_base} with e^{-lp_base} precomputed before the
  // row's sums — slower, and rho = 1 is no longer exact when logp == logp_behav)
  t.rho = __expf(t.lr);
  if (c.has_prox) {
    t.w = __expf(in.lpp - in.lpb);
    if (c.is_cap > 0.f) t.w = fminf(t.w, c.is_cap);
  }
  const float A = in.adv;
  const float rc = fminf(fmaxf(t.rho, c.lo), c.hi);
  t.J = fminf(t.rho * A, rc * A);
  t.clipped = (A > 0.f && t.rho > c.hi) || (A < 0.f && t.rho < c.lo);
  // dual clip (c > 1): for A < 0 the objective is max(J, c A); strict > (tie: J branch)
  t.dual = c.dual_clip > 1.f && A < 0.f && c.dual_clip * A > t.J;
  if (t.dual) t.J = c.dual_clip * A;
  float gr = (t.clipped || t.dual) ? 0.f : -t.w * A * t.rho;
  if (c.has_ref) {
    // k3 = e^{q} - q - 1 with q = logp_ref - logp; dk3/dlogp = 1 - e^{q}
    t.lq = in.lref - in.logp;
    gr += c.kl_coef * (-expm1f(t.lq));
  }
  return gr * c.invN;
}

// k3-type divergence e^x - 1 - x, cancellation-free near x = 0 (Taylor to x^6)
__device__ __forceinline__ float k3_of(float x, float ex) {
  return fabsf(x) < 0.125f
             ? x * x * (0.5f + x * (1.f / 6.f + x * (1.f / 24.f + x * (1.f / 120.f + x * (1.f / 720.f)))))
             : (ex - 1.f - x);
}

// statistics and the per-token loss m (L_pg + kl k3_ref) from ppo_grad's intermediates
__device__ __forceinline__ void ppo_stats(const PpoConst& c, const PpoRowIn& in, const PpoMid& t,
                                          RowStats& rs, float* loss_tok) {
  rs.stale = (t.base && t.lag > c.eta) ? 1.f : 0.f;
  rs.bad = ((in.valid && (in.tgt_status == 2 || in.tgt_status == 3)) || (t.base && t.lag < 0)) ? 1.f : 0.f;
  rs.loss = rs.clipped = rs.k3 = rs.ent = rs.rho = rs.m = rs.logp = 0.f;
  rs.kl_ref = rs.dual = rs.pg = 0.f;
  float L = 0.f;
  if (t.m) {
    const float Lpg = -t.w * t.J;
    L = Lpg;
    if (c.has_ref) {
      const float k3r = k3_of(t.lq, __expf(t.lq));
      L += c.kl_coef * k3r;
      rs.kl_ref = k3r;
    }
    rs.loss = L;
    rs.pg = Lpg;
    rs.clipped = t.clipped ? 1.f : 0.f;
    rs.dual = t.dual ? 1.f : 0.f;
    rs.k3 = k3_of(t.lr, t.rho);  // rho - 1 - ln rho
    rs.ent = in.H;
    rs.rho = t.rho;
    rs.m = 1.f;
    rs.logp = in.logp;
  }
  *loss_tok = L;
}

// Returns g = dLoss/dlogp for the row; fills rs and *loss_tok (m * (L_pg + kl k3_ref)).
__device__ __forceinline__ float ppo_row(const PpoConst& c, const PpoRowIn& in, RowStats& rs,
                                         float* loss_tok) {
  PpoMid t;
  const float g = ppo_grad(c, in, t);
  ppo_stats(c, in, t, rs, loss_tok);
  return g;
}

// forward-only statistics: usable rows count as "loss tokens" for entropy/logp sums
__device__ __forceinline__ void fwd_row_stats(const PpoRowIn& in, RowStats& rs) {
  const bool usable = in.tgt_status == 0;
  rs.loss = rs.clipped = rs.k3 = rs.rho = rs.stale = rs.kl_ref = rs.dual = rs.pg = 0.f;
  rs.m = usable ? 1.f : 0.f;
  rs.ent = usable ? in.H : 0.f;
  rs.logp = usable ? in.logp : 0.f;
  rs.bad = (in.tgt_status == 2 || in.tgt_status == 3) ? 1.f : 0.f;
}

__device__ __forceinline__ void acc_stats(double* acc, const RowStats& rs) {
  acc[0] += double(rs.loss);
  acc[1] += double(rs.clipped);
  acc[2] += double(rs.k3);
  acc[3] += double(rs.ent);
  acc[4] += double(rs.rho);
  acc[5] += double(rs.m);
  acc[6] += double(rs.stale);
  acc[7] += double(rs.bad);
  acc[8] += double(rs.logp);
  acc[9] += double(rs.kl_ref);
  acc[10] += double(rs.dual);
  acc[11] += double(rs.pg);
}

__device__ __forceinline__ void acc_stats_f(float* acc, const RowStats& rs) {
  acc[0] += rs.loss;
  acc[1] += rs.clipped;
  acc[2] += rs.k3;
  acc[3] += rs.ent;
  acc[4] += rs.rho;
  acc[5] += rs.m;
  acc[6] += rs.stale;
  acc[7] += rs.bad;
  acc[8] += rs.logp;
  acc[9] += rs.kl_ref;
  acc[10] += rs.dual;
  acc[11] += rs.pg;
}

// N for the 1/N normalisation: explicit, else the global token count from rlvla_advantages
__device__ __forceinline__ double loss_denominator(double denom, const double* adv_stats) {
  if (denom > 0.0) return denom;
  if (adv_stats) return adv_stats[RLVLA_STAT_N_TOK];
  return 0.0;
}

// CTA partials (12 slots) -> workspace; last CTA writes stats[6..18]
//   LOSS = (sum m L - ent_coef sum m H) / N, PG_LOSS = sum m L_pg / N, the rest raw sums.
// With p2p (nranks > 1) the last CTA also reduces slots 6..17 over the ranks in-kernel.
__device__ __forceinline__ void finish_loss_stats(const double* cta_acc, double* stats,
                                                  double* partials, unsigned* ctrl, double N,
                                                  int accumulate, float ent_coef,
                                                  const P2PDesc* p2p = nullptr) {
  if (threadIdx.x < kLossSlots)
    partials[size_t(blockIdx.x) * RLVLA_NSTATS + threadIdx.x] = cta_acc[threadIdx.x];
  __shared__ double tot[kLossSlots];
  if (last_block_reduce(ctrl, partials, kLossSlots, tot)) {
    if (threadIdx.x < kLossSlots) {
      const double invN = N > 0.0 ? 1.0 / N : 0.0;
      double v = tot[threadIdx.x];
      if (threadIdx.x == 0) v = (v - double(ent_coef) * tot[3]) * invN;
      if (threadIdx.x == 11) v *= invN;
      if (accumulate) v += stats[RLVLA_STAT_LOSS + threadIdx.x];
      tot[threadIdx.x] = v;
    }
    __syncthreads();
    if (p2p && p2p->nranks > 1) p2p_allreduce(tot, kLossSlots, *p2p);
    if (threadIdx.x < kLossSlots) stats[RLVLA_STAT_LOSS + threadIdx.x] = tot[threadIdx.x];
    if (threadIdx.x == 0) stats[RLVLA_STAT_DENOM] = N;
  }
}

}  // namespace rlvla
