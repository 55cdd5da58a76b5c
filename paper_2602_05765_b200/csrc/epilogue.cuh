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

// Returns g = dLoss/dlogp for the row; fills rs and *loss_tok (m * (L_pg + kl k3_ref)).
__device__ __forceinline__ float ppo_row(const PpoConst& c, const PpoRowIn& in, RowStats& rs,
                                         float* loss_tok) {
  const bool usable = in.tgt_status == 0;
  const int lag = c.cur_version - in.ver;
  const bool base = in.valid && usable;
  const bool m = base && lag >= 0 && lag <= c.eta;
  rs.stale = (base && lag > c.eta) ? 1.f : 0.f;
  rs.bad = ((in.valid && (in.tgt_status == 2 || in.tgt_status == 3)) || (base && lag < 0)) ? 1.f : 0.f;
  float g = 0.f, L = 0.f;
  rs.loss = rs.clipped = rs.k3 = rs.ent = rs.rho = rs.m = rs.logp = 0.f;
  rs.kl_ref = rs.dual = rs.pg = 0.f;
  if (m) {
    float lr, w;
    if (c.has_prox) {
      w = __expf(in.lpp - in.lpb);
      if (c.is_cap > 0.f) w = fminf(w, c.is_cap);
      lr = in.logp - in.lpp;
    } else {
      w = 1.f;
      lr = in.logp - in.lpb;
    }
    const float rho = __expf(lr);
    const float A = in.adv;
    const float rc = fminf(fmaxf(rho, c.lo), c.hi);
    float J = fminf(rho * A, rc * A);
    const bool clipped = (A > 0.f && rho > c.hi) || (A < 0.f && rho < c.lo);
    // dual clip (c > 1): for A < 0 the objective is max(J, c A); strict > (tie: J branch)
    const bool dual = c.dual_clip > 1.f && A < 0.f && c.dual_clip * A > J;
    if (dual) J = c.dual_clip * A;
    const float Lpg = -w * J;
    float gr = (clipped || dual) ? 0.f : -w * A * rho;
    L = Lpg;
    if (c.has_ref) {
      // k3 = e^{lr} - lr - 1 with lr = logp_ref - logp; dk3/dlogp = 1 - e^{lr}
      const float lq = in.lref - in.logp;
      const float k3r = fabsf(lq) < 0.125f
                            ? lq * lq * (0.5f + lq * (1.f / 6.f + lq * (1.f / 24.f + lq * (1.f / 120.f + lq * (1.f / 720.f)))))
                            : (__expf(lq) - 1.f - lq);
      L += c.kl_coef * k3r;
      gr += c.kl_coef * (-expm1f(lq));
      rs.kl_ref = k3r;
    }
    g = gr * c.invN;
    rs.loss = L;
    rs.pg = Lpg;
    rs.clipped = clipped ? 1.f : 0.f;
    rs.dual = dual ? 1.f : 0.f;
    // k3 = rho - 1 - ln rho = expm1(lr) - lr, cancellation-free near rho = 1 (Taylor to lr^6)
    rs.k3 = fabsf(lr) < 0.125f
                ? lr * lr * (0.5f + lr * (1.f / 6.f + lr * (1.f / 24.f + lr * (1.f / 120.f + lr * (1.f / 720.f)))))
                : (rho - 1.f - lr);
    rs.ent = in.H;
    rs.rho = rho;
    rs.m = 1.f;
    rs.logp = in.logp;
  }
  *loss_tok = L;
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

// N for the 1/N normalisation: explicit, else the global token count from rlvla_advantages
__device__ __forceinline__ double loss_denominator(double denom, const double* adv_stats) {
  if (denom > 0.0) return denom;
  if (adv_stats) return adv_stats[RLVLA_STAT_N_TOK];
  return 0.0;
}

// CTA partials (12 slots) -> workspace; last CTA writes stats[6..18]
//   LOSS = (sum m L - ent_coef sum m H) / N, PG_LOSS = sum m L_pg / N, the rest raw sums.
__device__ __forceinline__ void finish_loss_stats(const double* cta_acc, double* stats,
                                                  double* partials, unsigned* ctrl, double N,
                                                  int accumulate, float ent_coef) {
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
      stats[RLVLA_STAT_LOSS + threadIdx.x] = v;
    }
    if (threadIdx.x == 0) stats[RLVLA_STAT_DENOM] = N;
  }
}

}  // namespace rlvla
