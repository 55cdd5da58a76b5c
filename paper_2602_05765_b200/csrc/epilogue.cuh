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

// per-row contributions to stats slots 6..14 (in slot order)
struct RowStats {
  float loss;     // m * L (unnormalised)
  float clipped;  // m * [!active]
  float k3;       // m * (rho - 1 - ln rho)
  float ent;      // m * H
  float rho;      // m * rho
  float m;        // m
  float stale;    // usable on a filled step, lag > eta
  float bad;      // bad target / non-finite / lag < 0 on a filled step
  float logp;     // m * logp
};

struct PpoRowIn {
  int tgt_status;   // 0 usable, 1 ignore (-1), 2 bad target, 3 non-finite logp
  float logp;
  float H;          // entropy (0 when unavailable)
  float lpb, lpp;   // behaviour / proximal log-prob (lpp unused when !has_prox)
  float adv;
  int ver;
  int valid;        // step filled (slot_key != 0)
};

struct PpoConst {
  int has_prox;
  int cur_version, eta;
  float lo, hi, is_cap;
  float invN;
};

// Returns g = dLoss/dlogp for the row; fills rs and *loss_tok (m*L).
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
    L = -w * fminf(rho * A, rc * A);
    const bool clipped = (A > 0.f && rho > c.hi) || (A < 0.f && rho < c.lo);
    g = clipped ? 0.f : (-w * A * rho) * c.invN;
    rs.loss = L;
    rs.clipped = clipped ? 1.f : 0.f;
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
  rs.loss = rs.clipped = rs.k3 = rs.rho = rs.stale = 0.f;
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
}

// N for the 1/N normalisation: explicit, else the global token count from rlvla_advantages
__device__ __forceinline__ double loss_denominator(double denom, const double* adv_stats) {
  if (denom > 0.0) return denom;
  if (adv_stats) return adv_stats[RLVLA_STAT_N_TOK];
  return 0.0;
}

// CTA partials (9 slots) -> workspace; last CTA writes stats[6..15]
__device__ __forceinline__ void finish_loss_stats(const double* cta_acc, double* stats,
                                                  double* partials, unsigned* ctrl, double N,
                                                  int accumulate) {
  if (threadIdx.x < 9) partials[size_t(blockIdx.x) * RLVLA_NSTATS + threadIdx.x] = cta_acc[threadIdx.x];
  __shared__ double tot[9];
  if (last_block_reduce(ctrl, partials, 9, tot)) {
    if (threadIdx.x < 9) {
      double v = tot[threadIdx.x];
      if (threadIdx.x == 0) v = N > 0.0 ? v / N : 0.0;
      if (accumulate) v += stats[RLVLA_STAT_LOSS + threadIdx.x];
      stats[RLVLA_STAT_LOSS + threadIdx.x] = v;
    }
    if (threadIdx.x == 0) stats[RLVLA_STAT_DENOM] = N;
  }
}

}  // namespace rlvla
