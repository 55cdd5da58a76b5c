// ppo.cu — S4 over precomputed log-probs (rlvla_ppo_loss, K8) and the clipped value loss
// (rlvla_value_loss). The token-level path uses the same per-row epilogue as the fused
// log-prob kernels (epilogue.cuh): one thread per row, fp64 per-CTA partials summed in
// fixed order by the last CTA. The chunk-level path (ratio_level = 1, reading R21) gives
// each decision step one ratio exp(sum_a m (logp - logp_behav)): one warp per step.
// Paper anchors: P:62 (staleness), P:18 (decoupled objective), P:99 (action chunks).
#include "epilogue.cuh"

namespace rlvla {
namespace {

__device__ __forceinline__ void block_finish(double* acc, int nslot, const PpoArgs& a,
                                             unsigned* ctrl, double N, float ent_coef) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double red[8][kLossSlots];
  __shared__ double cta[kLossSlots];
  for (int k = 0; k < nslot; ++k) acc[k] = warp_sum_d(acc[k]);
  if (lane == 0)
    for (int k = 0; k < nslot; ++k) red[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < nslot) {
    double s = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    cta[threadIdx.x] = s;
  }
  __syncthreads();
  finish_loss_stats(cta, a.stats, a.ws.partials, ctrl, N, a.f.accumulate, ent_coef, &a.ws.p2p);
}

__global__ void __launch_bounds__(256) ppo_loss_kernel(PpoArgs a, PpoConst pc0) {
  PpoConst pc = pc0;
  const double N = loss_denominator(a.f.tok_denominator, a.f.adv_stats);
  pc.invN = N > 0.0 ? float(1.0 / N) : 0.f;
  double acc[kLossSlots] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int A = a.f.a_tok;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < a.rows;
       r += int64_t(gridDim.x) * blockDim.x) {
    const float lp = a.logp[r];
    const int t = a.target ? a.target[r] : 0;
    PpoRowIn in;
    in.tgt_status = (t == -1) ? 1 : (t < -1 ? 2 : (isfinite(lp) ? 0 : 3));
    in.logp = lp;
    in.H = 0.f;
    in.lpb = a.f.logp_behav[r];
    in.lpp = a.f.logp_prox ? a.f.logp_prox[r] : 0.f;
    in.lref = pc.has_ref ? a.f.logp_ref[r] : 0.f;
    const int64_t s = r / A;
    in.adv = a.f.adv[s];
    in.ver = a.f.version[s];
    in.valid = a.f.slot_key[s] != 0ull;
    RowStats rs;
    float lt;
    const float g = ppo_row(pc, in, rs, &lt);
    a.grad_logp[r] = g;
    if (a.loss_tok) a.loss_tok[r] = lt;
    acc_stats(acc, rs);
  }
  if (a.stats == nullptr) return;
  block_finish(acc, kLossSlots, a, a.ws.ctrl + CTRL_PPO, N, 0.f);
}

// Chunk-level ratio: warp per decision step s. m_a = valid [usable] [0 <= lag <= eta];
// standard: lr_s = sum_a m_a (logp_a - logp_behav_a), w_s = 1; decoupled: lr_s = sum_a m_a
// (logp_a - logp_prox_a), w_s = min(exp(sum_a m_a (logp_prox_a - logp_behav_a)), cap)
// (fixed xor-tree order); rho_s = e^{lr_s}; J = min(rho A, clip(rho) A), dual clip: for
// A < 0, J = max(J, c A); L_s = -w J on steps with >= 1 masked token, Loss = sum L_s /
// N_steps; grad = -w A rho [active] / N_steps on every masked token of the step (scaled by
// the second kernel once N_steps is known); loss_tok = L_s / n_tok(s) on the step's masked
// tokens. Stats: LOSS = PG_LOSS, N_CLIPPED / N_DUAL_CLIPPED / KL_K3_SUM / RATIO_SUM per
// step, N_LOSS_TOK, N_STALE_TOK, N_BAD_TOK, LOGP_SUM per token; DENOM = N_steps.
__device__ __forceinline__ int tok_status(const PpoArgs& a, int64_t r, float lp) {
  const int t = a.target ? a.target[r] : 0;
  return (t == -1) ? 1 : (t < -1 ? 2 : (isfinite(lp) ? 0 : 3));
}

__device__ __forceinline__ double* chunk_scratch(const PpoArgs& a) {
  return reinterpret_cast<double*>(a.ws.ctrl + 32);  // 1/N_steps for the scale pass
}

// Last CTA of the chunk path (or the single CTA of an empty call): tot = this call's raw
// per-slot sums (slot 9 = the call's loss-step count). Known N (explicit, or the global
// N_LOSS_STEPS of rlvla_advantages): scale, accumulate, then C3 in-kernel. Implicit N:
// the raw sums are reduced over the ranks first so N is the global step count; with the
// NCCL fallback (defer) the raw sums and the local count (DENOM slot) are written for the
// host allreduce and the scale kernel finishes.
__device__ void chunk_finish(const PpoArgs& a, double* tot) {
  const bool implicit = !(a.f.tok_denominator > 0.0) && a.f.adv_stats == nullptr;
  if (implicit && a.stats && a.ws.p2p.nranks > 1) p2p_exchange(tot, kLossSlots, a.ws.p2p);
  __syncthreads();
  const double Ns = a.f.tok_denominator > 0.0 ? a.f.tok_denominator
                    : (a.f.adv_stats ? a.f.adv_stats[RLVLA_STAT_N_LOSS_STEPS] : tot[9]);
  const double inv = Ns > 0.0 ? 1.0 / Ns : 0.0;
  __syncthreads();
  if (threadIdx.x < kLossSlots && a.stats) {
    double v = tot[threadIdx.x];
    if (!a.defer && (threadIdx.x == 0 || threadIdx.x == 11)) v *= inv;
    if (threadIdx.x == 9) v = 0.0;  // KL_REF_SUM: no reference term on this path
    if (a.f.accumulate) v += a.stats[RLVLA_STAT_LOSS + threadIdx.x];
    tot[threadIdx.x] = v;
  }
  __syncthreads();
  if (!implicit && a.stats && a.ws.p2p.nranks > 1) p2p_exchange(tot, kLossSlots, a.ws.p2p);  // C3
  if (threadIdx.x < kLossSlots && a.stats) a.stats[RLVLA_STAT_LOSS + threadIdx.x] = tot[threadIdx.x];
  if (threadIdx.x == 0) {
    if (a.stats) a.stats[RLVLA_STAT_DENOM] = Ns;  // defer: the local count, allreduced next
    *chunk_scratch(a) = inv;
  }
}

__global__ void __launch_bounds__(256) ppo_chunk_kernel(PpoArgs a, PpoConst pc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int A = a.f.a_tok;
  const int64_t S = a.rows / A;
  const int64_t gw = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  double acc[kLossSlots] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t s = gw; s < S; s += nw) {
    const bool valid = a.f.slot_key[s] != 0ull;
    const int lag = pc.cur_version - a.f.version[s];
    const bool step_ok = valid && lag >= 0 && lag <= pc.eta;
    float lr = 0.f, lw = 0.f, ntok = 0.f, nstale = 0.f, nbad = 0.f, lps = 0.f;
    for (int j = lane; j < A; j += 32) {
      const int64_t r = s * A + j;
      const float lp = a.logp[r];
      const int stt = tok_status(a, r, lp);
      const bool usable = valid && stt == 0;
      if (usable && step_ok) {
        if (pc.has_prox) {
          const float lpp = a.f.logp_prox[r];
          lr += lp - lpp;
          lw += lpp - a.f.logp_behav[r];
        } else {
          lr += lp - a.f.logp_behav[r];
        }
        ntok += 1.f;
        lps += lp;
      }
      if (usable && lag > pc.eta) nstale += 1.f;
      if ((valid && (stt == 2 || stt == 3)) || (usable && lag < 0)) nbad += 1.f;
    }
    lr = warp_sum(lr);
    lw = warp_sum(lw);
    ntok = warp_sum(ntok);
    nstale = warp_sum(nstale);
    nbad = warp_sum(nbad);
    lps = warp_sum(lps);
    const float rho = __expf(lr);
    float w = 1.f;
    if (pc.has_prox) {
      w = __expf(lw);
      if (pc.is_cap > 0.f) w = fminf(w, pc.is_cap);
    }
    const float Aa = a.f.adv[s];
    const float rc = fminf(fmaxf(rho, pc.lo), pc.hi);
    float J = fminf(rho * Aa, rc * Aa);
    const bool clipped = (Aa > 0.f && rho > pc.hi) || (Aa < 0.f && rho < pc.lo);
    const bool dual = pc.dual_clip > 1.f && Aa < 0.f && pc.dual_clip * Aa > J;
    if (dual) J = pc.dual_clip * Aa;
    const bool has = ntok > 0.f;
    const float gs = (has && !clipped && !dual) ? -w * Aa * rho : 0.f;
    const float lt = has ? -w * J / ntok : 0.f;
    for (int j = lane; j < A; j += 32) {
      const int64_t r = s * A + j;
      const bool m = step_ok && tok_status(a, r, a.logp[r]) == 0;
      a.grad_logp[r] = m ? gs : 0.f;
      if (a.loss_tok) a.loss_tok[r] = m ? lt : 0.f;
    }
    if (lane == 0) {
      if (has) {
        acc[0] += double(-w * J);
        acc[11] += double(-w * J);
        acc[1] += (clipped && !dual) ? 1.0 : 0.0;
        acc[10] += dual ? 1.0 : 0.0;
        acc[2] += double(fabsf(lr) < 0.125f
                             ? lr * lr * (0.5f + lr * (1.f / 6.f + lr * (1.f / 24.f + lr * (1.f / 120.f + lr * (1.f / 720.f)))))
                             : (rho - 1.f - lr));
        acc[4] += double(rho);
        acc[9] += 1.0;  // number of loss steps (-> DENOM, slot zeroed in chunk_finish)
      }
      acc[5] += double(ntok);
      acc[6] += double(nstale);
      acc[7] += double(nbad);
      acc[8] += double(lps);
    }
  }
  __shared__ double red[8][kLossSlots];
  for (int k = 0; k < kLossSlots; ++k) acc[k] = warp_sum_d(acc[k]);
  if (lane == 0)
    for (int k = 0; k < kLossSlots; ++k) red[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < kLossSlots) {
    double sum = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) sum += red[w][threadIdx.x];
    a.ws.partials[size_t(blockIdx.x) * RLVLA_NSTATS + threadIdx.x] = sum;
  }
  __shared__ double tot[kLossSlots];
  if (last_block_reduce(a.ws.ctrl + CTRL_PPO, a.ws.partials, kLossSlots, tot)) chunk_finish(a, tot);
}

// second pass of the chunk path: scale the per-token step gradients by 1/N_steps; with
// defer (NCCL fallback, implicit N) N is the allreduced count in stats[DENOM] and CTA 0
// also normalises the allreduced LOSS / PG_LOSS sums
__global__ void __launch_bounds__(256) ppo_chunk_scale_kernel(PpoArgs a) {
  float fi;
  if (a.defer) {
    const double N = a.stats[RLVLA_STAT_DENOM];
    const double inv = N > 0.0 ? 1.0 / N : 0.0;
    fi = float(inv);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.stats[RLVLA_STAT_LOSS] *= inv;
      a.stats[RLVLA_STAT_PG_LOSS] *= inv;
    }
  } else {
    fi = float(*chunk_scratch(a));
  }
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < a.rows;
       r += int64_t(gridDim.x) * blockDim.x)
    a.grad_logp[r] *= fi;
}

}  // namespace

cudaError_t launch_ppo_loss(const PpoArgs& a, cudaStream_t s) {
  // rows == 0 still launches one CTA when statistics are requested: the call's totals are
  // written (or accumulated) and, across ranks, this rank takes part in C3
  if (a.rows <= 0 && a.stats == nullptr) return cudaSuccess;
  PpoConst pc{};
  pc.has_prox = a.f.logp_prox != nullptr;
  pc.has_ref = a.f.logp_ref != nullptr && a.f.kl_coef != 0.f;
  pc.cur_version = a.f.cur_version;
  pc.eta = a.f.max_staleness;
  pc.lo = 1.f - a.f.eps_low;
  pc.hi = 1.f + a.f.eps_high;
  pc.is_cap = a.f.is_cap;
  pc.dual_clip = a.f.dual_clip;
  pc.kl_coef = a.f.kl_coef;
  pc.ent_coef = 0.f;  // no logits here: the entropy bonus lives in the logits path
  const int sms = device_info().sm_count;
  if (a.f.ratio_level == 1) {
    const int64_t S = a.rows / a.f.a_tok;
    int64_t blocks = (S + 7) / 8;
    if (blocks > int64_t(sms) * 4) blocks = int64_t(sms) * 4;
    if (blocks < 1) blocks = 1;
    ppo_chunk_kernel<<<int(blocks), 256, 0, s>>>(a, pc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || a.defer) return e;  // defer: the API allreduces, then scales
    return launch_ppo_chunk_scale(a, s);
  }
  int64_t blocks = (a.rows + 255) / 256;
  const int64_t cap = int64_t(sms) * 4;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  ppo_loss_kernel<<<int(blocks), 256, 0, s>>>(a, pc);
  return cudaGetLastError();
}

cudaError_t launch_ppo_chunk_scale(const PpoArgs& a, cudaStream_t s) {
  int64_t b2 = (a.rows + 255) / 256;
  const int64_t cap = int64_t(device_info().sm_count) * 4;
  if (b2 > cap) b2 = cap;
  if (b2 < 1) b2 = 1;
  ppo_chunk_scale_kernel<<<int(b2), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rlvla
