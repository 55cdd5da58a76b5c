// ppo.cu — S4 over precomputed log-probs (rlvla_ppo_loss, K8): the same per-row epilogue
// as the fused log-prob kernels (epilogue.cuh), one thread per row, fp64 per-CTA partials
// summed in fixed order by the last CTA. See epilogue.cuh for the definition and the
// paper anchors (P:62 staleness, P:18 decoupled objective).
#include "epilogue.cuh"

namespace rlvla {
namespace {

__global__ void __launch_bounds__(256) ppo_loss_kernel(PpoArgs a, PpoConst pc0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  PpoConst pc = pc0;
  const double N = loss_denominator(a.f.tok_denominator, a.f.adv_stats);
  pc.invN = N > 0.0 ? float(1.0 / N) : 0.f;
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
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
  __shared__ double red[8][9];
  __shared__ double cta[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) acc[k] = warp_sum_d(acc[k]);
  if (lane == 0)
    for (int k = 0; k < 9; ++k) red[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < 9) {
    double s = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    cta[threadIdx.x] = s;
  }
  __syncthreads();
  finish_loss_stats(cta, a.stats, a.ws.partials, a.ws.ctrl + CTRL_PPO, N, a.f.accumulate);
}

}  // namespace

cudaError_t launch_ppo_loss(const PpoArgs& a, cudaStream_t s) {
  if (a.rows <= 0) return cudaSuccess;
  PpoConst pc{};
  pc.has_prox = a.f.logp_prox != nullptr;
  pc.cur_version = a.f.cur_version;
  pc.eta = a.f.max_staleness;
  pc.lo = 1.f - a.f.eps_low;
  pc.hi = 1.f + a.f.eps_high;
  pc.is_cap = a.f.is_cap;
  int64_t blocks = (a.rows + 255) / 256;
  const int64_t cap = int64_t(device_info().sm_count) * 4;
  if (blocks > cap) blocks = cap;
  ppo_loss_kernel<<<int(blocks), 256, 0, s>>>(a, pc);
  return cudaGetLastError();
}

}  // namespace rlvla
