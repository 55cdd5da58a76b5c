// value.cu — clipped value-head loss per decision step (rlvla_value_loss; SURVEY NEXT-2,
// paper-silent, reading R22): L = 0.5 max((v - R)^2, (v_old + clip(v - v_old, -e, e) - R)^2),
// m = [filled][0 <= lag <= eta] (the staleness bound of P:62 applies to the value targets
// too), Loss = sum m L / N_v. One thread per step, fp64 per-CTA partials, fixed-order
// last-CTA reduction; a second pass applies 1/N_v when N_v is the call's own count.
#include "internal.cuh"

namespace rlvla {
namespace {

__device__ __forceinline__ double* value_scratch(const ValueArgs& a) {
  return reinterpret_cast<double*>(a.ws.ctrl + 34);  // 1/N_v for the scale pass
}

__global__ void __launch_bounds__(256) value_loss_kernel(ValueArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool explicit_n = a.denominator > 0.0;
  const float inv_e = explicit_n ? float(1.0 / a.denominator) : 1.f;
  double acc[3] = {0, 0, 0};  // sum m L, #clipped, sum m
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < a.n;
       s += int64_t(gridDim.x) * blockDim.x) {
    const int lag = a.cur_version - a.version[s];
    const bool m = a.slot_key[s] != 0ull && lag >= 0 && lag <= a.max_staleness;
    float g = 0.f, L = 0.f;
    bool use_c = false;
    if (m) {
      const float v = a.v_new[s], R = a.ret[s];
      const float du = v - R;
      float u = du * du;
      if (a.clip_eps > 0.f) {
        const float d = v - a.v_old[s];
        const float vc = a.v_old[s] + fminf(fmaxf(d, -a.clip_eps), a.clip_eps);
        const float dc = vc - R;
        const float c = dc * dc;
        // the clipped branch counts only where the clip moved v (inside the interval
        // v_clip == v, so c vs u would be a rounding coin-flip with the same gradient)
        use_c = fabsf(d) > a.clip_eps && c > u;
        g = use_c ? 0.f : du;  // outside the interval d clip / dv = 0
        L = 0.5f * fmaxf(u, c);
      } else {
        g = du;
        L = 0.5f * u;
      }
      acc[0] += double(L);
      acc[1] += use_c ? 1.0 : 0.0;
      acc[2] += 1.0;
    }
    a.grad_v[s] = m ? g * inv_e : 0.f;
    if (a.loss_step) a.loss_step[s] = L;
  }
  __shared__ double red[8][3];
  for (int k = 0; k < 3; ++k) acc[k] = warp_sum_d(acc[k]);
  if (lane == 0)
    for (int k = 0; k < 3; ++k) red[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < 3) {
    double sum = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) sum += red[w][threadIdx.x];
    a.ws.partials[size_t(blockIdx.x) * RLVLA_NSTATS + threadIdx.x] = sum;
  }
  __shared__ double tot[3];
  if (last_block_reduce(a.ws.ctrl + CTRL_VALUE, a.ws.partials, 3, tot)) {
    // implicit N_v: the raw sums are reduced over the ranks first (in-kernel), so N_v is the
    // global step count; with the NCCL fallback (defer) the raw sums go out and the scale
    // kernel finishes after the host allreduce
    if (!explicit_n && a.stats && a.ws.p2p.nranks > 1) p2p_exchange(tot, 3, a.ws.p2p);
    __syncthreads();
    const double N = explicit_n ? a.denominator : tot[2];
    const double inv = N > 0.0 ? 1.0 / N : 0.0;
    __syncthreads();
    if (threadIdx.x == 0) {
      *value_scratch(a) = inv;
      if (!a.defer) tot[0] *= inv;  // this rank's share of the loss, as the NCCL path reduces it
    }
    __syncthreads();
    if (explicit_n && a.stats && a.ws.p2p.nranks > 1) p2p_exchange(tot, 3, a.ws.p2p);  // in-kernel (NVLink)
    if (threadIdx.x == 0 && a.stats) {
      a.stats[RLVLA_STAT_VALUE_LOSS] = tot[0];
      a.stats[RLVLA_STAT_N_VALUE_CLIPPED] = tot[1];
      a.stats[RLVLA_STAT_N_VALUE_STEPS] = tot[2];
      a.stats[RLVLA_STAT_VALUE_DENOM] = a.defer ? 0.0 : N;
    }
  }
}

// second pass when N_v is the call's own count: scale the gradients by 1/N_v; with defer
// (NCCL fallback) N_v is the allreduced count in stats and CTA 0 normalises the loss slot
__global__ void __launch_bounds__(256) value_scale_kernel(ValueArgs a) {
  float fi;
  if (a.defer) {
    const double N = a.stats[RLVLA_STAT_N_VALUE_STEPS];
    const double inv = N > 0.0 ? 1.0 / N : 0.0;
    fi = float(inv);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.stats[RLVLA_STAT_VALUE_LOSS] *= inv;
      a.stats[RLVLA_STAT_VALUE_DENOM] = N;
    }
  } else {
    fi = float(*value_scratch(a));
  }
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < a.n;
       s += int64_t(gridDim.x) * blockDim.x)
    a.grad_v[s] *= fi;
}

int value_grid(int64_t n) {
  const int sms = device_info().sm_count;
  int64_t blocks = (n + 255) / 256;
  if (blocks > int64_t(sms) * 4) blocks = int64_t(sms) * 4;
  return blocks < 1 ? 1 : int(blocks);
}

}  // namespace

// n == 0 still launches one CTA when statistics are requested (this rank's zeros take part
// in the cross-rank reduction)
cudaError_t launch_value_loss(const ValueArgs& a, cudaStream_t s) {
  if (a.n <= 0 && a.stats == nullptr) return cudaSuccess;
  value_loss_kernel<<<value_grid(a.n), 256, 0, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || a.denominator > 0.0 || a.defer) return e;
  return launch_value_scale(a, s);
}

cudaError_t launch_value_scale(const ValueArgs& a, cudaStream_t s) {
  value_scale_kernel<<<value_grid(a.n), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rlvla
