// advantages.cu — S2: GAE reverse segmented scan (+ global whitening) and GRPO group
// normalisation. The paper never writes these ("Hyperparameters related to
// the optimizer and learning algorithm ... are omitted"); definitions are the
// textbook ones (GAE: Schulman et al. 2016; GRPO: Shao et al. 2024) with readings
// R7-R10.
//
// GAE as a scan: per step the recursion A_t = delta_t + c_t A_{t+1} is the affine map
// f_t(A) = delta_t + c_t A with c_t = gamma lam nt_t. One warp per env walks the T axis
// in 32-step tiles from the end; inside a tile a 5-level Hillis-Steele suffix scan of
// the maps (D, C) o (D', C') = (D + C D', C C') gives every lane its composed map, which
// is applied to the carry A of the tile to the right. Loads/stores are coalesced per
// tile; the dependency chain is ceil(T/32) tiles deep.
#include "internal.cuh"

namespace rlvla {
namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ bool step_ok_for_loss(int valid, int ver, const rlvla_adv_params& p,
                                                 int* stale, int* bad) {
  const int lag = p.cur_version - ver;
  *stale = valid && lag > p.max_staleness;
  *bad = valid && lag < 0;
  return valid && lag >= 0 && lag <= p.max_staleness;
}

// Tokens that will carry loss (target >= 0 on filled steps with 0 <= lag <= eta): one
// thread per token over the whole grid (the step's key/version are L1/L2 hits shared by
// its A tokens), four independent tokens in flight per thread so each pass of the loop
// costs one memory round trip whatever A is. The thread holding a step's token 0 also
// counts the step as a loss step (the chunk-ratio normaliser, slot N_LOSS_STEPS) when
// one of its tokens has target >= 0: its own token decides unless it is ignored (-1),
// only then are the step's later tokens read.
struct LossCounts {
  long long tok, steps;
};
__device__ __forceinline__ LossCounts count_loss_tokens(const AdvArgs& a) {
  const int64_t A = a.buf.a_tok;
  const int64_t ntok = int64_t(a.buf.n_env) * a.buf.t_steps * A;
  const int64_t gt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nt = int64_t(gridDim.x) * blockDim.x;
  LossCounts c{0, 0};
  for (int64_t k0 = gt; k0 < ntok; k0 += 4 * nt) {
    int tk[4], ver[4];
    bool first[4];
    unsigned long long key[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t k = k0 + u * nt;
      tk[u] = -1;
      key[u] = 0ull;
      ver[u] = 0;
      first[u] = false;
      if (k < ntok) {
        const int64_t s = ntok <= INT32_MAX ? int64_t(uint32_t(k) / uint32_t(A)) : k / A;
        tk[u] = a.buf.tokens[k];
        key[u] = a.buf.slot_key[s];
        ver[u] = a.buf.version[s];
        first[u] = k == s * A;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int lag = a.p.cur_version - ver[u];
      const bool ok = key[u] != 0ull && lag >= 0 && lag <= a.p.max_staleness;
      c.tok += (ok && tk[u] >= 0);
      if (ok && first[u]) {
        bool has = tk[u] >= 0;
        const int64_t k = k0 + u * nt;
        for (int64_t j = 1; !has && j < A; ++j) has = a.buf.tokens[k + j] >= 0;
        c.steps += has;
      }
    }
  }
  return c;
}

// ------------------------------------------------------------------------------------
// GAE pass 1: scan + per-CTA partials (n_valid, sum A, sum A^2, n_tok, n_stale, n_bad)
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gae_scan_kernel(AdvArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int E = a.buf.n_env, T = a.buf.t_steps;
  const float gamma = a.p.gamma, gl = a.p.gamma * a.p.lam;
  double s_n = 0, s_a = 0, s_a2 = 0;
  long long s_tok = 0, s_stale = 0, s_bad = 0;
  const int nwarps = gridDim.x * kWarpsPerBlock;
  for (int e = blockIdx.x * kWarpsPerBlock + warp; e < E; e += nwarps) {
    const float lv = a.last_value ? a.last_value[e] : 0.f;
    float carryA = 0.f, carryV = lv;
    int carry_v = 1;
    const int ntile = (T + 31) >> 5;
    for (int tile = ntile - 1; tile >= 0; --tile) {
      const int t = tile * 32 + lane;
      const bool in = t < T;
      const int64_t idx = int64_t(e) * T + t;
      float r = 0.f, V = 0.f, B = 0.f;
      int d = 0, v = 0, ver = 0;
      if (in) {
        r = a.buf.reward[idx];
        V = a.buf.value[idx];
        d = a.buf.done[idx];
        v = a.buf.slot_key[idx] != 0ull;
        ver = a.buf.version[idx];
        if (d == 2 && a.p.boot_value) B = a.p.boot_value[idx];  // truncation bootstrap
      }
      float Vn = __shfl_down_sync(0xffffffffu, V, 1);
      int vn = __shfl_down_sync(0xffffffffu, v, 1);
      if (lane == 31) {
        Vn = carryV;
        vn = carry_v;
      }
      if (t == T - 1) {
        Vn = lv;
        vn = 1;
      }
      // done 1 = termination, 2 = time-limit truncation (recursion cut, bootstrap from B)
      const float nt = (v && d == 0 && vn) ? 1.f : 0.f;
      const float tr = (d == 2) ? 1.f : 0.f;
      float D = v ? (r + gamma * fmaf(nt, Vn, tr * B) - V) : 0.f;
      float C = gl * nt;
      if (!in) {  // identity map on padding lanes
        D = 0.f;
        C = 1.f;
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const float Dn = __shfl_down_sync(0xffffffffu, D, off);
        const float Cn = __shfl_down_sync(0xffffffffu, C, off);
        if (lane + off < 32) {
          D = fmaf(C, Dn, D);
          C = C * Cn;
        }
      }
      const float Aval = fmaf(C, carryA, D);
      int stale, bad;
      const int ok = step_ok_for_loss(v, ver, a.p, &stale, &bad);
      if (in) {
        a.adv[idx] = v ? Aval : 0.f;
        if (a.ret) a.ret[idx] = v ? Aval + V : 0.f;
        if (v) {
          s_n += 1.0;
          s_a += double(Aval);
          s_a2 += double(Aval) * double(Aval);
        }
        s_stale += stale;
        s_bad += bad;
      }
      carryA = __shfl_sync(0xffffffffu, Aval, 0);
      carryV = __shfl_sync(0xffffffffu, V, 0);
      carry_v = __shfl_sync(0xffffffffu, v, 0);
    }
  }
  const LossCounts lc = count_loss_tokens(a);
  s_tok += lc.tok;
  // CTA partials: warp reduce then fixed-order over warps (slot 6 -> stats[N_LOSS_STEPS])
  __shared__ double red[kWarpsPerBlock][7];
  s_n = warp_sum_d(s_n);
  s_a = warp_sum_d(s_a);
  s_a2 = warp_sum_d(s_a2);
  const double t_tok = double(warp_sum_ll(s_tok));
  const double t_st = double(warp_sum_ll(s_stale));
  const double t_bad = double(warp_sum_ll(s_bad));
  const double t_steps = double(warp_sum_ll(lc.steps));
  if (lane == 0) {
    red[warp][0] = s_n;
    red[warp][1] = s_a;
    red[warp][2] = s_a2;
    red[warp][3] = t_tok;
    red[warp][4] = t_st;
    red[warp][5] = t_bad;
    red[warp][6] = t_steps;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double acc = 0;
    for (int w = 0; w < kWarpsPerBlock; ++w) acc += red[w][threadIdx.x];
    a.ws.partials[size_t(blockIdx.x) * RLVLA_NSTATS + threadIdx.x] = acc;
  }
  __shared__ double tot[7];
  if (last_block_reduce(a.ws.ctrl + CTRL_ADV, a.ws.partials, 7, tot)) {
    if (a.ws.p2p.nranks > 1) p2p_exchange(tot, 7, a.ws.p2p);  // C1 in-kernel (NVLink)
    if (threadIdx.x < 6) a.stats[threadIdx.x] = tot[threadIdx.x];
    if (threadIdx.x == 6) a.stats[RLVLA_STAT_N_LOSS_STEPS] = tot[6];
  }
}

// ------------------------------------------------------------------------------------
// GRPO pass 1: per-env returns R_e = sum_t valid r_t  -> ws.r_global[env_offset + e]
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) grpo_returns_kernel(AdvArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int E = a.buf.n_env, T = a.buf.t_steps;
  double s_n = 0;
  long long s_tok = 0, s_stale = 0, s_bad = 0;
  const int nwarps = gridDim.x * kWarpsPerBlock;
  for (int e = blockIdx.x * kWarpsPerBlock + warp; e < E; e += nwarps) {
    float R = 0.f;
    const int ntile = (T + 31) >> 5;
    for (int tile = 0; tile < ntile; ++tile) {
      const int t = tile * 32 + lane;
      const bool in = t < T;
      const int64_t idx = int64_t(e) * T + t;
      int v = 0, ver = 0;
      float r = 0.f;
      if (in) {
        v = a.buf.slot_key[idx] != 0ull;
        r = a.buf.reward[idx];
        ver = a.buf.version[idx];
      }
      if (v) R += r;
      s_n += v;
      int stale, bad;
      (void)step_ok_for_loss(v, ver, a.p, &stale, &bad);
      s_stale += stale;
      s_bad += bad;
    }
    R = warp_sum(R);  // fixed xor tree: identical for any rank count
    if (lane == 0) a.ws.r_global[a.p.env_offset + e] = R;
  }
  const LossCounts lc = count_loss_tokens(a);
  s_tok += lc.tok;
  __shared__ double red[kWarpsPerBlock][5];
  s_n = warp_sum_d(s_n);
  const double t_tok = double(warp_sum_ll(s_tok));
  const double t_st = double(warp_sum_ll(s_stale));
  const double t_bad = double(warp_sum_ll(s_bad));
  const double t_steps = double(warp_sum_ll(lc.steps));
  if (lane == 0) {
    red[warp][0] = s_n;
    red[warp][1] = t_tok;
    red[warp][2] = t_st;
    red[warp][3] = t_bad;
    red[warp][4] = t_steps;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double acc = 0;
    const int tx = int(threadIdx.x);
    // slots 0,3,4,5,6 <- red 0..4 (slot 6 -> stats[N_LOSS_STEPS]); slots 1,2 = 0
    const int src = tx == 0 ? 0 : (tx >= 3 ? tx - 2 : -1);
    if (src >= 0)
      for (int w = 0; w < kWarpsPerBlock; ++w) acc += red[w][src];
    a.ws.partials[size_t(blockIdx.x) * RLVLA_NSTATS + threadIdx.x] = acc;
  }
  __shared__ double tot[7];
  if (last_block_reduce(a.ws.ctrl + CTRL_ADV, a.ws.partials, 7, tot)) {
    // C1 + C2 in-kernel (NVLink): statistics summed, every rank's returns gathered
    if (a.ws.p2p.nranks > 1)
      p2p_exchange(tot, 7, a.ws.p2p, a.ws.r_global + a.p.env_offset, a.p.env_offset, E, a.ws.r_global,
                   a.p.n_env_global);
    if (threadIdx.x < 6) a.stats[threadIdx.x] = tot[threadIdx.x];
    if (threadIdx.x == 6) a.stats[RLVLA_STAT_N_LOSS_STEPS] = tot[6];
  }
}

// ------------------------------------------------------------------------------------
// GRPO pass 2: group statistics from the (gathered) returns, fixed member order
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) grpo_normalize_kernel(AdvArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int E = a.buf.n_env, T = a.buf.t_steps;
  const int Eg = a.p.n_env_global;
  const float* Rg = a.ws.r_global;
  const int nwarps = gridDim.x * kWarpsPerBlock;
  for (int e = blockIdx.x * kWarpsPerBlock + warp; e < E; e += nwarps) {
    const int ge = a.p.env_offset + e;
    double n = 0, s = 0;
    int gid, lo = 0, hi = Eg;
    if (a.p.group_id) {
      gid = a.p.group_id[ge];
    } else {
      gid = ge / a.p.group_size;
      lo = gid * a.p.group_size;
      hi = min(Eg, lo + a.p.group_size);
    }
    for (int j = lo + lane; j < hi; j += 32) {
      const bool mem = a.p.group_id ? (a.p.group_id[j] == gid) : true;
      if (mem) {
        n += 1.0;
        s += double(Rg[j]);
      }
    }
    n = warp_sum_d(n);
    s = warp_sum_d(s);
    const double mu = n > 0 ? s / n : 0.0;
    double ss = 0;
    for (int j = lo + lane; j < hi; j += 32) {
      const bool mem = a.p.group_id ? (a.p.group_id[j] == gid) : true;
      if (mem) {
        const double d = double(Rg[j]) - mu;
        ss += d * d;
      }
    }
    ss = warp_sum_d(ss);
    const float Re = Rg[ge];
    float Ae = 0.f;
    if (n >= 2.0) {
      const double sigma = sqrt(ss / (a.p.std_unbiased ? (n - 1.0) : n));
      Ae = float((double(Re) - mu) / (sigma + double(a.p.grpo_eps)));
    }
    for (int t = lane; t < T; t += 32) {
      const int64_t idx = int64_t(e) * T + t;
      const bool v = a.buf.slot_key[idx] != 0ull;
      a.adv[idx] = v ? Ae : 0.f;
      if (a.ret) a.ret[idx] = v ? Re : 0.f;
    }
  }
}

// GAE pass 2: global whitening with the (allreduced) stats slots 0..2 (reading R9)
__global__ void __launch_bounds__(256) whiten_kernel(AdvArgs a) {
  const double n = a.stats[RLVLA_STAT_N_VALID_STEPS];
  const double s1 = a.stats[RLVLA_STAT_SUM_ADV];
  const double s2 = a.stats[RLVLA_STAT_SUM_ADV2];
  const double mu = n > 0 ? s1 / n : 0.0;
  double var = n > 1 ? (s2 - n * mu * mu) / (n - 1.0) : 0.0;
  if (var < 0) var = 0;
  const double inv = 1.0 / (sqrt(var) + double(a.p.whiten_eps));
  const int64_t total = int64_t(a.buf.n_env) * a.buf.t_steps;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const bool v = a.buf.slot_key[i] != 0ull;
    a.adv[i] = v ? float((double(a.adv[i]) - mu) * inv) : 0.f;
  }
}

int adv_grid(int E) {
  int g = (E + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int cap = 4 * device_info().sm_count;
  if (g > cap) g = cap;
  if (g > kMaxPartialBlocks) g = kMaxPartialBlocks;
  return g < 1 ? 1 : g;
}

// pass 1 also sweeps the E*T*A tokens for the token count: ~4 tokens per thread
int pass1_grid(int E, int T, int A) {
  int g = adv_grid(E);
  const int64_t toks = int64_t(E) * T * A;
  int64_t gs = (toks + 4 * 256 - 1) / (4 * 256);
  const int cap = 8 * device_info().sm_count;
  if (gs > cap) gs = cap;
  if (gs > g) g = int(gs);
  if (g > kMaxPartialBlocks) g = kMaxPartialBlocks;
  return g;
}

}  // namespace

cudaError_t launch_adv_pass1(const AdvArgs& a, cudaStream_t s) {
  const int g = pass1_grid(a.buf.n_env, a.buf.t_steps, a.buf.a_tok);
  if (a.p.mode == RLVLA_ADV_GAE) gae_scan_kernel<<<g, 256, 0, s>>>(a);
  else grpo_returns_kernel<<<g, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_adv_pass2(const AdvArgs& a, cudaStream_t s) {
  if (a.p.mode == RLVLA_ADV_GAE) {
    if (!a.p.whiten) return cudaSuccess;
    const int64_t total = int64_t(a.buf.n_env) * a.buf.t_steps;
    int g = int((total + 255) / 256);
    const int cap = 4 * device_info().sm_count;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    whiten_kernel<<<g, 256, 0, s>>>(a);
  } else {
    grpo_normalize_kernel<<<adv_grid(a.buf.n_env), 256, 0, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace rlvla
