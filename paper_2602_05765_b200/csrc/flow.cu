// flow.cu — NEXT-4: log-likelihood of a flow / diffusion policy's action chunk as a chain of
// K Gaussian denoising transitions (reading R25; pi_0 / pi_0.5 / GR00T, P:39, P:77, P:99,
// Table 2 "Model Num Step" = 4), optionally fused with the PPO epilogue and its backward.
//
// Warp tiles of kTile = 4 decision steps (flow_kernel; the launch picks a compile-time row
// length for the paper's K x D shapes, 280 and 140):
//   pass 1  step by step, the row's n = K*D elements are streamed with 4-wide loads (mu in
//           f32 or bf16, x, optional ln sigma; a sigma schedule is a per-element 1/sigma
//           table in SMEM, so there is no division) and packed fp32x2 math; each lane's
//           partial sum of z^2 (and ln sigma) goes to SMEM [step][lane]
//   epilogue lane t owns step t of the tile: it sums the 32 partials in fixed order in fp64,
//           forms logp = -0.5 sum z^2 - sum ln sigma - n ln(2 pi)/2 and
//           H = sum ln sigma + n (ln 2 pi + 1)/2, and runs the shared PPO epilogue
//           (epilogue.cuh) — the per-step scalar work spread over the lanes
//   pass 2  step by step, g and c are broadcast and the backward re-reads the row (L1/L2):
//           dmu = g z / sigma,   dln sigma = g (z^2 - 1) - c     (c = ent_coef m / N)
// Rows whose length is not a multiple of 4 (or unaligned pointers) take scalar loops.
// Bytes per row: n (|mu| + 4 [+ 4 ln sigma]) read, n |mu| [+ 4 n] written.
#include "epilogue.cuh"

namespace rlvla {
namespace {

constexpr int kFlowWarps = 8;

template <typename T>
__device__ __forceinline__ float ld_mu(const void* p, int64_t i);
template <>
__device__ __forceinline__ float ld_mu<float>(const void* p, int64_t i) {
  return static_cast<const float*>(p)[i];
}
template <>
__device__ __forceinline__ float ld_mu<__nv_bfloat16>(const void* p, int64_t i) {
  return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}
template <typename T>
__device__ __forceinline__ void st_mu(void* p, int64_t i, float v);
template <>
__device__ __forceinline__ void st_mu<float>(void* p, int64_t i, float v) {
  static_cast<float*>(p)[i] = v;
}
template <>
__device__ __forceinline__ void st_mu<__nv_bfloat16>(void* p, int64_t i, float v) {
  static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
}

// 4 consecutive means as fp32 (one 8-byte bf16 or one 16-byte fp32 load)
template <typename T>
__device__ __forceinline__ float4 ld_mu4(const void* p, int64_t i);
template <>
__device__ __forceinline__ float4 ld_mu4<float>(const void* p, int64_t i) {
  return *reinterpret_cast<const float4*>(static_cast<const float*>(p) + i);
}
template <>
__device__ __forceinline__ float4 ld_mu4<__nv_bfloat16>(const void* p, int64_t i) {
  const uint2 w = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(p) + i);
  return make_float4(bf_lo(w.x), bf_hi(w.x), bf_lo(w.y), bf_hi(w.y));
}
template <typename T>
__device__ __forceinline__ void st_mu4(void* p, int64_t i, float4 v);
template <>
__device__ __forceinline__ void st_mu4<float>(void* p, int64_t i, float4 v) {
  *reinterpret_cast<float4*>(static_cast<float*>(p) + i) = v;
}
template <>
__device__ __forceinline__ void st_mu4<__nv_bfloat16>(void* p, int64_t i, float4 v) {
  *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p) + i) =
      make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
}

#ifndef RLVLA_FLOW_TILE
#define RLVLA_FLOW_TILE 4  // rows per warp tile (<= 32): one lane runs each row's epilogue
#endif
constexpr int kTile = RLVLA_FLOW_TILE;
constexpr int kPad = 33;  // partials [row][lane] padded: conflict-free row-wise reads

struct RowMeta4 {
  float lpb = 0.f, lpp = 0.f, lref = 0.f, adv = 0.f;
  int ver = 0;
  bool valid = true;
};

// One row's lane partials: q = sum z^2 and ls = sum ln sigma (learned) over the lane's
// elements. Row pointers are formed once, indices stay 32-bit.
template <typename T, bool VEC, int NQ>
__device__ __forceinline__ void row_partials(const T* mu0, const float* x0, const float* ls0,
                                             const float* s_isig, int64_t base, int n, bool learned,
                                             int lane, float& q, float& ls) {
  const T* mu = mu0 + base;
  const float* x = x0 + base;
  const float* lsd = learned ? ls0 + base : nullptr;
  q = 0.f;
  ls = 0.f;
  if (VEC) {
    float2 q2 = make_float2(0.f, 0.f);
    // NQ > 0: the row length is a compile-time constant (the paper's K D shapes), so the
    // loop unrolls into predicated copies with immediate offsets
    constexpr int kIters = NQ > 0 ? (NQ + 31) / 32 : 1;
    const int nq = NQ > 0 ? NQ : (n >> 2);
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      for (int gi = lane + 32 * it; gi < nq; gi += (NQ > 0 ? nq : 32)) {
        const int j = 4 * gi;
        const float4 m = ld_mu4<T>(mu, j);
        const float4 xv = *reinterpret_cast<const float4*>(x + j);
        float4 iv;
        if (learned) {
          const float4 l = *reinterpret_cast<const float4*>(lsd + j);
          iv = make_float4(__expf(-l.x), __expf(-l.y), __expf(-l.z), __expf(-l.w));
          ls += (l.x + l.y) + (l.z + l.w);
        } else {
          iv = *reinterpret_cast<const float4*>(s_isig + j);
        }
        // packed fp32x2 (FADD2 / FMUL2 / FFMA2): two elements per instruction
        const float2 za = __fmul2_rn(__fadd2_rn(make_float2(xv.x, xv.y), make_float2(-m.x, -m.y)),
                                     make_float2(iv.x, iv.y));
        const float2 zb = __fmul2_rn(__fadd2_rn(make_float2(xv.z, xv.w), make_float2(-m.z, -m.w)),
                                     make_float2(iv.z, iv.w));
        q2 = __ffma2_rn(za, za, __ffma2_rn(zb, zb, q2));
      }
    }
    q = q2.x + q2.y;
  } else {
    for (int j = lane; j < n; j += 32) {
      const float m = ld_mu<T>(mu, j);
      float iv;
      if (learned) {
        const float l = lsd[j];
        iv = __expf(-l);
        ls += l;
      } else {
        iv = s_isig[j];
      }
      const float zz = (x[j] - m) * iv;
      q = fmaf(zz, zz, q);
    }
  }
}

// dmu = g z / sigma, dln sigma = g (z^2 - 1) - c for one row (exact zeros when g = c = 0)
template <typename T, bool VEC, int NQ>
__device__ __forceinline__ void row_backward(const T* mu0, const float* x0, const float* ls0, T* dmu0,
                                             float* dls0, const float* s_isig, int64_t base, int n,
                                             bool learned, int lane, float g, float c) {
  const bool active = g != 0.f || c != 0.f;
  const T* mu = mu0 + base;
  const float* x = x0 + base;
  const float* lsd = learned ? ls0 + base : nullptr;
  T* dmu = dmu0 ? dmu0 + base : nullptr;
  float* dls = dls0 ? dls0 + base : nullptr;
  if (VEC) {
    constexpr int kIters = NQ > 0 ? (NQ + 31) / 32 : 1;
    const int nq = NQ > 0 ? NQ : (n >> 2);
#pragma unroll
    for (int it = 0; it < kIters; ++it)
    for (int gi = lane + 32 * it; gi < nq; gi += (NQ > 0 ? nq : 32)) {
      const int j = 4 * gi;
      float4 dm = make_float4(0.f, 0.f, 0.f, 0.f), dl = dm;
      if (active) {
        const float4 m = ld_mu4<T>(mu, j);
        const float4 xv = *reinterpret_cast<const float4*>(x + j);
        float4 iv;
        if (learned) {
          const float4 l = *reinterpret_cast<const float4*>(lsd + j);
          iv = make_float4(__expf(-l.x), __expf(-l.y), __expf(-l.z), __expf(-l.w));
        } else {
          iv = *reinterpret_cast<const float4*>(s_isig + j);
        }
        const float2 ia = make_float2(iv.x, iv.y), ib = make_float2(iv.z, iv.w);
        const float2 za = __fmul2_rn(__fadd2_rn(make_float2(xv.x, xv.y), make_float2(-m.x, -m.y)), ia);
        const float2 zb = __fmul2_rn(__fadd2_rn(make_float2(xv.z, xv.w), make_float2(-m.z, -m.w)), ib);
        const float2 g2 = make_float2(g, g);
        const float2 da = __fmul2_rn(__fmul2_rn(g2, za), ia), db = __fmul2_rn(__fmul2_rn(g2, zb), ib);
        dm = make_float4(da.x, da.y, db.x, db.y);
        const float z0 = za.x, z1 = za.y, z2 = zb.x, z3 = zb.y;
        if (dls)
          dl = make_float4(fmaf(g, fmaf(z0, z0, -1.f), -c), fmaf(g, fmaf(z1, z1, -1.f), -c),
                           fmaf(g, fmaf(z2, z2, -1.f), -c), fmaf(g, fmaf(z3, z3, -1.f), -c));
      }
      if (dmu) st_mu4<T>(dmu, j, dm);
      if (dls) *reinterpret_cast<float4*>(dls + j) = dl;
    }
  } else {
    for (int j = lane; j < n; j += 32) {
      float zz = 0.f, iv = 1.f;
      if (active) {
        const float m = ld_mu<T>(mu, j);
        iv = learned ? __expf(-lsd[j]) : s_isig[j];
        zz = (x[j] - m) * iv;
      }
      if (dmu) st_mu<T>(dmu, j, active ? g * zz * iv : 0.f);
      if (dls) dls[j] = active ? fmaf(g, fmaf(zz, zz, -1.f), -c) : 0.f;
    }
  }
}

// MODE 0: forward only, 1: fused PPO, 2: external backward (grad_logp given).
// A warp takes tiles of kTile rows. Pass 1: row by row, coalesced element-parallel loads,
// each lane's partial sums parked in SMEM [row][lane]. Epilogue: lane t owns row t of the
// tile: it sums the 32 partials in fixed order in fp64, forms logp / H and runs the PPO
// epilogue (its metadata loads are coalesced across lanes) — the per-row scalar work is
// spread over the lanes instead of repeated by all 32. Pass 2: row by row, g and c are
// broadcast and the backward re-reads the row (L1/L2) to write dmu / dln sigma.
// VEC: 4-wide vector loads (n % 4 == 0, aligned pointers); otherwise scalar loops.
#ifndef RLVLA_FLOW_MINB
#define RLVLA_FLOW_MINB 4  // resident CTAs per SM the register budget is sized for
#endif
template <typename T, int MODE, bool VEC, int NQ>
__global__ void __launch_bounds__(kFlowWarps * 32, RLVLA_FLOW_MINB) flow_kernel(FlowArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = a.c.n_steps, D = a.c.dim, n = NQ > 0 ? 4 * NQ : K * D;
  const bool learned = a.c.log_std != nullptr;
  const bool want_stats = a.stats != nullptr && MODE != 2;
  // the row arrays in registers once (not re-read from the parameter bank per row)
  const T* const mu0 = static_cast<const T*>(a.c.mu);
  const float* const x0 = a.c.x;
  const float* const ls0 = a.c.log_std;
  T* const dmu0 = static_cast<T*>(a.dmu);
  float* const dls0 = a.dlog_std;
  extern __shared__ __align__(16) float dsm[];
  float* s_isig = dsm;                                        // [n] (sigma schedule)
  float* pq = dsm + ((n + 3) & ~3) + warp * 2 * kTile * kPad;  // [kTile][kPad] per warp
  float* pl = pq + kTile * kPad;
  __shared__ double s_lnsig;
  // sigma schedule: 1/sigma per element (no division or k = j / D in the loops) and
  // D sum_k ln sigma_k in fp64, once per CTA
  if (!learned) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) s_isig[j] = 1.f / a.c.sigma_k[j / D];
    if (threadIdx.x == 0) {
      double acc = 0.0;
      for (int k = 0; k < K; ++k) acc += log(double(a.c.sigma_k[k]));
      s_lnsig = acc * double(D);
    }
  }
  __syncthreads();
  const double cst = 0.5 * 1.8378770664093453 * double(n);  // n ln(2 pi) / 2
  PpoConst pc{};
  double Nden = 0.0;
  if (MODE == 1) {
    pc.has_prox = a.f.logp_prox != nullptr;
    pc.has_ref = a.f.logp_ref != nullptr && a.f.kl_coef != 0.f;
    pc.cur_version = a.f.cur_version;
    pc.eta = a.f.max_staleness;
    pc.lo = 1.f - a.f.eps_low;
    pc.hi = 1.f + a.f.eps_high;
    pc.is_cap = a.f.is_cap;
    pc.dual_clip = a.f.dual_clip;
    pc.kl_coef = a.f.kl_coef;
    pc.ent_coef = a.f.ent_coef;
    Nden = loss_denominator(a.f.tok_denominator, a.f.adv_stats);
    pc.invN = Nden > 0.0 ? float(1.0 / Nden) : 0.f;
  }
  // per-lane statistics of the few rows this lane owns in fp32 (deterministic order); the
  // warp, CTA and grid reductions are fp64
  float acc[kLossSlots] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t ntiles = (a.c.rows + kTile - 1) / kTile;
  const int64_t gw = int64_t(blockIdx.x) * kFlowWarps + warp, nw = int64_t(gridDim.x) * kFlowWarps;
  for (int64_t tile = gw; tile < ntiles; tile += nw) {
    const int64_t r0 = tile * kTile;
    const int nt = int(a.c.rows - r0 < kTile ? a.c.rows - r0 : kTile);
    const int64_t r = r0 + lane;  // the row whose epilogue this lane runs (lane < nt)
    // epilogue inputs first: their (coalesced) loads overlap pass 1
    RowMeta4 mt;
    float gin = 0.f;
    if (lane < nt) {
      if (MODE == 1) {
        mt.lpb = a.f.logp_behav[r];
        mt.lpp = a.f.logp_prox ? a.f.logp_prox[r] : 0.f;
        mt.lref = pc.has_ref ? a.f.logp_ref[r] : 0.f;
        mt.adv = a.f.adv[r];
        mt.ver = a.f.version[r];
        mt.valid = a.f.slot_key[r] != 0ull;
      } else if (MODE == 2) {
        gin = a.grad_logp[r];
      }
    }
    float g = 0.f, c = 0.f;
    if (MODE != 2) {
#pragma unroll 2
      for (int t = 0; t < nt; ++t) {  // pass 1: lane partials of each row -> SMEM
        float q, ls;
        row_partials<T, VEC, NQ>(mu0, x0, ls0, s_isig, (r0 + t) * n, n, learned, lane, q, ls);
        pq[t * kPad + lane] = q;
        if (learned) pl[t * kPad + lane] = ls;
      }
      __syncwarp();
      if (lane < nt) {
        double qd = 0.0, ld = 0.0;
        for (int l = 0; l < 32; ++l) {  // fixed order, fp64
          qd += double(pq[lane * kPad + l]);
          if (learned) ld += double(pl[lane * kPad + l]);
        }
        const double lnsig = learned ? ld : s_lnsig;
        const float logp = float(-0.5 * qd - lnsig - cst);
        const float H = float(lnsig + cst + 0.5 * double(n));
        PpoRowIn in;
        in.tgt_status = isfinite(logp) ? 0 : 3;
        in.logp = logp;
        in.H = H;
        RowStats rs;
        float lt = 0.f;
        if (MODE == 1) {
          in.lpb = mt.lpb;
          in.lpp = mt.lpp;
          in.lref = mt.lref;
          in.adv = mt.adv;
          in.ver = mt.ver;
          in.valid = mt.valid;
          PpoMid t;
          g = ppo_grad(pc, in, t);
          c = t.m ? pc.ent_coef * pc.invN : 0.f;
          ppo_stats(pc, in, t, rs, &lt);
          if (a.f.out_grad_logp) a.f.out_grad_logp[r] = g;
          if (a.f.out_loss_tok) a.f.out_loss_tok[r] = lt;
        } else {
          fwd_row_stats(in, rs);
        }
        if (a.logp) a.logp[r] = logp;
        if (want_stats) acc_stats_f(acc, rs);
      }
      __syncwarp();  // the partials are read before the next tile overwrites them
    } else {
      g = gin;
    }
    if (MODE != 0 && (a.dmu != nullptr || a.dlog_std != nullptr)) {
#pragma unroll 2
      for (int t = 0; t < nt; ++t) {  // pass 2 (the rows were just read: L1/L2 hits)
        const float gt = __shfl_sync(0xffffffffu, g, t);
        const float ct = __shfl_sync(0xffffffffu, c, t);
        row_backward<T, VEC, NQ>(mu0, x0, ls0, dmu0, dls0, s_isig, (r0 + t) * n, n, learned, lane, gt, ct);
      }
    }
  }
  if (!want_stats) return;
  __shared__ double red[kFlowWarps][kLossSlots];
  __shared__ double cta[kLossSlots];
  double accd[kLossSlots];
  for (int k = 0; k < kLossSlots; ++k) accd[k] = warp_sum_d(double(acc[k]));
  if (lane == 0)
    for (int k = 0; k < kLossSlots; ++k) red[warp][k] = accd[k];
  __syncthreads();
  if (threadIdx.x < kLossSlots) {
    double sm = 0;
    for (int w = 0; w < kFlowWarps; ++w) sm += red[w][threadIdx.x];
    cta[threadIdx.x] = sm;
  }
  __syncthreads();
  finish_loss_stats(cta, a.stats, a.ws.partials, a.ws.ctrl + CTRL_FLOW, Nden,
                    MODE == 1 ? a.f.accumulate : 0, MODE == 1 ? a.f.ent_coef : 0.f, &a.ws.p2p);
}

size_t flow_smem(int n) { return size_t((n + 3) & ~3) * 4 + size_t(kFlowWarps) * 2 * kTile * kPad * 4; }

// grid = all resident CTAs (occupancy of the instantiation), fewer for small problems
template <typename T, int MODE, bool VEC, int NQ>
cudaError_t launch_m(const FlowArgs& a, cudaStream_t s) {
  const int n = a.c.n_steps * a.c.dim;
  const size_t smem = flow_smem(n);
  static size_t attr[kMaxDevices] = {};  // the SMEM opt-in is a per-device attribute
  const int dev = device_info().device;
  size_t dummy = 0;
  size_t& cached = (dev >= 0 && dev < kMaxDevices) ? attr[dev] : dummy;
  if (smem > 48 * 1024 && cached < smem) {
    cudaError_t e = cudaFuncSetAttribute(flow_kernel<T, MODE, VEC, NQ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    cached = smem;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, flow_kernel<T, MODE, VEC, NQ>,
                                                                kFlowWarps * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t tiles = (a.c.rows + kTile - 1) / kTile;
  int64_t grid = (tiles + kFlowWarps - 1) / kFlowWarps;
  const int64_t cap = int64_t(device_info().sm_count) * per_sm;
  if (grid > cap) grid = cap;
  flow_kernel<T, MODE, VEC, NQ><<<int(grid), kFlowWarps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename T, bool VEC, int NQ>
cudaError_t launch_q(const FlowArgs& a, cudaStream_t s) {
  if (a.grad_logp) return launch_m<T, 2, VEC, NQ>(a, s);
  if (a.fused) return launch_m<T, 1, VEC, NQ>(a, s);
  return launch_m<T, 0, VEC, NQ>(a, s);
}

// the paper's shapes (Table 2: K = 4 denoising steps, chunk 10 or 5 x 7 DoF) get a compile-time
// row length; every other 4-aligned shape the runtime one
template <typename T, bool VEC>
cudaError_t launch_v(const FlowArgs& a, cudaStream_t s) {
  const int n = a.c.n_steps * a.c.dim;
  if (VEC && n == 280) return launch_q<T, VEC, 70>(a, s);
  if (VEC && n == 140) return launch_q<T, VEC, 35>(a, s);
  return launch_q<T, VEC, 0>(a, s);
}

template <typename T>
cudaError_t launch_t(const FlowArgs& a, cudaStream_t s) {
  const int n = a.c.n_steps * a.c.dim;
  const size_t eb = sizeof(T);
  const bool aligned = reinterpret_cast<uintptr_t>(a.c.mu) % (4 * eb) == 0 &&
                       reinterpret_cast<uintptr_t>(a.c.x) % 16 == 0 &&
                       (!a.c.log_std || reinterpret_cast<uintptr_t>(a.c.log_std) % 16 == 0) &&
                       (!a.dmu || reinterpret_cast<uintptr_t>(a.dmu) % (4 * eb) == 0) &&
                       (!a.dlog_std || reinterpret_cast<uintptr_t>(a.dlog_std) % 16 == 0);
  const bool vec = n % 4 == 0 && aligned;
  return vec ? launch_v<T, true>(a, s) : launch_v<T, false>(a, s);
}

}  // namespace

cudaError_t launch_flow(const FlowArgs& a, cudaStream_t s) {
  if (a.c.rows <= 0) return cudaSuccess;
  return a.c.mu_dtype == RLVLA_BF16 ? launch_t<__nv_bfloat16>(a, s) : launch_t<float>(a, s);
}

}  // namespace rlvla
