// flow.cu — NEXT-4: log-likelihood of a flow / diffusion policy's action chunk as a chain of
// K Gaussian denoising transitions (reading R25; pi_0 / pi_0.5 / GR00T, P:39, P:77, P:99,
// Table 2 "Model Num Step" = 4), optionally fused with the PPO epilogue and its backward.
//
// Warp tiles of kTile = 4 decision steps:
//   pass 1  step by step, the row's n = K*D elements are read with 4-wide loads (mu in f32 or
//           bf16, x, optional ln sigma; a sigma schedule is a per-element 1/sigma table in
//           SMEM, so there is no division) and packed fp32x2 math; each lane keeps its partial
//           sums of z^2 (and ln sigma) of the four steps in registers
//   epilogue a fixed fp64 butterfly (row_totals4) leaves step t's totals at lane t, which forms
//           logp = -0.5 sum z^2 - sum ln sigma - n ln(2 pi)/2 and
//           H = sum ln sigma + n (ln 2 pi + 1)/2, and runs the shared PPO epilogue
//           (epilogue.cuh) — the per-step scalar work spread over the lanes
//   pass 2  step by step, g and c are broadcast and the backward writes
//           dmu = g (z / sigma),   dln sigma = g (z^2 - 1) - c     (c = ent_coef m / N)
// Two kernels run this tile: flow_tma_kernel for the paper's K x D shapes (280, 140 elements;
// each warp's tiles staged HBM -> SMEM by bulk copies one or two tiles ahead, pass 1 leaving
// z / sigma in place for pass 2) and flow_kernel for any other shape (direct loads; rows whose
// length is not a multiple of 4, or unaligned pointers, take scalar loops).
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


constexpr int kTile = 4;  // decision steps per warp tile: lane t < 4 runs step t's epilogue

// a row's PPO inputs as loaded: kept raw (the key is not compared yet) so that no
// instruction consumes a load before pass 1 has run — the loads' latency hides behind it
struct RowMeta4 {
  float lpb = 0.f, lpp = 0.f, lref = 0.f, adv = 0.f;
  int ver = 0;
  unsigned long long key = 1ull;
};

// The four rows' totals of the lanes' fp32 partials, in fp64: a butterfly reduce-scatter
// (xor 16 halves the rows each lane carries, xor 8 halves them again, xor 4/2/1 finish row
// (lane >> 3) & 3), then lane t < 4 fetches row t. A fixed tree: the bits do not depend on
// timing or on which warp runs the tile.
__device__ __forceinline__ double row_totals4(const float (&v)[kTile], int lane) {
  const bool h = lane & 16, b = lane & 8;
  const double d0 = v[0], d1 = v[1], d2 = v[2], d3 = v[3];
  const double e0 = (h ? d2 : d0) + __shfl_xor_sync(0xffffffffu, h ? d0 : d2, 16);
  const double e1 = (h ? d3 : d1) + __shfl_xor_sync(0xffffffffu, h ? d1 : d3, 16);
  double f = (b ? e1 : e0) + __shfl_xor_sync(0xffffffffu, b ? e0 : e1, 8);
  f += __shfl_xor_sync(0xffffffffu, f, 4);
  f += __shfl_xor_sync(0xffffffffu, f, 2);
  f += __shfl_xor_sync(0xffffffffu, f, 1);
  return __shfl_sync(0xffffffffu, f, (lane & 3) * 8);
}

// One row's lane partials: q = sum z^2 and ls = sum ln sigma (learned) over the lane's
// elements, z = (x - mu) / sigma. Row pointers are formed once, indices stay 32-bit.
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
        const float2 ia = make_float2(iv.x, iv.y), ib = make_float2(iv.z, iv.w);
        const float2 za = __fmul2_rn(__fadd2_rn(make_float2(xv.x, xv.y), make_float2(-m.x, -m.y)), ia);
        const float2 zb = __fmul2_rn(__fadd2_rn(make_float2(xv.z, xv.w), make_float2(-m.z, -m.w)), ib);
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

// dmu = g (z / sigma), dln sigma = g (z^2 - 1) - c for one row (exact zeros when g = c = 0);
// the row is read at `base` of mu0 / x0 / ls0 (global memory or a staged SMEM tile) and
// written at `dbase` of dmu0 / dls0
template <typename T, bool VEC, int NQ>
__device__ __forceinline__ void row_backward(const T* mu0, const float* x0, const float* ls0, T* dmu0,
                                             float* dls0, const float* s_isig, int64_t base,
                                             int64_t dbase, int n, bool learned, int lane, float g,
                                             float c) {
  const bool active = g != 0.f || c != 0.f;
  const T* mu = mu0 + base;
  const float* x = x0 + base;
  const float* lsd = learned ? ls0 + base : nullptr;
  T* dmu = dmu0 ? dmu0 + dbase : nullptr;
  float* dls = dls0 ? dls0 + dbase : nullptr;
  if (VEC) {
    constexpr int kIters = NQ > 0 ? (NQ + 31) / 32 : 1;
    const int nq = NQ > 0 ? NQ : (n >> 2);
    const float2 g2 = make_float2(g, g);
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
        const float2 wa = __fmul2_rn(za, ia), wb = __fmul2_rn(zb, ib);
        const float2 da = __fmul2_rn(g2, wa), db = __fmul2_rn(g2, wb);
        dm = make_float4(da.x, da.y, db.x, db.y);
        if (dls)
          dl = make_float4(fmaf(g, fmaf(za.x, za.x, -1.f), -c), fmaf(g, fmaf(za.y, za.y, -1.f), -c),
                           fmaf(g, fmaf(zb.x, zb.x, -1.f), -c), fmaf(g, fmaf(zb.y, zb.y, -1.f), -c));
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
      if (dmu) st_mu<T>(dmu, j, active ? g * (zz * iv) : 0.f);
      if (dls) dls[j] = active ? fmaf(g, fmaf(zz, zz, -1.f), -c) : 0.f;
    }
  }
}

// Per-CTA constants of one launch (the sigma schedule's 1/sigma table lives in SMEM)
struct FlowCtx {
  PpoConst pc;
  double Nden, cst, lnsig;
  const float* s_isig;
  int n;
  bool learned, want_stats;
};

template <int MODE>
__device__ __forceinline__ FlowCtx flow_setup(const FlowArgs& a, int n, float* s_isig, int table,
                                              double* s_lnsig) {
  FlowCtx x{};
  const int K = a.c.n_steps, D = a.c.dim;
  x.n = n;
  x.learned = a.c.log_std != nullptr;
  x.want_stats = a.stats != nullptr && MODE != 2;
  x.s_isig = s_isig;
  // sigma schedule: 1/sigma per element of `table` = n (a row) or 4n (a tile's rows) — no
  // division or k = j / D in the loops — and D sum_k ln sigma_k in fp64, once per CTA
  if (!x.learned) {
    for (int j = threadIdx.x; j < table; j += blockDim.x) s_isig[j] = 1.f / a.c.sigma_k[(j % n) / D];
    if (threadIdx.x == 0) {
      double acc = 0.0;
      for (int k = 0; k < K; ++k) acc += log(double(a.c.sigma_k[k]));
      *s_lnsig = acc * double(D);
    }
  }
  x.cst = 0.5 * 1.8378770664093453 * double(n);  // n ln(2 pi) / 2
  if (MODE == 1) {
    PpoConst& pc = x.pc;
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
    x.Nden = loss_denominator(a.f.tok_denominator, a.f.adv_stats);
    pc.invN = x.Nden > 0.0 ? float(1.0 / x.Nden) : 0.f;
  }
  return x;
}

// MODE 0: forward only, 1: fused PPO, 2: external backward (grad_logp given).
// A warp tile is rows r0 .. r0+nt-1 (nt <= 4). Its PPO inputs are loaded first (coalesced, one
// row per lane; no branch: lanes >= nt re-load row r0, so that no reconvergence point forces the
// loads to complete before pass 1 has run)
template <int MODE>
__device__ __forceinline__ RowMeta4 load_meta(const FlowArgs& a, const FlowCtx& x, int64_t r0,
                                              int nt, int lane, float& gin) {
  const int64_t rl = lane < nt ? r0 + lane : r0;
  RowMeta4 mt;
  gin = 0.f;
  if (MODE == 1) {
    mt.lpb = a.f.logp_behav[rl];
    mt.lpp = a.f.logp_prox ? a.f.logp_prox[rl] : 0.f;
    mt.lref = x.pc.has_ref ? a.f.logp_ref[rl] : 0.f;
    mt.adv = a.f.adv[rl];
    mt.ver = a.f.version[rl];
    mt.key = a.f.slot_key[rl];
  } else if (MODE == 2) {
    gin = a.grad_logp[rl];
  }
  return mt;
}

// Epilogue: lane t < nt owns row t, whose fp64 totals row_totals4 left there: logp / H and the
// PPO epilogue — the per-row scalar work spread over the lanes instead of repeated by all 32.
// Returns the row's g = dL/dlogp and c (entropy term); acc: the lane's fp32 statistics.
template <int MODE>
__device__ __forceinline__ void tile_epilogue(const FlowArgs& a, const FlowCtx& x, const RowMeta4& mt,
                                              double qd, double ld, int n, int64_t r0, int nt,
                                              int lane, float* acc, float& g, float& c) {
  g = c = 0.f;
  if (lane >= nt) return;
  const int64_t r = r0 + lane;
  const double lnsig = x.learned ? ld : x.lnsig;
  const float logp = float(-0.5 * qd - lnsig - x.cst);
  const float H = float(lnsig + x.cst + 0.5 * double(n));
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
    in.valid = mt.key != 0ull;
    PpoMid t;
    g = ppo_grad(x.pc, in, t);
    c = t.m ? x.pc.ent_coef * x.pc.invN : 0.f;
    ppo_stats(x.pc, in, t, rs, &lt);
    if (a.f.out_grad_logp) a.f.out_grad_logp[r] = g;
    if (a.f.out_loss_tok) a.f.out_loss_tok[r] = lt;
  } else {
    fwd_row_stats(in, rs);
  }
  if (a.logp) a.logp[r] = logp;
  if (x.want_stats) acc_stats_f(acc, rs);
}

// Row-by-row tile (any shape): read at element offset `sbase` of mu_s / x_s / ls_s (the global
// arrays, or a staged SMEM copy of the tile at sbase 0), written at the rows' global offsets.
// Pass 1: coalesced element-parallel loads, the lane partials of all four rows in registers.
// Pass 2: g and c are broadcast row by row and the backward re-reads the row.
// VEC: 4-wide vector loads (n % 4 == 0, aligned pointers); otherwise scalar loops.
template <typename T, int MODE, bool VEC, int NQ>
__device__ __forceinline__ void flow_tile(const FlowArgs& a, const FlowCtx& x, const T* mu_s,
                                          const float* x_s, const float* ls_s, int64_t sbase,
                                          int64_t r0, int nt, float* acc, int lane) {
  const int n = NQ > 0 ? 4 * NQ : x.n;
  const bool learned = x.learned;
  float gin;
  const RowMeta4 mt = load_meta<MODE>(a, x, r0, nt, lane, gin);
  float g = gin, c = 0.f;
  if (MODE != 2) {
    float q[kTile], l[kTile];
#pragma unroll
    for (int t = 0; t < kTile; ++t) {  // pass 1: each lane's partials of the four rows
      q[t] = l[t] = 0.f;
      if (t < nt)
        row_partials<T, VEC, NQ>(mu_s, x_s, ls_s, x.s_isig, sbase + int64_t(t) * n, n, learned, lane,
                                 q[t], l[t]);
    }
    const double qd = row_totals4(q, lane);
    const double ld = learned ? row_totals4(l, lane) : 0.0;
    tile_epilogue<MODE>(a, x, mt, qd, ld, n, r0, nt, lane, acc, g, c);
  }
  if (MODE != 0 && (a.dmu != nullptr || a.dlog_std != nullptr)) {
#pragma unroll 2
    for (int t = 0; t < nt; ++t) {  // pass 2 (the rows were just read: SMEM, L1 or L2)
      const float gt = __shfl_sync(0xffffffffu, g, t);
      const float ct = __shfl_sync(0xffffffffu, c, t);
      row_backward<T, VEC, NQ>(mu_s, x_s, ls_s, static_cast<T*>(a.dmu), a.dlog_std, x.s_isig,
                               sbase + int64_t(t) * n, (r0 + t) * n, n, learned, lane, gt, ct);
    }
  }
}

// Flat tile (a full, staged tile of the paper's shapes; MODE 0 or 1): the tile's four rows are
// contiguous in the stage and in dmu / dln sigma, so both passes walk its kTile NQ quads
// lane-strided as one array — no per-row loop tails. A 32-quad step spans at most two rows
// (NQ >= 32), so the row of a quad is a compile-time constant or one compare. Pass 1 leaves what
// the backward needs in place of x (and ln sigma): w = z / sigma for a sigma schedule, z and
// 1/sigma when learned (each lane rewrites only the quads it read), so pass 2 is a load, a
// multiply and a store per element. s_isig holds the tile's 4n elements; mt: the tile's PPO
// inputs, loaded by the caller a tile ahead (their latency under a saturated HBM exceeds a pass).
template <typename T, int MODE, int NQ, bool LEARNED>
__device__ __forceinline__ void flow_tile_flat(const FlowArgs& a, const FlowCtx& x, const T* mu_s,
                                               float* x_s, float* ls_s, int64_t r0,
                                               const RowMeta4& mt, float* acc, int lane) {
  static_assert(NQ >= 32 && MODE != 2, "flat tiles: rows of >= 128 elements, a pass 1");
  constexpr int n = 4 * NQ, kQ = kTile * NQ, kIt = (kQ + 31) / 32;
  float2 q2[kTile];
  float l[kTile];
#pragma unroll
  for (int t = 0; t < kTile; ++t) {
    q2[t] = make_float2(0.f, 0.f);
    l[t] = 0.f;
  }
#pragma unroll
  for (int i = 0; i < kIt; ++i) {  // pass 1
    const int qd = lane + 32 * i;
    if ((i + 1) * 32 <= kQ || qd < kQ) {
      const int j = 4 * qd;
      const float4 m = ld_mu4<T>(mu_s, j);
      const float4 xv = *reinterpret_cast<const float4*>(x_s + j);
      float4 iv;
      if (LEARNED) {
        const float4 lv = *reinterpret_cast<const float4*>(ls_s + j);
        iv = make_float4(__expf(-lv.x), __expf(-lv.y), __expf(-lv.z), __expf(-lv.w));
        const float ls = (lv.x + lv.y) + (lv.z + lv.w);
        const int lo = (32 * i) / NQ, hi = (32 * i + 31) / NQ < kTile ? (32 * i + 31) / NQ : kTile - 1;
        if (lo == hi) {
          l[lo] += ls;
        } else {
          const bool up = qd >= hi * NQ;
          l[lo] += up ? 0.f : ls;
          l[hi] += up ? ls : 0.f;
        }
      } else {
        iv = *reinterpret_cast<const float4*>(x.s_isig + j);
      }
      const float2 ia = make_float2(iv.x, iv.y), ib = make_float2(iv.z, iv.w);
      const float2 za = __fmul2_rn(__fadd2_rn(make_float2(xv.x, xv.y), make_float2(-m.x, -m.y)), ia);
      const float2 zb = __fmul2_rn(__fadd2_rn(make_float2(xv.z, xv.w), make_float2(-m.z, -m.w)), ib);
      const int lo = (32 * i) / NQ, hi = (32 * i + 31) / NQ < kTile ? (32 * i + 31) / NQ : kTile - 1;
      if (lo == hi) {
        q2[lo] = __ffma2_rn(za, za, __ffma2_rn(zb, zb, q2[lo]));
      } else {
        const bool up = qd >= hi * NQ;
        const float2 sl = __ffma2_rn(za, za, __ffma2_rn(zb, zb, q2[lo]));
        const float2 sh = __ffma2_rn(za, za, __ffma2_rn(zb, zb, q2[hi]));
        q2[lo] = up ? q2[lo] : sl;
        q2[hi] = up ? sh : q2[hi];
      }
      if (MODE == 1) {
        if (LEARNED) {
          *reinterpret_cast<float4*>(x_s + j) = make_float4(za.x, za.y, zb.x, zb.y);
          *reinterpret_cast<float4*>(ls_s + j) = iv;
        } else {
          const float2 wa = __fmul2_rn(za, ia), wb = __fmul2_rn(zb, ib);
          *reinterpret_cast<float4*>(x_s + j) = make_float4(wa.x, wa.y, wb.x, wb.y);
        }
      }
    }
  }
  float q[kTile];
#pragma unroll
  for (int t = 0; t < kTile; ++t) q[t] = q2[t].x + q2[t].y;
  const double qd = row_totals4(q, lane);
  const double ld = LEARNED ? row_totals4(l, lane) : 0.0;
  float g, c;
  tile_epilogue<MODE>(a, x, mt, qd, ld, n, r0, kTile, lane, acc, g, c);
  if (MODE == 0 || (a.dmu == nullptr && a.dlog_std == nullptr)) return;
  __syncwarp();
  float gt[kTile], ct[kTile];
  bool all_active = true;
#pragma unroll
  for (int t = 0; t < kTile; ++t) {
    gt[t] = __shfl_sync(0xffffffffu, g, t);
    ct[t] = LEARNED ? __shfl_sync(0xffffffffu, c, t) : 0.f;
    all_active = all_active && (gt[t] != 0.f || ct[t] != 0.f);
  }
  T* const dmu = a.dmu ? static_cast<T*>(a.dmu) + r0 * n : nullptr;
  float* const dls = LEARNED && a.dlog_std ? a.dlog_std + r0 * n : nullptr;
#pragma unroll
  for (int i = 0; i < kIt; ++i) {  // pass 2
    const int qd = lane + 32 * i;
    if ((i + 1) * 32 <= kQ || qd < kQ) {
      const int j = 4 * qd;
      const int lo = (32 * i) / NQ, hi = (32 * i + 31) / NQ < kTile ? (32 * i + 31) / NQ : kTile - 1;
      const bool up = lo != hi && qd >= hi * NQ;
      const float gq = up ? gt[hi] : gt[lo];
      const float cq = up ? ct[hi] : ct[lo];
      const float2 g2 = make_float2(gq, gq);
      float4 dm, dl = make_float4(0.f, 0.f, 0.f, 0.f);
      if (LEARNED) {
        const float4 z = *reinterpret_cast<const float4*>(x_s + j);
        const float4 iv = *reinterpret_cast<const float4*>(ls_s + j);
        const float2 da = __fmul2_rn(g2, __fmul2_rn(make_float2(z.x, z.y), make_float2(iv.x, iv.y)));
        const float2 db = __fmul2_rn(g2, __fmul2_rn(make_float2(z.z, z.w), make_float2(iv.z, iv.w)));
        dm = make_float4(da.x, da.y, db.x, db.y);
        dl = make_float4(fmaf(gq, fmaf(z.x, z.x, -1.f), -cq), fmaf(gq, fmaf(z.y, z.y, -1.f), -cq),
                         fmaf(gq, fmaf(z.z, z.z, -1.f), -cq), fmaf(gq, fmaf(z.w, z.w, -1.f), -cq));
      } else {
        const float4 w = *reinterpret_cast<const float4*>(x_s + j);
        const float2 da = __fmul2_rn(g2, make_float2(w.x, w.y));
        const float2 db = __fmul2_rn(g2, make_float2(w.z, w.w));
        dm = make_float4(da.x, da.y, db.x, db.y);
      }
      if (!all_active && gq == 0.f && cq == 0.f) {  // masked row: exact zeros
        dm = make_float4(0.f, 0.f, 0.f, 0.f);
        dl = dm;
      }
      if (dmu) st_mu4<T>(dmu, j, dm);
      if (dls) *reinterpret_cast<float4*>(dls + j) = dl;
    }
  }
}

// The CTA's statistics: warp sums in fp64, then the warps in fixed order, then the grid
template <int MODE, int WARPS>
__device__ __forceinline__ void flow_finish(const FlowArgs& a, const FlowCtx& x, const float* acc,
                                            int warp, int lane) {
  __shared__ double red[WARPS][kLossSlots];
  __shared__ double cta[kLossSlots];
  double accd[kLossSlots];
  for (int k = 0; k < kLossSlots; ++k) accd[k] = warp_sum_d(double(acc[k]));
  if (lane == 0)
    for (int k = 0; k < kLossSlots; ++k) red[warp][k] = accd[k];
  __syncthreads();
  if (threadIdx.x < kLossSlots) {
    double sm = 0;
    for (int w = 0; w < WARPS; ++w) sm += red[w][threadIdx.x];
    cta[threadIdx.x] = sm;
  }
  __syncthreads();
  finish_loss_stats(cta, a.stats, a.ws.partials, a.ws.ctrl + CTRL_FLOW, x.Nden,
                    MODE == 1 ? a.f.accumulate : 0, MODE == 1 ? a.f.ent_coef : 0.f, &a.ws.p2p);
}

#ifndef RLVLA_FLOW_LOADPOL
#define RLVLA_FLOW_LOADPOL 0  // TMA tile loads: 0 L2 evict_first, 1 evict_normal
#endif
#ifndef RLVLA_FLOW_MINB
#define RLVLA_FLOW_MINB 4  // resident CTAs per SM the register budget is sized for
#endif
// Direct-load kernel: any row length, rows streamed straight from global memory.
template <typename T, int MODE, bool VEC, int NQ>
__global__ void __launch_bounds__(kFlowWarps * 32, RLVLA_FLOW_MINB) flow_kernel(FlowArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = NQ > 0 ? 4 * NQ : a.c.n_steps * a.c.dim;
  extern __shared__ __align__(16) float dsm[];  // [n] 1/sigma (sigma schedule)
  __shared__ double s_lnsig;
  FlowCtx x = flow_setup<MODE>(a, n, dsm, n, &s_lnsig);
  __syncthreads();
  x.lnsig = s_lnsig;
  // per-lane statistics of the few rows this lane owns in fp32 (deterministic order); the
  // warp, CTA and grid reductions are fp64
  float acc[kLossSlots] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t ntiles = (a.c.rows + kTile - 1) / kTile;
  const int64_t gw = int64_t(blockIdx.x) * kFlowWarps + warp, nw = int64_t(gridDim.x) * kFlowWarps;
  for (int64_t tile = gw; tile < ntiles; tile += nw) {
    const int64_t r0 = tile * kTile;
    const int nt = int(a.c.rows - r0 < kTile ? a.c.rows - r0 : kTile);
    flow_tile<T, MODE, VEC, NQ>(a, x, static_cast<const T*>(a.c.mu), a.c.x, a.c.log_std, r0 * n, r0,
                                nt, acc, lane);
  }
  if (!x.want_stats) return;
  flow_finish<MODE, kFlowWarps>(a, x, acc, warp, lane);
}

// TMA-staged kernel for the paper's compile-time row lengths (NQ > 0, 16-byte aligned arrays):
// every warp runs its own ring of STAGES tile buffers in SMEM, filled by 1-D bulk copies
// (one per array per tile, mbarrier tx completion, L2 evict_first) that lane 0 issues
// STAGES tiles ahead, so the HBM reads of the next tiles are in flight while the warp
// computes on the current one; flow_tile_flat then works on the stage (MODE 2, which has no
// pass 1, takes the row-by-row tile on it). The last, partial tile (rows % 4) is read directly
// by the one warp that owns it.
// CTA shapes (warps, ring stages per warp): 8 x 2 with a sigma schedule (2 CTAs per SM fit),
// 4 x 2 with learned ln sigma (stages twice the size: 2 CTAs of 4 measured faster than 1 of 8),
// and 16 x 1 for a sigma schedule with fewer than ~4 tiles per warp of the 8 x 2 grid (one
// update of 24,576 steps: more, shallower warps finish the few tiles sooner) —
// profiles/r1/FLOW.md
#ifndef RLVLA_FLOW_16W_MINB
#define RLVLA_FLOW_16W_MINB 0  // 1: cap the 16-warp shape at 64 registers (2 CTAs per SM; A/B: spills, slower)
#endif
#ifndef RLVLA_FLOW_L2_LEAD
#define RLVLA_FLOW_L2_LEAD 0  // 1: L2 prefetch of the next tile beyond the SMEM ring (A/B: slower)
#endif
#ifndef RLVLA_FLOW_SMALL_WARPS
#define RLVLA_FLOW_SMALL_WARPS 16  // warps of the single-stage small-call shape (16, 12 or 8)
#endif
#ifndef RLVLA_FLOW_SMALL_TILES
#define RLVLA_FLOW_SMALL_TILES 9472  // tiles below which the 16 x 1 shape runs (0: never)
#endif

template <typename T, int NQ>
__host__ __device__ constexpr int tma_stage_bytes(bool learned) {
  return kTile * 4 * NQ * (int(sizeof(T)) + 4 + (learned ? 4 : 0));
}
// barriers, then the tile's 1/sigma table (4n floats), then the per-warp rings
template <int NQ, int WARPS, int STAGES>
__host__ __device__ constexpr int tma_ring_offset() {
  return ((8 * WARPS * STAGES + 4 * kTile * 4 * NQ) + 127) & ~127;
}

template <typename T, int MODE, int NQ, bool LEARNED, int WARPS, int STAGES>
// (RLVLA_FLOW_16W_MINB=1 holds 16-warp CTAs to 64 registers so that two fit per SM with their
// SMEM rings — ~1.3 tiles per warp instead of ~2.6 for one paper-sized update; measured slower
// from the spills it forces, so off)
__global__ void __launch_bounds__(WARPS * 32, RLVLA_FLOW_16W_MINB && WARPS == 16 ? 2 : 1) flow_tma_kernel(FlowArgs a) {
  constexpr int kTmaWarps = WARPS, kFlowStages = STAGES;
  constexpr int n = 4 * NQ;
  constexpr int kMuB = kTile * n * int(sizeof(T)), kXB = kTile * n * 4;
  constexpr int stage_b = tma_stage_bytes<T, NQ>(LEARNED);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  extern __shared__ __align__(128) unsigned char tsm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(tsm) + warp * kFlowStages;  // [warp][stage]
  float* s_isig = reinterpret_cast<float*>(tsm + 8 * kTmaWarps * kFlowStages);
  unsigned char* ring = tsm + tma_ring_offset<NQ, kTmaWarps, kFlowStages>() + size_t(warp) * kFlowStages * stage_b;
  __shared__ double s_lnsig;
  FlowCtx x = flow_setup<MODE>(a, n, s_isig, kTile * n, &s_lnsig);
  if (lane == 0) {
    for (int st = 0; st < kFlowStages; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
  }
  __syncthreads();
  x.lnsig = s_lnsig;
  float acc[kLossSlots] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t nfull = a.c.rows / kTile;
  const int64_t gw = int64_t(blockIdx.x) * kTmaWarps + warp, nw = int64_t(gridDim.x) * kTmaWarps;
  const int64_t cnt = gw < nfull ? (nfull - gw + nw - 1) / nw : 0;  // this warp's full tiles
  const T* const mu0 = static_cast<const T*>(a.c.mu);
#if RLVLA_FLOW_LOADPOL
  const uint64_t pol = policy_evict_normal();
#else
  const uint64_t pol = policy_evict_first();
#endif
  auto issue = [&](int64_t i) {  // lane 0: tile gw + i nw -> stage i % kFlowStages
    const int64_t e0 = (gw + i * nw) * kTile * n;
    unsigned char* st = ring + (i % kFlowStages) * stage_b;
    uint64_t* bar = &bars[i % kFlowStages];
    mbar_arrive_expect_tx(bar, uint32_t(stage_b));
    bulk_g2s(st, mu0 + e0, kMuB, bar, pol);
    bulk_g2s(st + kMuB, a.c.x + e0, kXB, bar, pol);
    if (LEARNED) bulk_g2s(st + kMuB + kXB, a.c.log_std + e0, kXB, bar, pol);
  };
  // L2 lead: the tile after the ones in the SMEM ring is prefetched into L2 (bulk prefetch,
  // no SMEM), so its TMA fill — issued only once a stage frees up — is an L2 hit
  auto prefetch = [&](int64_t i) {
    const int64_t e0 = (gw + i * nw) * kTile * n;
    bulk_prefetch_l2(mu0 + e0, uint32_t(kMuB));
    bulk_prefetch_l2(a.c.x + e0, uint32_t(kXB));
    if (LEARNED) bulk_prefetch_l2(a.c.log_std + e0, uint32_t(kXB));
  };
  if (lane == 0) {
    for (int64_t i = 0; i < cnt && i < kFlowStages; ++i) issue(i);
    if (RLVLA_FLOW_L2_LEAD && kFlowStages < cnt) prefetch(kFlowStages);
  }
  float gin;
  RowMeta4 mt_next = load_meta<MODE>(a, x, gw < nfull ? gw * kTile : 0, kTile, lane, gin);
  for (int64_t i = 0; i < cnt; ++i) {
    unsigned char* st = ring + (i % kFlowStages) * stage_b;
    mbar_wait(&bars[i % kFlowStages], uint32_t((i / kFlowStages) & 1));
    const int64_t r0 = (gw + i * nw) * kTile;
    if constexpr (MODE == 2)
      flow_tile<T, MODE, true, NQ>(a, x, reinterpret_cast<const T*>(st),
                                   reinterpret_cast<const float*>(st + kMuB),
                                   reinterpret_cast<const float*>(st + kMuB + kXB), 0, r0, kTile, acc,
                                   lane);
    else {
      const RowMeta4 mt = mt_next;  // the next tile's inputs (the last tile re-loads its own)
      mt_next = load_meta<MODE>(a, x, (gw + (i + 1 < cnt ? i + 1 : i) * nw) * kTile, kTile, lane, gin);
      flow_tile_flat<T, MODE, NQ, LEARNED>(a, x, reinterpret_cast<const T*>(st),
                                           reinterpret_cast<float*>(st + kMuB),
                                           reinterpret_cast<float*>(st + kMuB + kXB), r0, mt, acc, lane);
    }
    // the stage's generic-proxy reads and rewrites are ordered before its next TMA fill
    fence_proxy_async();
    __syncwarp();
    if (lane == 0 && i + kFlowStages < cnt) {
      issue(i + kFlowStages);
      if (RLVLA_FLOW_L2_LEAD && i + kFlowStages + 1 < cnt) prefetch(i + kFlowStages + 1);
    }
  }
  const int64_t tail = a.c.rows - nfull * kTile;
  if (tail > 0 && gw == nfull % nw)
    flow_tile<T, MODE, true, NQ>(a, x, mu0, a.c.x, a.c.log_std, nfull * kTile * n, nfull * kTile,
                                 int(tail), acc, lane);
  if (!x.want_stats) return;
  flow_finish<MODE, kTmaWarps>(a, x, acc, warp, lane);
}

size_t flow_smem(int n) { return size_t((n + 3) & ~3) * 4; }

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

// TMA-staged launch: CTAs of WARPS warps, as many as fit (SMEM-bound), fewer for small
// problems
template <typename T, int MODE, int NQ, bool LEARNED, int WARPS, int STAGES>
cudaError_t launch_tma(const FlowArgs& a, cudaStream_t s) {
  constexpr int kTmaWarps = WARPS;
  const size_t smem = size_t(tma_ring_offset<NQ, WARPS, STAGES>()) +
                      size_t(WARPS) * STAGES * tma_stage_bytes<T, NQ>(LEARNED);
  static size_t attr[kMaxDevices] = {};
  const int dev = device_info().device;
  size_t dummy = 0;
  size_t& cached = (dev >= 0 && dev < kMaxDevices) ? attr[dev] : dummy;
  if (smem > 48 * 1024 && cached < smem) {
    cudaError_t e = cudaFuncSetAttribute(flow_tma_kernel<T, MODE, NQ, LEARNED, WARPS, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    // the whole unified L1/SMEM for shared memory, so that two SMEM-heavy CTAs fit per SM
    e = cudaFuncSetAttribute(flow_tma_kernel<T, MODE, NQ, LEARNED, WARPS, STAGES>,
                             cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    cached = smem;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, flow_tma_kernel<T, MODE, NQ, LEARNED, WARPS, STAGES>,
                                                                kTmaWarps * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t tiles = (a.c.rows + kTile - 1) / kTile;
  int64_t grid = (tiles + kTmaWarps - 1) / kTmaWarps;
  const int64_t cap = int64_t(persistent_sms()) * per_sm;
  if (grid > cap) grid = cap;
  flow_tma_kernel<T, MODE, NQ, LEARNED, WARPS, STAGES><<<int(grid), kTmaWarps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int NQ, bool LEARNED, int WARPS, int STAGES>
cudaError_t launch_tma_m(const FlowArgs& a, cudaStream_t s, int mode) {
  if (mode == 2) return launch_tma<T, 2, NQ, LEARNED, WARPS, STAGES>(a, s);
  if (mode == 1) return launch_tma<T, 1, NQ, LEARNED, WARPS, STAGES>(a, s);
  return launch_tma<T, 0, NQ, LEARNED, WARPS, STAGES>(a, s);
}

#ifndef RLVLA_FLOW_TMA
#define RLVLA_FLOW_TMA 1  // 0: the paper's shapes take the direct kernel too (A/B)
#endif
template <typename T, bool VEC, int NQ>
cudaError_t launch_q(const FlowArgs& a, cudaStream_t s) {
  // bulk copies need 16-byte aligned tiles: the arrays' bases (a tile is a multiple of 16 B)
  if constexpr (RLVLA_FLOW_TMA && VEC && NQ > 0) {
    if (reinterpret_cast<uintptr_t>(a.c.mu) % 16 == 0 && reinterpret_cast<uintptr_t>(a.c.x) % 16 == 0 &&
        (!a.c.log_std || reinterpret_cast<uintptr_t>(a.c.log_std) % 16 == 0)) {
      const int mode = a.grad_logp ? 2 : a.fused ? 1 : 0;
      if (a.c.log_std != nullptr) return launch_tma_m<T, NQ, true, 4, 2>(a, s, mode);
      if ((a.c.rows + kTile - 1) / kTile < RLVLA_FLOW_SMALL_TILES)
        return launch_tma_m<T, NQ, false, RLVLA_FLOW_SMALL_WARPS, 1>(a, s, mode);
      return launch_tma_m<T, NQ, false, 8, 2>(a, s, mode);
    }
  }
  if (a.grad_logp) return launch_m<T, 2, VEC, NQ>(a, s);
  if (a.fused) return launch_m<T, 1, VEC, NQ>(a, s);
  return launch_m<T, 0, VEC, NQ>(a, s);
}

// the paper's shapes (Table 2: K = 4 denoising steps, chunk 10 or 5 x 7 DoF) get a compile-time
// row length; every other 4-aligned shape the runtime one
template <typename T, bool VEC>
cudaError_t launch_v(const FlowArgs& a, cudaStream_t s) {
  const int n = a.c.n_steps * a.c.dim;
  if constexpr (VEC) {
    if (n == 280) return launch_q<T, VEC, 70>(a, s);
    if (n == 140) return launch_q<T, VEC, 35>(a, s);
  }
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
