// logprob.cu — S3 (+S4): action-token log-softmax + gather, forward and backward, fused
// with the PPO epilogue. The dominant kernel of the path: >= 99.98% of its HBM bytes are
// one read of the logits and one write of dlogits.
//
// Definition (P:39 action tokens; textbook log-softmax, reading R3-R5):
//   lse = m + ln sum_j e^{x_j - m}, logp = x_a - lse, H = lse - sum_j p_j x_j,
//   dx_j = g (1[j=a] - p_j) [+ c p_j (log p_j + H) with the entropy bonus, c = m beta_H/N].
//
// Three kernels, one per size class:
//   lp_tma_kernel     bf16, 2048 < V <= 32768 (OpenVLA 32000 vocab). Persistent, one CTA
//                     per SM, two independent 512-thread row groups; rows staged HBM ->
//                     SMEM by TMA bulk copies in a 3-stage ring (details at the kernel).
//   lp_warp_kernel    V <= 2048 (e.g. the 256-bin tiny config): one warp per row,
//                     register-resident row via 128-bit loads.
//   lp_generic_kernel any V / alignment / dtype: one CTA per row, three passes.
#include "epilogue.cuh"

namespace rlvla {
namespace {

enum { MODE_FWD = 0, MODE_FUSED = 1, MODE_BWD = 2 };

// (Measured and rejected: a NaN-guarded per-vector redo instead of the per-element -inf
// clamp in the entropy partial — 4% slower, the per-vector branch costs more than it saves.)
// build-time switches for A/B timing (tools/ab_variants.py); defaults are the product
#ifndef RLVLA_TGT_INLOOP
#define RLVLA_TGT_INLOOP 0  // 1: the target dlogit merged into its vector inside pass C
#endif
#ifndef RLVLA_L2_PREFETCH
#define RLVLA_L2_PREFETCH 0  // 1: L2 prefetch of the row a stage is refilled with, a row ahead (A/B: slower)
#endif
#ifndef RLVLA_ISSUED_SLEEP_NS
#define RLVLA_ISSUED_SLEEP_NS 64  // back-off of the stage-issue poll (0: spin)
#endif
#ifndef RLVLA_FUSED_NEGINF
#define RLVLA_FUSED_NEGINF 1  // 0: the fused kernel skips the target inside the pass-B loop
#endif
#ifndef RLVLA_PASSC_BF16
#define RLVLA_PASSC_BF16 1  // 0: pass C in fp32 (unpack, FMUL2, pack) instead of bf16 HFMA2
#endif
#ifndef RLVLA_RING_ONLY
#define RLVLA_RING_ONLY 0  // 1: diagnostic, TMA ring + stores only (results wrong; A/B ceiling)
#endif
#ifndef RLVLA_TMA_STG
#define RLVLA_TMA_STG 1  // dlogits stores of the TMA kernel: 0 st.global.cs, 1 st.global (wb), 2 st.global.L1::no_allocate
#endif
#ifndef RLVLA_TMA_LOADPOL
#define RLVLA_TMA_LOADPOL 1  // TMA row loads: 0 L2 evict_first, 1 evict_normal, 2 no hint, 3 evict_last, 4 evict_unchanged
#endif
#ifndef RLVLA_ROW_LOADPOL
#define RLVLA_ROW_LOADPOL 0  // row kernel's last-use loads: 0 L2 evict_first, 1 evict_normal
#endif
#ifndef RLVLA_TMA_SPLIT
#define RLVLA_TMA_SPLIT 1  // bulk copies per row (A/B)
#endif
#ifndef RLVLA_DX_BULK
#define RLVLA_DX_BULK 0  // 1: pass C writes dlogits into the stage, one TMA bulk store per row
#endif
#ifndef RLVLA_NFULL_FUSED
#define RLVLA_NFULL_FUSED 1  // 0: every vector of the fused kernel bounds-checked
#endif

constexpr uint32_t kNegClampPair = 0xF180F180u;  // bf16x2 (-2^100, -2^100)

__device__ __forceinline__ void stg_dx(uint4* p, uint4 v) {
#if RLVLA_TMA_STG == 1
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
#elif RLVLA_TMA_STG == 2
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
#else
  stg_stream(p, v);
#endif
}

// -inf -> -1e30, NaN kept (a comparison with NaN is false)
__device__ __forceinline__ float clamp_ninf(float t) { return t < -1e30f ? -1e30f : t; }

struct Lp {
  const void* x;
  int64_t rows;
  int V;
  int64_t ld;
  const int32_t* target;
  float* logp;
  float* lse_out;
  const float* lse_in;
  const float* g_in;
  void* dx;
  // fused PPO
  const float* lpb;
  const float* lpp;
  const float* lref;
  const float* adv;
  const int32_t* ver;
  const uint64_t* key;
  int A;
  PpoConst pc;
  double N;                  // > 0: explicit N; else read adv_stats[N_TOK] on the device
  const double* adv_stats;
  float* out_g;
  float* out_L;
  int accumulate;
  // stats
  double* stats;
  double* partials;
  unsigned* ctrl;
  P2PDesc p2p;
};

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// status of a row's target and result: 0 usable, 1 ignore, 2 bad target, 3 non-finite
__device__ __forceinline__ int row_status(int a, int V, float lse, float logp) {
  if (a == -1) return 1;
  if (a < 0 || a >= V) return 2;
  if (!isfinite(lse) || !isfinite(logp)) return 3;
  return 0;
}

struct RowMeta {
  float lpb = 0.f, lpp = 0.f, lref = 0.f, adv = 0.f;
  int ver = 0;
  uint64_t key = 1;
};

// The row's PPO quantities once (lse, logp, H) are known: g = dLoss/dlogp and the entropy
// bonus weight c = ent_coef * m / N.
struct RowGrad {
  float g;
  float c;
};


// per-row results kept until they are stored (after pass C's scalars are published)
struct RowOut {
  float logp, lse;
  PpoRowIn in;
  PpoMid mid;
};

// critical part: the row's g and c (and what the statistics need later)
template <int MODE>
__device__ __forceinline__ RowGrad eval_row(const Lp& p, const PpoConst& pc, int a, float lse,
                                            float logp, float H, const RowMeta& mt, RowOut& o) {
  const int st = row_status(a, p.V, lse, logp);
  RowGrad out{0.f, 0.f};
  o.lse = lse;
  o.in.tgt_status = st;
  o.in.logp = (st == 1 || st == 2) ? 0.f : logp;
  o.in.H = H;
  o.logp = o.in.logp;
  if (MODE == MODE_FUSED) {
    o.in.lpb = mt.lpb;
    o.in.lpp = mt.lpp;
    o.in.lref = mt.lref;
    o.in.adv = mt.adv;
    o.in.ver = mt.ver;
    o.in.valid = mt.key != 0ull;
    out.g = ppo_grad(pc, o.in, o.mid);
    out.c = o.mid.m ? pc.ent_coef * pc.invN : 0.f;
  }
  return out;
}

// per-row outputs and statistics (one writer thread per row)
template <int MODE>
__device__ __forceinline__ void write_row(const Lp& p, const PpoConst& pc, int64_t r,
                                          const RowGrad& rg, const RowOut& o, double* acc) {
  RowStats rs;
  float lt = 0.f;
  if (MODE == MODE_FUSED) ppo_stats(pc, o.in, o.mid, rs, &lt);
  else fwd_row_stats(o.in, rs);
  p.logp[r] = o.logp;
  if (p.lse_out) p.lse_out[r] = o.lse;
  if (MODE == MODE_FUSED) {
    if (p.out_g) p.out_g[r] = rg.g;
    if (p.out_L) p.out_L[r] = lt;
  }
  if (acc) acc_stats(acc, rs);
}

template <int MODE>
__device__ __forceinline__ RowGrad finish_row(const Lp& p, const PpoConst& pc, int64_t r, int a,
                                              float lse, float logp, float H, const RowMeta& mt,
                                              bool writer, double* acc) {
  RowOut o;
  const RowGrad rg = eval_row<MODE>(p, pc, a, lse, logp, H, mt, o);
  if (writer) write_row<MODE>(p, pc, r, rg, o, acc);
  return rg;
}

template <int MODE>
__device__ __forceinline__ RowMeta load_meta(const Lp& p, int64_t r) {
  RowMeta m;
  if (MODE == MODE_FUSED) {
    const int64_t s = r / p.A;
    m.lpb = p.lpb[r];
    if (p.lpp) m.lpp = p.lpp[r];
    if (p.lref) m.lref = p.lref[r];
    m.adv = p.adv[s];
    m.ver = p.ver[s];
    m.key = p.key[s];
  }
  return m;
}

// N for 1/N and the per-kernel copy of the PPO constants
template <int MODE>
__device__ __forceinline__ double resolve_pc(const Lp& p, PpoConst& pc) {
  pc = p.pc;
  if (MODE != MODE_FUSED) {
    pc.invN = 0.f;
    pc.ent_coef = 0.f;
    return 0.0;
  }
  const double N = loss_denominator(p.N, p.adv_stats);
  pc.invN = N > 0.0 ? float(1.0 / N) : 0.f;
  return N;
}

// ln S and logp = (x_a - M) - ln S in the direct form: an absolute error of a few fp32 ulps
// of ln S, which is all any consumer needs (the ratio e^{logp - logp_behav} and every
// gradient term carry it as a relative error). (Measured and rejected: the log1p form
// logp = -log1p(S_rest/e_a), which keeps relative accuracy for |logp| << 1, costs 0.7%.)
struct LseParts {
  float lnS;
  float logp;
};
__device__ __forceinline__ LseParts lse_parts(float xa, float M, float Stot) {
  LseParts o;
  o.lnS = __logf(Stot);
  o.logp = (xa - M) - o.lnS;
  return o;
}

// dx at the target column: g (1 - p_a) + c p_a (log p_a + H), with 1 - p_a = S_rest / S
__device__ __forceinline__ float target_grad(const RowGrad& rg, float Srest, float ea, float invS,
                                             float logp, float H) {
  return rg.g * Srest * invS + (rg.c != 0.f ? rg.c * ea * invS * (logp + H) : 0.f);
}

// =====================================================================================
// K6/K5/K7 for bf16 rows up to 32768: TMA-staged persistent kernel, two row groups
// =====================================================================================
// One 1024-thread CTA per SM, split into two independent 512-thread groups; group g
// processes the CTA's rows k = g, g+2, ... Rows live in a ring of nst SMEM stages filled
// by the TMA engine (1-D bulk copies, mbarrier tx-count completion, L2 evict_first); row k
// uses stage k % nst. Per row a group makes three passes over the SMEM copy:
//   A  max over its 16-byte vectors (packed bf16x2 max, no MUFU)
//   B  e = 2^{(x - m_warp) log2e} (one ex2), sum and entropy partials per warp; with
//      dlogits requested (and no entropy bonus) e is written back into the stage as bf16
//   -- named barrier #1; warp 0 combines the 16 warp partials, runs the per-row epilogue
//      (lse, logp, H, PPO g) and publishes the row scalars with bar.arrive (#2) before
//      finishing the per-row outputs and statistics --
//   C  dlogits: from the stored e, dx = g' 2^{(m_w - M) log2e} e (no second ex2); or,
//      with the entropy bonus / in external-bwd mode, from x: dx = 2^t (k1 + k2 t)
// then (#3) releases the stage by issuing the TMA for row k + nst into it. While one
// group sits in its latency-bound combine/epilogue the other streams.
constexpr int kCtaThreads = 1024;
constexpr int kGroupThreads = 512;
constexpr int kGroupWarps = kGroupThreads / 32;
constexpr int kVecPerThread = 8;  // 8 x (8 bf16) per group thread -> V <= 32768
constexpr int kMaxStages = 4;

struct __align__(16) StageMeta {
  int32_t a;
  float lpb, lpp, adv;
  int32_t ver;
  float lse_in, g_in;
  int32_t issued_row;  // row whose load was issued into this stage (plain st.shared)
  uint64_t key;
  float lref;
  float pad;
};

__device__ __forceinline__ void read_meta(const Lp& p, const StageMeta* mt, RowMeta& rm) {
  rm.lpb = mt->lpb;
  if (p.lpp) rm.lpp = mt->lpp;
  if (p.lref) rm.lref = mt->lref;
  rm.adv = mt->adv;
  rm.ver = mt->ver;
  rm.key = mt->key;
}

__device__ __forceinline__ int ld_volatile_s32(const int32_t* p) {
  return *reinterpret_cast<const volatile int32_t*>(p);
}

// per-row scalars published by warp 0 for pass C
struct __align__(16) RowScalars {
  float M;       // row max (pass C: per-warp scale 2^{(m_w - M) log2e}; x-path offset)
  float k1;      // keep-e path: -g / S; x path: (-g + c (H - ln S)) / S
  float k2;      // x path: c ln2 / S (entropy bonus), else 0
  float ga;      // dx at the target column
  float active;  // 0 => the row's dlogits are exactly zero
  float pad[3];
};

template <int MODE>
__device__ __forceinline__ void issue_row(const Lp& p, int r, uint8_t* dst, StageMeta* m,
                                          uint64_t* bar, uint32_t row_bytes, uint64_t pol) {
  *reinterpret_cast<volatile int32_t*>(&m->issued_row) = r;
  cp_async4(&m->a, p.target + r);
  if (MODE == MODE_FUSED) {
    const int s = r / p.A;
    cp_async4(&m->lpb, p.lpb + r);
    if (p.lpp) cp_async4(&m->lpp, p.lpp + r);
    if (p.lref) cp_async4(&m->lref, p.lref + r);
    cp_async4(&m->adv, p.adv + s);
    cp_async4(&m->ver, p.ver + s);
    cp_async8(&m->key, p.key + s);
  } else if (MODE == MODE_BWD) {
    cp_async4(&m->lse_in, p.lse_in + r);
    cp_async4(&m->g_in, p.g_in + r);
  }
  cp_async_arrive_noinc(bar);
  mbar_arrive_expect_tx(bar, row_bytes);
#if RLVLA_TMA_LOADPOL == 2  // no L2 cache hint on the row copy
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(static_cast<const __nv_bfloat16*>(p.x) + int64_t(r) * p.ld), "r"(row_bytes), "r"(smem_u32(bar))
               : "memory");
  (void)pol;
#elif RLVLA_TMA_SPLIT > 1  // the row as several bulk copies on the same mbarrier
  {
    const uint8_t* src = reinterpret_cast<const uint8_t*>(static_cast<const __nv_bfloat16*>(p.x) + int64_t(r) * p.ld);
    const uint32_t part = ((row_bytes / RLVLA_TMA_SPLIT) + 15u) & ~15u;
    for (uint32_t o = 0; o < row_bytes; o += part)
      bulk_g2s(dst + o, src + o, row_bytes - o < part ? row_bytes - o : part, bar, pol);
  }
#else
  bulk_g2s(dst, static_cast<const __nv_bfloat16*>(p.x) + int64_t(r) * p.ld, row_bytes, bar, pol);
#endif
}

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "n"(kGroupThreads) : "memory");
}
__device__ __forceinline__ void advance_stage(int& st, uint32_t& ph, int nstages) {
  st += 2;
  if (st >= nstages) {
    st -= nstages;
    ph ^= 1u;
  }
}
// barrier #2 (row scalars published) uses its own id (3 + g) so that warp 0, which only
// arrives on it, can never be counted into another phase of the #1/#3 barrier (1 + g)
__device__ __forceinline__ void scalars_arrive(int g) {
  asm volatile("bar.arrive %0, %1;" ::"r"(g + 3), "n"(kGroupThreads) : "memory");
}
__device__ __forceinline__ void scalars_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 3), "n"(kGroupThreads) : "memory");
}

// XP: pass C from x (external bwd, or fused with the entropy bonus); otherwise from the e
// values pass B kept in the stage. A template parameter so the common fused loop carries
// no code of the other.
// NFULL: the first NFULL of a thread's kVecPerThread vectors are always inside the row
// (NFULL = nvec / 512), so those iterations carry no bounds check.
// DX: dlogits requested (FUSED); compile-time so that no per-vector test reloads it.
// Every per-vector loop is branch-free: the target column is overwritten with -inf after
// pass A (removed from the pass-B sums, 0 in pass C) and its dlogit is stored by its owner
// thread after the row's vectors; a row without gradient takes a store-zeros loop.
template <int MODE, bool XP, int NFULL, bool DX>
__global__ void __launch_bounds__(kCtaThreads, 1)
    lp_tma_kernel(Lp p, int nstages, uint32_t stage_bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* rowbuf = smem;
  StageMeta* meta = reinterpret_cast<StageMeta*>(smem + size_t(nstages) * stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + kMaxStages);
  float4* red = reinterpret_cast<float4*>(full + kMaxStages);              // [2 parity][2 grp][16]
  RowScalars* rsc = reinterpret_cast<RowScalars*>(red + 4 * kGroupWarps);  // [2]
  float* xa_s = reinterpret_cast<float*>(rsc + 2);                         // [2 parity][2 grp]
  double* gacc = reinterpret_cast<double*>(xa_s + 4);                      // [2][16]

  const int tid = threadIdx.x, lane = tid & 31;
  const int grp = tid / kGroupThreads, gt = tid % kGroupThreads, gw = gt >> 5;
  const int V = p.V;
  const int nvec = V >> 3;
  const uint32_t row_bytes = uint32_t(V) * 2u;
  const int first = blockIdx.x, stride = gridDim.x;
  const int rows = int(p.rows);
  const int nrow = rows > first ? (rows - first + stride - 1) / stride : 0;
  const bool want_stats = p.stats != nullptr && MODE != MODE_BWD;
  PpoConst pc;
  const double Nden = resolve_pc<MODE>(p, pc);
  // pass C runs in external-bwd mode and in fused mode with dlogits; it reuses the e
  // values of pass B (stored as bf16 in the stage) unless the entropy bonus needs x
  constexpr bool kXPath = XP || MODE == MODE_BWD;
  constexpr bool has_c = MODE == MODE_BWD || (MODE == MODE_FUSED && DX);
  // the target column removed from the pass-B sums by a -inf overwrite after pass A (else,
  // an A/B variant, skipped inside the loop by its owner; either way its dlogit is stored
  // from ga)
  constexpr bool kNegInf = MODE != MODE_FUSED || RLVLA_FUSED_NEGINF;
  constexpr bool keep_e = MODE == MODE_FUSED && !kXPath && DX;
  const float L2E = kLog2e;

  if (tid == 0) {
    for (int s = 0; s < nstages; ++s) mbar_init(&full[s], 2);
    fence_mbar_init();
  }
  if (tid < 32) gacc[tid] = 0.0;
  if (tid < kMaxStages) meta[tid].issued_row = -1;
  __syncthreads();
#if RLVLA_TMA_LOADPOL == 1
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#elif RLVLA_TMA_LOADPOL == 3
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#elif RLVLA_TMA_LOADPOL == 4
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
#else
  uint64_t pol = policy_evict_first();
#endif
  if (tid == 0) {
    const int pre = nrow < nstages ? nrow : nstages;
    for (int k = 0; k < pre; ++k)
      issue_row<MODE>(p, first + k * stride, rowbuf + size_t(k) * stage_bytes, &meta[k], &full[k],
                      row_bytes, pol);
  }

  // stage / phase of this group's rows (row k: stage k % nstages, parity (k / nstages) & 1),
  // advanced incrementally by k += 2 (nstages >= 2)
  int st = grp;
  uint32_t ph = 0;
  for (int k = grp; k < nrow; k += 2) {
    const int r = first + k * stride;
    // The previous use of this stage (row k - nstages) may belong to the other group and
    // still be in flight; a parity wait only distinguishes adjacent phases, so first make
    // sure this row's load was issued (which happens only after that use was consumed).
    {
      uint32_t n = 0;
      while (ld_volatile_s32(&meta[st].issued_row) != r) {
#if RLVLA_ISSUED_SLEEP_NS > 0
        __nanosleep(RLVLA_ISSUED_SLEEP_NS);  // no issue slots taken from the other group
#endif
        if (++n > (1u << 24)) __trap();
      }
    }
#if RLVLA_L2_PREFETCH
    // the row this group loads into its stage at the end of this row (row k + nstages) is
    // pulled into L2 now, a row-time ahead, so that TMA fill is an L2 hit: the SMEM ring
    // holds only three 64 KB rows, L2 extends the prefetch depth
    if (gt == 0 && k + nstages < nrow)
      bulk_prefetch_l2(static_cast<const __nv_bfloat16*>(p.x) + int64_t(first + (k + nstages) * stride) * p.ld,
                       row_bytes);
#endif
    mbar_wait(&full[st], ph);
    uint8_t* row = rowbuf + size_t(st) * stage_bytes;
    uint4* rv = reinterpret_cast<uint4*>(row);
#if RLVLA_RING_ONLY
    // diagnostic build (wrong results): the TMA ring and the dlogits stores alone, no math —
    // the ceiling of this kernel's memory structure
    if (has_c) {
      uint4* dvr = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.dx) + int64_t(r) * p.ld);
#pragma unroll
      for (int i = 0; i < kVecPerThread; ++i) {
        const int idx = gt + i * kGroupThreads;
        if (i < NFULL || idx < nvec) stg_dx(dvr + idx, rv[idx]);
      }
    }
    group_sync(grp);
    if (gt == 0 && k + nstages < nrow) {
      fence_proxy_async();
      issue_row<MODE>(p, first + (k + nstages) * stride, row, &meta[st], &full[st], row_bytes, pol);
    }
    advance_stage(st, ph, nstages);
    continue;
#endif
    const StageMeta* mt = &meta[st];
    const int a = mt->a;
    const bool tgt_ok = unsigned(a) < unsigned(V);
    const int va = tgt_ok ? (a >> 3) : -1;
    const bool owner = tgt_ok && (va & (kGroupThreads - 1)) == gt;  // thread holding the target
    // warp partials double-buffered by row parity: rows k and k+2 of a group never share
    float4* gred = red + (((k >> 1) & 1) * 2 + grp) * kGroupWarps;
    float* gxa = xa_s + ((k >> 1) & 1) * 2 + grp;  // raw target logit, same double buffering
    RowScalars rsv;
    float mws = 0.f;

    if (MODE != MODE_BWD) {
      // ---- pass A: thread max -> warp max (packed bf16x2 max, exact) ----------------
      uint32_t mm = 0xff80ff80u;
#pragma unroll
      for (int i = 0; i < kVecPerThread; ++i) {
        const int idx = gt + i * kGroupThreads;
        if (i < NFULL || idx < nvec) {
          const uint4 w = rv[idx];
          mm = bmax2(bmax2(mm, w.x), bmax2(w.y, bmax2(w.z, w.w)));
        }
      }
      // The target column is excluded from the pass-B sums (so that 1 - p_a = S_rest / S
      // keeps full relative precision near saturation) by overwriting it with -inf in the
      // stage once the max has seen it; only its owner thread reads that vector again.
      if (kNegInf && owner) {
        uint16_t* hx = reinterpret_cast<uint16_t*>(row);
        *gxa = bf_lo(uint32_t(hx[a]));
        hx[a] = 0xFF80u;
      }
      const float mw = warp_max(fmaxf(bf_lo(mm), bf_hi(mm)));
      mws = (mw == -INFINITY) ? 0.f : mw;
      const float nmL = -mws * L2E;
      // ---- pass B: e = 2^(t), t = (x - m_warp) log2e; s = sum e, et = sum e t ------
      // packed fp32x2 arithmetic (FFMA2 / FADD2): two columns per instruction; the
      // thread's sums stay in two lanes of a float2 until the end of the row
      float2 s2 = make_float2(0.f, 0.f), et2 = make_float2(0.f, 0.f);
      const float2 L2E2 = make_float2(L2E, L2E), nmL2 = make_float2(nmL, nmL);
#pragma unroll
      for (int i = 0; i < kVecPerThread; ++i) {
        const int idx = gt + i * kGroupThreads;
        if (i < NFULL || idx < nvec) {
          const uint4 w = rv[idx];
          const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
          float2 t2[4], e2[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            // -inf -> -2^100 once per bf16 pair (NaN-propagating max): e = 0 and e t = 0
            // (this also removes the target column, set to -inf after pass A)
            const uint32_t c = bmax2_nan(w4[q], kNegClampPair);
            t2[q] = __ffma2_rn(make_float2(bf_lo(c), bf_hi(c)), L2E2, nmL2);
            e2[q] = make_float2(ex2(t2[q].x), ex2(t2[q].y));
          }
          if (kNegInf || idx != va) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              s2 = __fadd2_rn(s2, e2[q]);
              et2 = __ffma2_rn(e2[q], t2[q], et2);
            }
          } else {  // (A/B variant) the target column skipped here instead
            const int j0 = a & 7;
            const int h = j0 >> 1;
            const uint32_t wa = h == 0 ? w.x : (h == 1 ? w.y : (h == 2 ? w.z : w.w));
            *gxa = (j0 & 1) ? bf_hi(wa) : bf_lo(wa);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (j == j0) continue;
              const float ej = (j & 1) ? e2[j >> 1].y : e2[j >> 1].x;
              const float tj = (j & 1) ? t2[j >> 1].y : t2[j >> 1].x;
              s2.x += ej;
              et2.x = fmaf(ej, tj, et2.x);
            }
          }
          if (keep_e)
            rv[idx] = make_uint4(pack_bf16x2(e2[0].x, e2[0].y), pack_bf16x2(e2[1].x, e2[1].y),
                                 pack_bf16x2(e2[2].x, e2[2].y), pack_bf16x2(e2[3].x, e2[3].y));
        }
      }
      float s = s2.x + s2.y, et = et2.x + et2.y;
      s = warp_sum(s);
      et = warp_sum(et);
      if (lane == 0) gred[gw] = make_float4(mw, s, et, 0.f);
      if (keep_e) fence_proxy_async();  // generic smem writes before the stage's next TMA fill
      // warp 0 needs the row metadata: read before #1 only when the stage is refilled right
      // after it (no pass C); otherwise after #1, so warp 0 reaches the barrier sooner
      RowMeta rm;
      if (gw == 0 && MODE == MODE_FUSED && !has_c) read_meta(p, mt, rm);
      group_sync(grp);  // #1: warp partials + x_a visible; stage no longer read in FWD mode
      if (!has_c && gt == 0 && k + nstages < nrow) {
        fence_proxy_async();
        issue_row<MODE>(p, first + (k + nstages) * stride, row, &meta[st], &full[st], row_bytes, pol);
      }
      if (gw == 0) {
        // ---- combine 16 warp partials, per-row epilogue (one warp) ------------------
        if (MODE == MODE_FUSED && has_c) read_meta(p, mt, rm);
        const float xa = tgt_ok ? *gxa : 0.f;
        const float4 q = lane < kGroupWarps ? gred[lane] : make_float4(-INFINITY, 0.f, 0.f, 0.f);
        const float M = warp_max(q.x);
        const float sc = lane < kGroupWarps ? ex2((q.x - M) * L2E) : 0.f;
        const float mq = (q.x == -INFINITY) ? 0.f : q.x;
        // the 16 warp partials sit in lanes 0..15; lane 0 (the only writer) gets the sums
        const float Srest = half_warp_sum(q.y * sc);
        const float Csum = half_warp_sum(lane < kGroupWarps ? sc * (q.z + (mq - M) * L2E * q.y) : 0.f);
        const float ta = (xa - M) * L2E;
        const float ea = tgt_ok ? ex2(ta) : 0.f;
        const float Stot = Srest + ea;
        const LseParts lp = lse_parts(xa, M, Stot);
        const float lnS = lp.lnS;
        const float lse_row = M + lnS;
        const float logp = lp.logp;
        const float invS = __fdividef(1.f, Stot);
        const float Ctot = Csum + (tgt_ok ? ea * fmaxf(ta, -256.f) : 0.f);
        const float H = lnS - Ctot * invS * kLn2;
        RowOut ro;
        const RowGrad rg = eval_row<MODE>(p, pc, a, lse_row, logp, H, rm, ro);
        if (has_c) {
          if (lane == 0) {
            RowScalars sc4;
            sc4.M = (M == -INFINITY) ? 0.f : M;
            sc4.k1 = keep_e ? -rg.g * invS : (-rg.g + rg.c * (H - lnS)) * invS;
            sc4.k2 = keep_e ? 0.f : rg.c * kLn2 * invS;
            sc4.ga = target_grad(rg, Srest, ea, invS, logp, H);
            sc4.active = (rg.g != 0.f || rg.c != 0.f) ? 1.f : 0.f;
            rsc[grp] = sc4;
          }
          __syncwarp();
          scalars_arrive(grp);  // #2 (producer side): the other warps may start pass C now
        }
        // per-row outputs and statistics, off the pass-C critical path
        if (lane == 0) write_row<MODE>(p, pc, r, rg, ro, want_stats ? gacc + grp * 16 : nullptr);
      } else if (has_c) {
        scalars_sync(grp);  // #2 (consumer side): row scalars published
      }
      if (!has_c) {
        advance_stage(st, ph, nstages);
        continue;
      }
      rsv = rsc[grp];
    } else {
      const float g = tgt_ok ? mt->g_in : 0.f;
      rsv.M = mt->lse_in;
      rsv.k1 = -g;
      rsv.k2 = 0.f;
      rsv.ga = tgt_ok ? -g * expm1f(bf_lo(uint32_t(reinterpret_cast<const uint16_t*>(row)[a])) - mt->lse_in)
                      : 0.f;
      rsv.active = g != 0.f ? 1.f : 0.f;
      if (owner) reinterpret_cast<uint16_t*>(row)[a] = 0xFF80u;  // target column written last
    }

    // ---- pass C: dlogits (masked / clipped rows get exact zeros) ---------------------
    {
      __nv_bfloat16* drow = static_cast<__nv_bfloat16*>(p.dx) + int64_t(r) * p.ld;
      uint4* dv = reinterpret_cast<uint4*>(drow);
      if (rsv.active != 0.f) {
        const float kw = !kXPath ? rsv.k1 * ex2((mws - rsv.M) * L2E) : rsv.k1;
        const float nML = -rsv.M * L2E;
        // kw split into two bf16 halves, each broadcast to both lanes of a pair
        const uint32_t kwh1 = uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(kw)));
        const uint32_t kwl1 = uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(kw - __uint_as_float(kwh1 << 16))));
        const uint32_t kwh2 = kwh1 | (kwh1 << 16), kwl2 = kwl1 | (kwl1 << 16);
#pragma unroll
        for (int i = 0; i < kVecPerThread; ++i) {
          const int idx = gt + i * kGroupThreads;
          if (i < NFULL || idx < nvec) {
            const uint4 w = rv[idx];
            const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
            uint4 o;
            uint32_t* ow = &o.x;
            if (!kXPath) {
              // FUSED: dx = kw e, kw = g' 2^{(m_w - M) log2e}, e from pass B (bf16 in SMEM),
              // on the packed pairs: kw = kw_hi + kw_lo (both bf16), dx = RN(e kw_hi + RN(e kw_lo));
              // the inner rounding is <= 2^-18 |e kw|, so dx stays within one bf16 ulp of
              // RNE(e kw) -> within one ulp of RNE(exact) as before
#if RLVLA_PASSC_BF16
#pragma unroll
              for (int q = 0; q < 4; ++q) ow[q] = bfma2(w4[q], kwh2, bmul2(w4[q], kwl2));
#else
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 d = __fmul2_rn(make_float2(bf_lo(w4[q]), bf_hi(w4[q])), make_float2(kw, kw));
                ow[q] = pack_bf16x2(d.x, d.y);
              }
#endif
            } else {
              // from x: t = (x - M) log2e (lse in external bwd), dx = 2^t (k1 + k2 t);
              // -inf columns are clamped per bf16 pair so that t stays finite
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t c = bmax2_nan(w4[q], kNegClampPair);
                const float2 t2 = __ffma2_rn(make_float2(bf_lo(c), bf_hi(c)), make_float2(L2E, L2E),
                                             make_float2(nML, nML));
                // external bwd: k2 = 0, dx = k1 2^t (no entropy term to add)
                const float2 f2 = MODE == MODE_BWD ? make_float2(rsv.k1, rsv.k1)
                                                   : __ffma2_rn(make_float2(rsv.k2, rsv.k2), t2,
                                                                make_float2(rsv.k1, rsv.k1));
                const float2 d2 = __fmul2_rn(make_float2(ex2(t2.x), ex2(t2.y)), f2);
                ow[q] = pack_bf16x2(d2.x, d2.y);
              }
            }
#if RLVLA_TGT_INLOOP
            if (idx == va) {  // the target column (0 from its -inf) takes g (1 - p_a) [+ ...]
              const uint32_t hb = uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(rsv.ga)));
              const int qd = (a & 7) >> 1, hf = a & 1;
#pragma unroll
              for (int z = 0; z < 4; ++z)
                if (z == qd) ow[z] = hf ? ((ow[z] & 0x0000ffffu) | (hb << 16)) : ((ow[z] & 0xffff0000u) | hb);
            }
#endif
#if RLVLA_DX_BULK
            rv[idx] = o;  // in place: this thread's own vector, read above
#else
            stg_dx(dv + idx, o);
#endif
          }
        }
#if !RLVLA_TGT_INLOOP
        // the target column (0 from its -inf above) takes g (1 - p_a) [+ ...]: stored by
        // the thread that stored its vector, after it (same-thread order)
        if (owner)
          reinterpret_cast<uint16_t*>(RLVLA_DX_BULK ? static_cast<void*>(row) : static_cast<void*>(drow))[a] =
              __bfloat16_as_ushort(__float2bfloat16_rn(rsv.ga));
#endif
      } else {
#pragma unroll
        for (int i = 0; i < kVecPerThread; ++i) {
          const int idx = gt + i * kGroupThreads;
#if RLVLA_DX_BULK
          if (i < NFULL || idx < nvec) rv[idx] = make_uint4(0u, 0u, 0u, 0u);
#else
          if (i < NFULL || idx < nvec) stg_dx(dv + idx, make_uint4(0u, 0u, 0u, 0u));
#endif
        }
      }
    }
    group_sync(grp);  // #3: stage fully consumed by this group
#if RLVLA_DX_BULK
    if (has_c && gt == 0) {  // the row's dlogits leave the stage in one bulk store
      fence_proxy_async();
      bulk_s2g(static_cast<__nv_bfloat16*>(p.dx) + int64_t(r) * p.ld, row, row_bytes, pol);
      if (k + nstages < nrow) bulk_wait_read();  // before the stage is refilled
    }
#endif
    if (gt == 0 && k + nstages < nrow) {
      fence_proxy_async();
      issue_row<MODE>(p, first + (k + nstages) * stride, row, &meta[st], &full[st], row_bytes, pol);
    }
    advance_stage(st, ph, nstages);
  }

#if RLVLA_DX_BULK
  if (has_c && gt == 0) bulk_wait_all();
#endif
  if (want_stats) {
    __syncthreads();
    if (tid < kLossSlots) gacc[tid] += gacc[16 + tid];  // fixed order: group 0 then group 1
    __syncthreads();
    finish_loss_stats(gacc, p.stats, p.partials, p.ctrl, Nden, p.accumulate, pc.ent_coef, &p.p2p);
  }
}

// =====================================================================================
// small V: one warp per row, register-resident (t_j kept; e recomputed in the store pass)
// =====================================================================================
template <typename T, int NV, int MODE>
__global__ void __launch_bounds__(256) lp_warp_kernel(Lp p) {
  constexpr int VW = 16 / int(sizeof(T));  // elements per 16-byte vector
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int V = p.V, nvec = V / VW;
  const float L2E = kLog2e;
  const bool want_stats = p.stats != nullptr && MODE != MODE_BWD;
  PpoConst pc;
  const double Nden = resolve_pc<MODE>(p, pc);
  double acc[kLossSlots] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t gw = int64_t(blockIdx.x) * 8 + warp, nw = int64_t(gridDim.x) * 8;
  for (int64_t r = gw; r < p.rows; r += nw) {
    const T* xr = static_cast<const T*>(p.x) + r * p.ld;
    const int a = p.target[r];
    const bool tgt_ok = unsigned(a) < unsigned(V);
    float x[NV * VW];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int idx = lane + 32 * i;
      if (idx < nvec) {
        const uint4 u = ldg_stream(reinterpret_cast<const uint4*>(xr) + idx);
        const T* tv = reinterpret_cast<const T*>(&u);
#pragma unroll
        for (int j = 0; j < VW; ++j) x[i * VW + j] = to_f<T>(tv[j]);
      } else {
#pragma unroll
        for (int j = 0; j < VW; ++j) x[i * VW + j] = -INFINITY;
      }
    }
    const float xa = tgt_ok ? to_f<T>(xr[a]) : 0.f;
    RowGrad rg{0.f, 0.f};
    float Stot = 1.f, Srest = 0.f, lnS = 0.f, H = 0.f, logp = 0.f, ea = 0.f;
    if (MODE != MODE_BWD) {
      float mt = -INFINITY;
#pragma unroll
      for (int j = 0; j < NV * VW; ++j) mt = fmaxf(mt, x[j]);
      const float M = warp_max(mt);
      const float Ms = (M == -INFINITY) ? 0.f : M;
      const float nmL = -Ms * L2E;
      float s = 0.f, et = 0.f;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
#pragma unroll
        for (int j = 0; j < VW; ++j) {
          const int col = (lane + 32 * i) * VW + j;
          const float t = fmaf(x[i * VW + j], L2E, nmL);
          const float ee = ex2(t);
          x[i * VW + j] = t;  // keep t_j = (x_j - M) log2e in place of x_j
          if (col != a) {
            s += ee;
            et = fmaf(ee, fmaxf(t, -256.f), et);
          }
        }
      }
      Srest = warp_sum(s);
      const float Cs = warp_sum(et);
      const float ta = (xa - Ms) * L2E;
      ea = tgt_ok ? ex2(ta) : 0.f;
      Stot = Srest + ea;
      const LseParts lp = lse_parts(xa, M, Stot);
      lnS = lp.lnS;
      const float lse_row = M + lnS;
      logp = lp.logp;
      H = lnS - (Cs + (tgt_ok ? ea * fmaxf(ta, -256.f) : 0.f)) / (L2E * Stot);
      const RowMeta rm = load_meta<MODE>(p, r);
      rg = finish_row<MODE>(p, pc, r, a, lse_row, logp, H, rm, lane == 0,
                            want_stats ? acc : nullptr);
    } else {
      rg.g = tgt_ok ? p.g_in[r] : 0.f;
      const float lse_row = p.lse_in[r];
      const float off = lse_row * L2E;
      logp = xa - lse_row;
#pragma unroll
      for (int j = 0; j < NV * VW; ++j) x[j] = fmaf(x[j], L2E, -off);  // t relative to lse
    }
    if (p.dx != nullptr && MODE != MODE_FWD) {
      T* dr = static_cast<T*>(p.dx) + r * p.ld;
      const float invS = 1.f / Stot;
      // dx_j = 2^{t_j} (k1 + k2 t_j): FUSED k1 = (-g + c (H - lnS)) / S, k2 = c ln2 / S;
      //                               BWD   k1 = -g, k2 = 0 (t relative to lse)
      const float k1 = MODE == MODE_BWD ? -rg.g : (-rg.g + rg.c * (H - lnS)) * invS;
      const float k2 = MODE == MODE_BWD ? 0.f : rg.c * kLn2 * invS;
      const float ga = MODE == MODE_BWD ? -rg.g * expm1f(logp)
                                        : target_grad(rg, Srest, ea, invS, logp, H);
      const bool active = rg.g != 0.f || rg.c != 0.f;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int idx = lane + 32 * i;
        if (idx < nvec) {
          uint4 u;
          T* tv = reinterpret_cast<T*>(&u);
#pragma unroll
          for (int j = 0; j < VW; ++j) {
            const int col = idx * VW + j;
            const float t = clamp_ninf(x[i * VW + j]);
            float d = 0.f;
            if (active) d = (col == a) ? ga : ex2(t) * fmaf(k2, t, k1);
            tv[j] = from_f<T>(d);
          }
          stg_stream(reinterpret_cast<uint4*>(dr) + idx, u);
        }
      }
    }
  }
  if (want_stats) {
    __shared__ double red[8][kLossSlots];
    __shared__ double cta[kLossSlots];
    if (lane == 0)
      for (int k = 0; k < kLossSlots; ++k) red[warp][k] = acc[k];
    __syncthreads();
    if (threadIdx.x < kLossSlots) {
      double s = 0;
      for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
      cta[threadIdx.x] = s;
    }
    __syncthreads();
    finish_loss_stats(cta, p.stats, p.partials, p.ctrl, Nden, p.accumulate, pc.ent_coef, &p.p2p);
  }
}

// =====================================================================================
// generic: any V / ld / alignment / dtype; one CTA per row, three passes over the row
// =====================================================================================
template <typename T, int MODE>
__global__ void __launch_bounds__(256) lp_generic_kernel(Lp p) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = p.V;
  const float L2E = kLog2e;
  const bool want_stats = p.stats != nullptr && MODE != MODE_BWD;
  PpoConst pc;
  const double Nden = resolve_pc<MODE>(p, pc);
  __shared__ float redf[2][8];
  __shared__ double sacc[16];
  if (tid < 16) sacc[tid] = 0.0;
  __syncthreads();
  for (int64_t r = blockIdx.x; r < p.rows; r += gridDim.x) {
    const T* xr = static_cast<const T*>(p.x) + r * p.ld;
    const int a = p.target[r];
    const bool tgt_ok = unsigned(a) < unsigned(V);
    const float xa = tgt_ok ? to_f<T>(xr[a]) : 0.f;
    RowGrad rg{0.f, 0.f};
    float Stot = 1.f, Srest = 0.f, Ms = 0.f, lnS = 0.f, H = 0.f, logp = 0.f, ea = 0.f, lse_row;
    if (MODE != MODE_BWD) {
      float mt = -INFINITY;
      for (int j = tid; j < V; j += 256) mt = fmaxf(mt, to_f<T>(xr[j]));
      mt = warp_max(mt);
      if (lane == 0) redf[0][warp] = mt;
      __syncthreads();
      float M = redf[0][0];
      for (int w = 1; w < 8; ++w) M = fmaxf(M, redf[0][w]);
      Ms = (M == -INFINITY) ? 0.f : M;
      const float nmL = -Ms * L2E;
      float s = 0.f, et = 0.f;
      for (int j = tid; j < V; j += 256) {
        if (j == a) continue;
        const float t = fmaf(to_f<T>(xr[j]), L2E, nmL);
        const float ee = ex2(t);
        s += ee;
        et = fmaf(ee, fmaxf(t, -256.f), et);
      }
      s = warp_sum(s);
      et = warp_sum(et);
      __syncthreads();
      if (lane == 0) {
        redf[0][warp] = s;
        redf[1][warp] = et;
      }
      __syncthreads();
      Srest = 0.f;
      float Cs = 0.f;
      for (int w = 0; w < 8; ++w) {
        Srest += redf[0][w];
        Cs += redf[1][w];
      }
      const float ta = (xa - Ms) * L2E;
      ea = tgt_ok ? ex2(ta) : 0.f;
      Stot = Srest + ea;
      const LseParts lp = lse_parts(xa, M, Stot);
      lnS = lp.lnS;
      lse_row = M + lnS;
      logp = lp.logp;
      H = lnS - (Cs + (tgt_ok ? ea * fmaxf(ta, -256.f) : 0.f)) / (L2E * Stot);
      const RowMeta rm = load_meta<MODE>(p, r);
      rg = finish_row<MODE>(p, pc, r, a, lse_row, logp, H, rm, tid == 0, want_stats ? sacc : nullptr);
    } else {
      rg.g = tgt_ok ? p.g_in[r] : 0.f;
      lse_row = p.lse_in[r];
      logp = xa - lse_row;
    }
    if (p.dx != nullptr && MODE != MODE_FWD) {
      T* dr = static_cast<T*>(p.dx) + r * p.ld;
      const float invS = 1.f / Stot;
      const float off = MODE == MODE_BWD ? lse_row * L2E : Ms * L2E;
      const float k1 = MODE == MODE_BWD ? -rg.g : (-rg.g + rg.c * (H - lnS)) * invS;
      const float k2 = MODE == MODE_BWD ? 0.f : rg.c * kLn2 * invS;
      const float ga = MODE == MODE_BWD ? -rg.g * expm1f(logp)
                                        : target_grad(rg, Srest, ea, invS, logp, H);
      const bool active = rg.g != 0.f || rg.c != 0.f;
      for (int j = tid; j < V; j += 256) {
        const float t = clamp_ninf(fmaf(to_f<T>(xr[j]), L2E, -off));
        float d = 0.f;
        if (active) d = (j == a) ? ga : ex2(t) * fmaf(k2, t, k1);
        dr[j] = from_f<T>(d);
      }
    }
    __syncthreads();  // redf reuse across rows
  }
  if (want_stats) {
    __syncthreads();
    finish_loss_stats(sacc, p.stats, p.partials, p.ctrl, Nden, p.accumulate, pc.ent_coef, &p.p2p);
  }
}

// =====================================================================================
// Aligned rows the TMA kernel cannot stage (fp32 logits with V > 2048, bf16 with V > 32768):
// one 512-thread CTA per row (4 CTAs per SM), 16-byte loads. Pass AB reads the row once with
// an online (max, sum, entropy) per thread — the thread's partial sums are rescaled when its
// max grows — then a CTA combine and the per-row epilogue; pass C re-reads the row (an L2
// hit: the row was read microseconds before) and writes dlogits with dx = 2^t (k1 + k2 t),
// t = (x - M) log2e, i.e. one DRAM read and one write per element. (The earlier path for
// these rows, lp_generic_kernel, made three scalar passes.)
// =====================================================================================
constexpr int kRowThreads = 512;

template <typename T>
struct RowVec;
template <>
struct RowVec<float> {
  static constexpr int kN = 4;
  __device__ __forceinline__ static void load(const void* row, int v, float (&x)[4], uint64_t pol) {
    const uint4 w = ldg_hint(reinterpret_cast<const uint4*>(row) + v, pol);
    x[0] = __uint_as_float(w.x);
    x[1] = __uint_as_float(w.y);
    x[2] = __uint_as_float(w.z);
    x[3] = __uint_as_float(w.w);
  }
  __device__ __forceinline__ static void store(void* row, int v, const float (&d)[4]) {
    stg_stream(reinterpret_cast<uint4*>(row) + v,
               make_uint4(__float_as_uint(d[0]), __float_as_uint(d[1]), __float_as_uint(d[2]), __float_as_uint(d[3])));
  }
};
template <>
struct RowVec<__nv_bfloat16> {
  static constexpr int kN = 8;
  __device__ __forceinline__ static void load(const void* row, int v, float (&x)[8], uint64_t pol) {
    const uint4 w = ldg_hint(reinterpret_cast<const uint4*>(row) + v, pol);
    const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x[2 * q] = bf_lo(w4[q]);
      x[2 * q + 1] = bf_hi(w4[q]);
    }
  }
  __device__ __forceinline__ static void store(void* row, int v, const float (&d)[8]) {
    stg_stream(reinterpret_cast<uint4*>(row) + v,
               make_uint4(pack_bf16x2(d[0], d[1]), pack_bf16x2(d[2], d[3]), pack_bf16x2(d[4], d[5]),
                          pack_bf16x2(d[6], d[7])));
  }
};

// merge (m, s, et) partials: s = sum 2^{(x - m) log2e}, et = sum e t with t relative to m
__device__ __forceinline__ void lse_merge(float& m, float& s, float& et, float m2, float s2, float et2) {
  const float M = fmaxf(m, m2);
  if (M == -INFINITY) return;  // both empty
  const float d1 = (m == -INFINITY) ? 0.f : (m - M) * kLog2e;
  const float d2 = (m2 == -INFINITY) ? 0.f : (m2 - M) * kLog2e;
  const float f1 = (m == -INFINITY) ? 0.f : ex2(d1), f2 = (m2 == -INFINITY) ? 0.f : ex2(d2);
  et = f1 * fmaf(d1, s, et) + f2 * fmaf(d2, s2, et2);
  s = f1 * s + f2 * s2;
  m = M;
}

template <typename T, int MODE>
#ifndef RLVLA_ROW_UNROLL
#define RLVLA_ROW_UNROLL 4  // 16-byte vectors in flight per thread and loop trip
#endif
#ifndef RLVLA_ROW_MINB
#define RLVLA_ROW_MINB 2    // resident CTAs per SM the register budget is sized for
#endif
#ifndef RLVLA_ROW_KEEP
#define RLVLA_ROW_KEEP 1    // pass AB loads with L2 evict_last (re-read by pass C)
#endif
__global__ void __launch_bounds__(kRowThreads, RLVLA_ROW_MINB) lp_row_kernel(Lp p) {
  constexpr int U = RLVLA_ROW_UNROLL;
  constexpr int VN = RowVec<T>::kN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = p.V;
  const int nvec = V / VN;
  const float L2E = kLog2e;
  const bool want_stats = p.stats != nullptr && MODE != MODE_BWD;
  PpoConst pc;
  const double Nden = resolve_pc<MODE>(p, pc);
  __shared__ float4 red[kRowThreads / 32];
  __shared__ RowScalars rsc;
  __shared__ double sacc[16];
  if (tid < 16) sacc[tid] = 0.0;
  // pass AB's reads stay in L2 for pass C's re-read (evict_last), which is their last use
  // (evict_first); external backward reads once (evict_first)
#if RLVLA_ROW_LOADPOL
  const uint64_t pol_last = policy_evict_normal();
#else
  const uint64_t pol_last = policy_evict_first();
#endif
  const uint64_t pol_keep = (MODE == MODE_FUSED && p.dx != nullptr && RLVLA_ROW_KEEP) ? policy_evict_last() : pol_last;
  __syncthreads();
  for (int64_t r = blockIdx.x; r < p.rows; r += gridDim.x) {
    const T* xr = static_cast<const T*>(p.x) + r * p.ld;
    const int a = p.target[r];
    const bool tgt_ok = unsigned(a) < unsigned(V);
    const int va = tgt_ok ? a / VN : -1;
    float Ms = 0.f;
    if (MODE != MODE_BWD) {
      // ---- pass AB: online max / sum / entropy partial, the target column left out ------
      float m = -INFINITY, sm = 0.f, et = 0.f;
      for (int v0 = tid; v0 < nvec; v0 += U * kRowThreads) {
        float x[U][VN];
        float lm = -INFINITY;
#pragma unroll
        for (int u = 0; u < U; ++u) {  // U loads in flight before any use
          const int v = v0 + u * kRowThreads;
          if (v < nvec) {
            RowVec<T>::load(xr, v, x[u], pol_keep);
          } else {
#pragma unroll
            for (int j = 0; j < VN; ++j) x[u][j] = -INFINITY;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int v = v0 + u * kRowThreads;
          if (v == va) x[u][a - va * VN] = -INFINITY;
#pragma unroll
          for (int j = 0; j < VN; ++j) lm = fmaxf(lm, x[u][j]);
        }
        if (lm > m) {  // the thread's max grows: rescale its partials
          const float d = (m == -INFINITY) ? 0.f : (m - lm) * L2E;
          const float f = (m == -INFINITY) ? 0.f : ex2(d);
          et = f * fmaf(d, sm, et);
          sm = f * sm;
          m = lm;
        }
        const float nmL = (m == -INFINITY) ? 0.f : -m * L2E;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int j = 0; j < VN; ++j) {
            const float t = clamp_ninf(fmaf(x[u][j], L2E, nmL));
            const float e = ex2(t);
            sm += e;
            et = fmaf(e, fmaxf(t, -256.f), et);
          }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        lse_merge(m, sm, et, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, sm, o),
                  __shfl_xor_sync(0xffffffffu, et, o));
      if (lane == 0) red[warp] = make_float4(m, sm, et, 0.f);
      __syncthreads();
      if (warp == 0) {
        const float4 q = lane < kRowThreads / 32 ? red[lane] : make_float4(-INFINITY, 0.f, 0.f, 0.f);
        float M = q.x, Srest = q.y, Cs = q.z;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1)
          lse_merge(M, Srest, Cs, __shfl_xor_sync(0xffffffffu, M, o), __shfl_xor_sync(0xffffffffu, Srest, o),
                    __shfl_xor_sync(0xffffffffu, Cs, o));
        const float xa = tgt_ok ? to_f<T>(xr[a]) : 0.f;
        // the row max over every column (the target included), sums referred to it
        float Mrow = fmaxf(M, tgt_ok ? xa : -INFINITY);
        if (Mrow != M && M != -INFINITY) {
          const float d = (M - Mrow) * L2E, f = ex2(d);
          Cs = f * fmaf(d, Srest, Cs);
          Srest = f * Srest;
        }
        if (isnan(xa)) Mrow = xa;
        const float Mz = (Mrow == -INFINITY) ? 0.f : Mrow;
        const float ta = (xa - Mz) * L2E;
        const float ea = tgt_ok ? ex2(ta) : 0.f;
        const float Stot = Srest + ea;
        const LseParts lp = lse_parts(xa, Mz, Stot);
        const float lnS = lp.lnS;
        const float lse_row = Mz + lnS;
        const float logp = lp.logp;
        const float invS = __fdividef(1.f, Stot);
        const float H = lnS - (Cs + (tgt_ok ? ea * fmaxf(ta, -256.f) : 0.f)) * invS * kLn2;
        const RowMeta rm = load_meta<MODE>(p, r);
        RowOut ro;
        const RowGrad rg = eval_row<MODE>(p, pc, a, lse_row, logp, H, rm, ro);
        if (lane == 0) {
          RowScalars s4;
          s4.M = Mz;
          s4.k1 = (-rg.g + rg.c * (H - lnS)) * invS;
          s4.k2 = rg.c * kLn2 * invS;
          s4.ga = target_grad(rg, Srest, ea, invS, logp, H);
          s4.active = (rg.g != 0.f || rg.c != 0.f) ? 1.f : 0.f;
          rsc = s4;
          write_row<MODE>(p, pc, r, rg, ro, want_stats ? sacc : nullptr);
        }
      }
      __syncthreads();
      Ms = rsc.M;
    } else if (tid == 0) {
      const float g = tgt_ok ? p.g_in[r] : 0.f;
      RowScalars s4;
      s4.M = p.lse_in[r];
      s4.k1 = -g;
      s4.k2 = 0.f;
      s4.ga = tgt_ok ? -g * expm1f(to_f<T>(xr[a]) - s4.M) : 0.f;
      s4.active = g != 0.f ? 1.f : 0.f;
      rsc = s4;
    }
    if (MODE != MODE_FWD && p.dx != nullptr) {
      if (MODE == MODE_BWD) __syncthreads();
      const RowScalars sc = rsc;
      (void)Ms;
      T* dr = static_cast<T*>(p.dx) + r * p.ld;
      const float nML = -sc.M * L2E;
      for (int v0 = tid; v0 < nvec; v0 += U * kRowThreads) {
        float x[U][VN];
        if (sc.active != 0.f) {
#pragma unroll
          for (int u = 0; u < U; ++u)  // U loads in flight (L2: the row was just read)
            if (v0 + u * kRowThreads < nvec) RowVec<T>::load(xr, v0 + u * kRowThreads, x[u], pol_last);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int v = v0 + u * kRowThreads;
          if (v >= nvec) break;
          float d[VN];
          if (sc.active != 0.f) {
#pragma unroll
            for (int j = 0; j < VN; ++j) {
              const float t = clamp_ninf(fmaf(x[u][j], L2E, nML));
              d[j] = ex2(t) * fmaf(sc.k2, t, sc.k1);
            }
            if (v == va) d[a - va * VN] = sc.ga;
          } else {
#pragma unroll
            for (int j = 0; j < VN; ++j) d[j] = 0.f;
          }
          RowVec<T>::store(dr, v, d);
        }
      }
    }
    __syncthreads();  // red / rsc reuse across rows
  }
  if (want_stats) {
    __syncthreads();
    finish_loss_stats(sacc, p.stats, p.partials, p.ctrl, Nden, p.accumulate, pc.ent_coef, &p.p2p);
  }
}

Lp make_lp(const LpArgs& a) {
  Lp p{};
  p.x = a.x.ptr;
  p.rows = a.x.rows;
  p.V = a.x.vocab;
  p.ld = a.x.ld;
  p.target = a.target;
  p.logp = a.logp;
  p.lse_out = a.grad_logp ? nullptr : a.lse;
  p.lse_in = a.grad_logp ? a.lse : nullptr;
  p.g_in = a.grad_logp;
  p.dx = a.dlogits;
  p.stats = a.stats;
  p.p2p = a.ws.p2p;
  p.partials = a.ws.partials;
  p.ctrl = a.ws.ctrl + CTRL_LOGPROB;
  if (a.fused) {
    p.lpb = a.f.logp_behav;
    p.lpp = a.f.logp_prox;
    p.lref = (a.f.logp_ref != nullptr && a.f.kl_coef != 0.f) ? a.f.logp_ref : nullptr;
    p.adv = a.f.adv;
    p.ver = a.f.version;
    p.key = a.f.slot_key;
    p.A = a.f.a_tok;
    p.pc.has_prox = a.f.logp_prox != nullptr;
    p.pc.has_ref = p.lref != nullptr;
    p.pc.cur_version = a.f.cur_version;
    p.pc.eta = a.f.max_staleness;
    p.pc.lo = 1.f - a.f.eps_low;
    p.pc.hi = 1.f + a.f.eps_high;
    p.pc.is_cap = a.f.is_cap;
    p.pc.dual_clip = a.f.dual_clip;
    p.pc.kl_coef = a.f.kl_coef;
    p.pc.ent_coef = a.f.ent_coef;
    p.out_g = a.f.out_grad_logp;
    p.out_L = a.f.out_loss_tok;
    p.accumulate = a.f.accumulate;
    p.N = a.f.tok_denominator;
    p.adv_stats = a.f.adv_stats;
  }
  return p;
}

template <int MODE>
cudaError_t launch_mode(const LpArgs& a, Lp p, cudaStream_t s) {
  const LpPath path = select_lp_path(a);
  const int sms = device_info().sm_count;
  const int64_t R = a.x.rows;
  if (R <= 0) return cudaSuccess;
  if (path == LP_PATH_TMA) {
    const uint32_t row_bytes = uint32_t(a.x.vocab) * 2u;
    const uint32_t stage_bytes = (row_bytes + 127u) & ~127u;
    const size_t fixed = kMaxStages * sizeof(StageMeta) + kMaxStages * 8 +
                         4 * kGroupWarps * sizeof(float4) + 2 * sizeof(RowScalars) +
                         4 * sizeof(float) + 32 * sizeof(double);
    int nst = int((size_t(device_info().smem_optin) - fixed - 2048) / stage_bytes);
    if (nst > kMaxStages) nst = kMaxStages;
    if (nst < 2) return cudaErrorInvalidConfiguration;
    const size_t smem = size_t(nst) * stage_bytes + fixed;
    // dynamic smem limit = opt-in max minus the kernel's static smem
    const bool xp = MODE == MODE_FUSED && a.f.ent_coef != 0.f && a.dlogits != nullptr;
    const int nvec = a.x.vocab >> 3;
    // V > 28672 (OpenVLA 32000): 7 unchecked vectors
    const bool f7 = nvec / kGroupThreads >= 7 && (MODE != MODE_FUSED || RLVLA_NFULL_FUSED);
    const bool dx = MODE == MODE_FUSED && a.dlogits != nullptr;
    // kernel instance: [xp][f7][dx]
    using Fn = void (*)(Lp, int, uint32_t);
    constexpr bool kDx = MODE != MODE_FWD;  // FWD never writes dlogits
    Fn fns[2][2][2] = {{{lp_tma_kernel<MODE, false, 0, false>, lp_tma_kernel<MODE, false, 0, kDx>},
                        {lp_tma_kernel<MODE, false, 7, false>, lp_tma_kernel<MODE, false, 7, kDx>}},
                       {{lp_tma_kernel<MODE, true, 0, false>, lp_tma_kernel<MODE, true, 0, kDx>},
                        {lp_tma_kernel<MODE, true, 7, false>, lp_tma_kernel<MODE, true, 7, kDx>}}};
    const Fn kern = fns[xp][f7][MODE == MODE_BWD ? 1 : (dx ? 1 : 0)];
    const void* fn = reinterpret_cast<const void*>(kern);
    // the opt-in SMEM limit is a per-device function attribute: cached per device
    static int attr_dyn[kMaxDevices][3][2][2][2] = {};
    const int dev = device_info().device;
    int dummy = 0;
    int& cached = (dev >= 0 && dev < kMaxDevices) ? attr_dyn[dev][MODE][xp][f7][dx] : dummy;
    if (cached < int(smem)) {
      cudaFuncAttributes fa{};
      cudaError_t e = cudaFuncGetAttributes(&fa, fn);
      if (e != cudaSuccess) return e;
      if (smem + fa.sharedSizeBytes > size_t(device_info().smem_optin)) return cudaErrorInvalidConfiguration;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
      cached = int(smem);
    }
    const int psms = persistent_sms();
    int grid = int(R < psms ? R : psms);
    kern<<<grid, kCtaThreads, smem, s>>>(p, nst, stage_bytes);
    return cudaGetLastError();
  }
  if (path == LP_PATH_WARP) {
    const int VW = a.x.dtype == RLVLA_BF16 ? 8 : 4;
    const int nv = (a.x.vocab / VW + 31) / 32;  // vectors per lane
    int64_t blocks = (R + 7) / 8;
    const int64_t cap = int64_t(sms) * 8;
    if (blocks > cap) blocks = cap;
    const int g = int(blocks);
    if (a.x.dtype == RLVLA_BF16) {
      if (nv <= 1) lp_warp_kernel<__nv_bfloat16, 1, MODE><<<g, 256, 0, s>>>(p);
      else if (nv <= 4) lp_warp_kernel<__nv_bfloat16, 4, MODE><<<g, 256, 0, s>>>(p);
      else lp_warp_kernel<__nv_bfloat16, 8, MODE><<<g, 256, 0, s>>>(p);
    } else {
      if (nv <= 2) lp_warp_kernel<float, 2, MODE><<<g, 256, 0, s>>>(p);
      else if (nv <= 4) lp_warp_kernel<float, 4, MODE><<<g, 256, 0, s>>>(p);
      else lp_warp_kernel<float, 8, MODE><<<g, 256, 0, s>>>(p);
    }
    return cudaGetLastError();
  }
  if (path == LP_PATH_ROW) {
    int64_t blocks = R;
    const int64_t cap = int64_t(sms) * RLVLA_ROW_MINB;
    if (blocks > cap) blocks = cap;
    if (a.x.dtype == RLVLA_BF16) lp_row_kernel<__nv_bfloat16, MODE><<<int(blocks), kRowThreads, 0, s>>>(p);
    else lp_row_kernel<float, MODE><<<int(blocks), kRowThreads, 0, s>>>(p);
    return cudaGetLastError();
  }
  int64_t blocks = R;
  const int64_t cap = int64_t(sms) * 8;
  if (blocks > cap) blocks = cap;
  if (a.x.dtype == RLVLA_BF16) lp_generic_kernel<__nv_bfloat16, MODE><<<int(blocks), 256, 0, s>>>(p);
  else lp_generic_kernel<float, MODE><<<int(blocks), 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

LpPath select_lp_path(const LpArgs& a) {
  const int V = a.x.vocab;
  const int VW = a.x.dtype == RLVLA_BF16 ? 8 : 4;
  const uintptr_t xp = reinterpret_cast<uintptr_t>(a.x.ptr);
  const uintptr_t dp = reinterpret_cast<uintptr_t>(a.dlogits);
  const bool aligned = (xp % 16 == 0) && (dp % 16 == 0) && (V % VW == 0) && (a.x.ld % VW == 0);
  if (!aligned) return LP_PATH_GENERIC;
  if (V <= 32 * 8 * VW && V / VW <= 256) return LP_PATH_WARP;
  if (a.x.dtype == RLVLA_BF16 && V <= kGroupThreads * kVecPerThread * 8 && a.x.rows < (int64_t(1) << 31))
    return LP_PATH_TMA;
  return LP_PATH_ROW;
}

cudaError_t launch_logprob(const LpArgs& a, cudaStream_t s) {
  const Lp p = make_lp(a);
  if (a.fused) return launch_mode<MODE_FUSED>(a, p, s);
  if (a.grad_logp) return launch_mode<MODE_BWD>(a, p, s);
  return launch_mode<MODE_FWD>(a, p, s);
}

}  // namespace rlvla
