// internal.cuh — device helpers and launch declarations shared by the librlvla kernels.
// Nothing here is shared with oracle/ (the CPU reference is numpy).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "rlvla.h"

namespace rlvla {

constexpr int kMaxPartialBlocks = 2048;          // per-CTA fp64 partial rows in workspace
constexpr size_t kCtrlBytes = 256;               // control words (last-block counters)
constexpr size_t kPartialBytes = size_t(kMaxPartialBlocks) * RLVLA_NSTATS * sizeof(double);
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// control-word indices (uint32 each) inside the workspace header
enum { CTRL_SCATTER = 0, CTRL_ADV = 1, CTRL_LOGPROB = 2, CTRL_PPO = 3, CTRL_ADV2 = 4, CTRL_VALUE = 5,
       CTRL_BOFFER = 6, CTRL_BPOLL = 7, CTRL_FLOW = 8 };
// ctrl words 32..35 hold two doubles of per-call scratch (chunk-ratio and value-loss 1/N)

// ------------------------------------------------------------------------------------
// In-kernel cross-rank reduction over NVLink peer memory (SURVEY §8(e) "Phase 4"): the
// last CTA of a statistics kernel pushes its slots into every rank's mailbox (P2P stores,
// CUDA IPC-mapped), raises a release flag there, waits for every rank's flag in its own
// mailbox and sums the ranks in fixed order — the compute step and its collective in ONE
// kernel, no NCCL launch. Mailbox per rank: kP2PChannels channels of
//   data[2 parity][kP2PMaxRanks][kP2PSlots] f64, flags[2 parity][kP2PMaxRanks] u64
// A call's sequence number s (a per-rank device counter per channel, identical on every
// rank because calls are made in the same order) selects parity s & 1: a rank can be at
// most one call ahead of any other on a channel, so two buffers suffice.
constexpr int kP2PMaxRanks = 8;
constexpr int kP2PSlots = 32;
constexpr int kP2PChannels = 4;
enum { P2P_CH_LOSS = 0, P2P_CH_ADV = 1, P2P_CH_VALUE = 2 };
constexpr size_t kP2PChanData = size_t(2) * kP2PMaxRanks * kP2PSlots * sizeof(double);
constexpr size_t kP2PChanBytes = kP2PChanData + size_t(2) * kP2PMaxRanks * sizeof(unsigned long long);
// gather region (C2: GRPO returns of all ranks), [2 parity][kP2PMaxEnvGlobal] f32
constexpr int kP2PMaxEnvGlobal = 32768;
constexpr size_t kP2PGatherOffset = kP2PChannels * kP2PChanBytes;
constexpr size_t kP2PMboxBytes = kP2PGatherOffset + size_t(2) * kP2PMaxEnvGlobal * sizeof(float);

struct P2PDesc {
  int nranks = 0;  // 0 or 1: no exchange
  int rank = 0;
  int ch = 0;
  uint8_t* mbox[kP2PMaxRanks] = {};  // every rank's mailbox mapped here (mbox[rank]: own)
  unsigned long long* seq = nullptr;  // own per-channel call counters
};

struct Workspace {
  unsigned* ctrl;      // [64]
  double* partials;    // [kMaxPartialBlocks][RLVLA_NSTATS]
  float* r_global;     // [n_env_global] (GRPO returns)
  P2PDesc p2p;         // set by the API when the call reduces over ranks in-kernel
};

inline Workspace carve(void* ws) {
  Workspace w{};
  uint8_t* b = static_cast<uint8_t*>(ws);
  w.ctrl = reinterpret_cast<unsigned*>(b);
  w.partials = reinterpret_cast<double*>(b + kCtrlBytes);
  w.r_global = reinterpret_cast<float*>(b + kCtrlBytes + kPartialBytes);
  return w;
}

// ------------------------------------------------------------------------------------
// device helpers
// ------------------------------------------------------------------------------------
// warp max in one instruction (sm_100a redux.sync .f32 -> CREDUX.MAX.F32); without .NaN
// a NaN input is ignored like fmaxf's
__device__ __forceinline__ float warp_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
// sum over lanes 0..15 (xor tree within each half-warp: the result is valid in lanes 0..15)
__device__ __forceinline__ float half_warp_sum(float v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 2^x on the MUFU (ex2.approx.ftz.f32): one SFU op per call.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// bf16 pair (one 32-bit word) -> two fp32, exact (bf16 = top half of fp32)
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
// two fp32 -> bf16x2 word, round to nearest even (cvt.rn.bf16x2.f32)
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// packed bf16x2 max (one HMNMX2 per pair); NaN inputs are dropped here and propagate
// through the exponent sums instead (reading R5).
__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
  __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a);
  __nv_bfloat162 y = *reinterpret_cast<__nv_bfloat162*>(&b);
  __nv_bfloat162 z = __hmax2(x, y);
  return *reinterpret_cast<uint32_t*>(&z);
}

// packed bf16x2 max that propagates NaN (HMNMX2.NAN)
// packed bf16x2 products with one rounding each (HMUL2 / HFMA2 .BF16): a*b, a*b + c
__device__ __forceinline__ uint32_t bmul2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t bfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t bmax2_nan(uint32_t a, uint32_t b) {
  __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a);
  __nv_bfloat162 y = *reinterpret_cast<__nv_bfloat162*>(&b);
  __nv_bfloat162 z = __hmax2_nan(x, y);
  return *reinterpret_cast<uint32_t*>(&z);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mbarrier / bulk-async-copy (TMA engine) wrappers, sm_90+ PTX (SASS: SYNCS.*, UBLKCP)
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: the waiting thread sleeps in the barrier unit until
// the phase completes (or the hint, in ns, expires) instead of re-issuing polls that take
// issue slots from the warps that have work
#ifndef RLVLA_MBAR_HINT_NS
#define RLVLA_MBAR_HINT_NS 1000000
#endif
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
#if RLVLA_MBAR_HINT_NS > 0
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(RLVLA_MBAR_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#endif
  return ok != 0u;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t n = 0;
  // a phase that never completes traps after ~16 s (hinted waits) instead of hanging the GPU
  while (!mbar_try_wait(bar, parity)) {
    if (++n > (RLVLA_MBAR_HINT_NS > 0 ? (1u << 14) : (1u << 20))) __trap();
  }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D bulk copy global -> shared, completion counted on `bar` in bytes
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// 1-D bulk copy shared -> global (TMA store), tracked in the issuing thread's bulk group
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
      "r"(smem_u32(src)), "r"(bytes), "l"(pol)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// this thread's bulk stores have finished READING their SMEM source (it may be refilled)
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// ... and have completed their global writes
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// bulk prefetch of global memory into L2 (no SMEM destination, no completion to wait for)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// small async copies (LDGSTS) whose completion arrives on an mbarrier (noinc)
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 16-byte load with an L2 eviction-policy hint (L1 not allocated)
__device__ __forceinline__ uint4 ldg_hint(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// Last-block-done finalize: each CTA has written partials[blockIdx.x][0..nslot); the
// last CTA to arrive sums them in fixed CTA order (deterministic, no float atomics) and
// returns true in every thread of that CTA. Caller uses `out` (per-slot total) then.
__device__ __forceinline__ bool last_block_reduce(unsigned* ctrl_word, const double* partials,
                                                  int nslot, double* out_smem) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev = atomicAdd(ctrl_word, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  // one warp per slot: lane l sums CTAs l, l + 32, ... in order (8 loads in flight), then a
  // fixed xor tree — deterministic for a given grid, and G/32 dependent steps instead of G
  const int lane = threadIdx.x & 31, nw = int(blockDim.x >> 5);
  for (int s = int(threadIdx.x >> 5); s < nslot; s += nw) {
    double acc = 0.0;
#pragma unroll 8
    for (unsigned b = lane; b < gridDim.x; b += 32) acc += __ldcg(partials + size_t(b) * RLVLA_NSTATS + s);
    acc = warp_sum_d(acc);
    if (lane == 0) out_smem[s] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ctrl_word = 0u;  // leave the workspace reusable
  return true;
}

// Sum vals[0..n) (SMEM, n <= kP2PSlots) over the ranks of d, in place; optionally also
// allgather a float slice: this rank's gsrc[0..glen) lands at [goff, goff + glen) of gdst
// [0..gtotal) on every rank (gtotal <= kP2PMaxEnvGlobal). Called by every thread of ONE CTA
// (the last of its grid). One flag per rank covers both. See P2PDesc.
__device__ __forceinline__ void p2p_exchange(double* vals, int n, const P2PDesc& d,
                                             const float* gsrc = nullptr, int goff = 0, int glen = 0,
                                             float* gdst = nullptr, int gtotal = 0) {
  __shared__ unsigned long long s_seq;
  if (threadIdx.x == 0) {
    s_seq = d.seq[d.ch] + 1ull;
    d.seq[d.ch] = s_seq;
  }
  __syncthreads();
  const unsigned long long sq = s_seq;
  const int par = int(sq & 1ull);
  const size_t dofs = size_t(d.ch) * kP2PChanBytes;
  const size_t gofs = kP2PGatherOffset + size_t(par) * kP2PMaxEnvGlobal * sizeof(float);
  // 1) my slots (and my slice) into every rank's mailbox (NVLink stores to peers)
  for (int i = threadIdx.x; i < d.nranks * n; i += blockDim.x) {
    const int pr = i / n, k = i - pr * n;
    double* dst = reinterpret_cast<double*>(d.mbox[pr] + dofs) + (par * kP2PMaxRanks + d.rank) * kP2PSlots + k;
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(dst), "d"(vals[k]) : "memory");
  }
  for (int i = threadIdx.x; i < d.nranks * glen; i += blockDim.x) {
    const int pr = i / glen, k = i - pr * glen;
    float* dst = reinterpret_cast<float*>(d.mbox[pr] + gofs) + goff + k;
    asm volatile("st.relaxed.sys.global.f32 [%0], %1;" ::"l"(dst), "f"(__ldcg(gsrc + k)) : "memory");
  }
  __threadfence_system();
  __syncthreads();
  // 2) raise my flag at every rank (release: the data above is visible first)
  if (threadIdx.x < d.nranks) {
    unsigned long long* f = reinterpret_cast<unsigned long long*>(d.mbox[threadIdx.x] + dofs + kP2PChanData) +
                            par * kP2PMaxRanks + d.rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(sq) : "memory");
  }
  // 3) wait for every rank's flag in my mailbox
  if (threadIdx.x < d.nranks) {
    const unsigned long long* f =
        reinterpret_cast<const unsigned long long*>(d.mbox[d.rank] + dofs + kP2PChanData) + par * kP2PMaxRanks +
        threadIdx.x;
    unsigned long long v;
    uint32_t it = 0;
    do {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      // a rank never arrived (crashed, or calls out of order): fail loudly after ~2^27 polls
      // (about a minute) instead of hanging the GPU
      if (++it > (1u << 27)) __trap();
    } while (v != sq);
  }
  __syncthreads();
  // 4) fixed rank order sum; the gathered slices copied out
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double* src = reinterpret_cast<const double*>(d.mbox[d.rank] + dofs) + par * kP2PMaxRanks * kP2PSlots + k;
    double acc = 0.0;
    for (int r = 0; r < d.nranks; ++r) {
      double v;
      asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(src + r * kP2PSlots) : "memory");
      acc += v;
    }
    vals[k] = acc;
  }
  for (int k = threadIdx.x; k < gtotal; k += blockDim.x) {
    float v;
    asm volatile("ld.relaxed.sys.global.f32 %0, [%1];"
                 : "=f"(v)
                 : "l"(reinterpret_cast<const float*>(d.mbox[d.rank] + gofs) + k)
                 : "memory");
    gdst[k] = v;
  }
  __syncthreads();
}
__device__ __forceinline__ void p2p_allreduce(double* vals, int n, const P2PDesc& d) { p2p_exchange(vals, n, d); }

// ------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------
constexpr int kMaxDevices = 64;  // per-device host caches
struct DeviceInfo {
  int device = -1;
  int sm_count = 0;
  int smem_optin = 0;
};
const DeviceInfo& device_info();          // cached per device (thread-safe)
// SMs the persistent (grid-stride, one-CTA-per-SM) kernels leave free for concurrent work on
// other streams (rlvla_set_reserved_sms); their grid is sm_count - reserved (>= 1)
int persistent_sms();
bool sync_check_enabled();

// launches (return cudaError_t of the launch)
struct ScatterArgs {
  rlvla_traj_buffer buf;
  rlvla_step_batch rec;
  int32_t cur_version;
  uint64_t seq_base;
  int64_t* counters;
};
cudaError_t launch_scatter(const ScatterArgs& a, cudaStream_t s);

struct AdvArgs {
  rlvla_traj_buffer buf;
  const float* last_value;
  rlvla_adv_params p;
  float* adv;
  float* ret;
  double* stats;
  Workspace ws;
};
cudaError_t launch_adv_pass1(const AdvArgs& a, cudaStream_t s);   // GAE scan | GRPO returns
cudaError_t launch_adv_pass2(const AdvArgs& a, cudaStream_t s);   // whiten | GRPO normalise

struct LpArgs {
  rlvla_logits x;
  const int32_t* target;
  float* logp;
  float* lse;
  const float* grad_logp;
  bool fused;
  rlvla_ppo_args f;
  void* dlogits;
  double* stats;
  Workspace ws;
};
enum LpPath { LP_PATH_TMA = 0, LP_PATH_WARP = 1, LP_PATH_GENERIC = 2, LP_PATH_ROW = 3 };
LpPath select_lp_path(const LpArgs& a);
cudaError_t launch_logprob(const LpArgs& a, cudaStream_t s);

struct PpoArgs {
  const float* logp;
  int64_t rows;
  const int32_t* target;
  rlvla_ppo_args f;
  float* grad_logp;
  float* loss_tok;
  double* stats;
  Workspace ws;
  int defer;  // chunk path, implicit N over NCCL: raw sums out, scale after the allreduce
};
cudaError_t launch_ppo_loss(const PpoArgs& a, cudaStream_t s);
cudaError_t launch_ppo_chunk_scale(const PpoArgs& a, cudaStream_t s);

struct ValueArgs {
  const float* v_new;
  const float* v_old;
  const float* ret;
  const uint64_t* slot_key;
  const int32_t* version;
  int64_t n;
  int32_t cur_version, max_staleness;
  float clip_eps;
  double denominator;
  float* grad_v;
  float* loss_step;
  double* stats;
  Workspace ws;
  int defer;  // implicit N_v over NCCL: raw sums out, scale after the allreduce
};
cudaError_t launch_value_loss(const ValueArgs& a, cudaStream_t s);
cudaError_t launch_value_scale(const ValueArgs& a, cudaStream_t s);

struct BatchOfferArgs {
  rlvla_batch_queue q;
  const int32_t* env_id;
  const int64_t* enqueue_time;
  int32_t n;
  int64_t now;
  const uint8_t* obs_src;
  int64_t* counters;
  Workspace ws;
};
struct BatchPollArgs {
  rlvla_batch_queue q;
  int64_t now;
  int32_t b_max;
  int64_t t_max;
  int32_t* out_env;
  int64_t* out_time;
  uint8_t* out_obs;
  int32_t* out_n;
  Workspace ws;
};
constexpr int kMaxOffer = 1024;

struct FlowArgs {
  rlvla_gauss_chain c;
  float* logp;
  const float* grad_logp;
  int fused;
  rlvla_ppo_args f;
  void* dmu;
  float* dlog_std;
  double* stats;
  Workspace ws;
};
constexpr int kFlowMaxElems = 4096;
cudaError_t launch_flow(const FlowArgs& a, cudaStream_t s);
cudaError_t launch_batch_offer(const BatchOfferArgs& a, cudaStream_t s);
cudaError_t launch_batch_poll(const BatchPollArgs& a, cudaStream_t s);

}  // namespace rlvla
