// scatter.cu — S1: out-of-order step records -> trajectory buffer (K1a claim, K1b write).
//
// Paper: trajectories carry their policy version (§3.1); requests from subsets of
// envs arrive early / out of order (§3.2); samples accumulate in the trajectory
// buffer (§3.3). Reading R6: sequential-replay semantics with
// key = (version << 40) | seq, newest key wins, every extra arrival is a duplicate.
//
// GPU formulation (thread-order independent, hence bit-exact vs the replay):
//   claim: one thread per record; u64 atomicMax(slot_key, key) returns the previous key.
//          Exactly one valid record per slot per call observes the pre-call key, so
//          written = #(old == 0) and dup = #(old != 0) match the replay counts.
//   write: after all claims, a record whose key equals the slot's final key is the unique
//          winner and copies its payload (one warp per record, coalesced over a_tok).
// M <= 1024 (an Eq. (1) arrival chunk, B_max = 64 in the paper's setting) runs as one
// CTA (claim, __syncthreads, write) — one launch; larger M uses two grid launches.
#include "internal.cuh"

namespace rlvla {
namespace {

constexpr int kVersionShift = 40;
#ifndef RLVLA_SCATTER_EPT
#define RLVLA_SCATTER_EPT 4  // payload elements per thread of the one-CTA path (A/B)
#endif
// (Measured and rejected: deciding winners in SMEM from atomicMax's return value instead of
// re-reading the key — 4.6 -> 6.5 us per 64-record call.)
#ifndef RLVLA_SCATTER_PDL
#define RLVLA_SCATTER_PDL 1  // programmatic dependent launch between arrival chunks (A/B)
#endif

struct Claim {
  int valid;
  uint64_t key;
  int64_t slot;
};

struct RecHead {
  int e, t, v;
};
__device__ __forceinline__ RecHead load_head(const ScatterArgs& a, int i) {
  return RecHead{a.rec.env_id[i], a.rec.step[i], a.rec.version[i]};
}

__device__ __forceinline__ Claim claim_head(const ScatterArgs& a, int i, RecHead h, long long cnt[4],
                                            unsigned long long* old_out) {
  Claim c{0, 0, 0};
  const int e = h.e, t = h.t, v = h.v;
  if (e < 0 || e >= a.buf.n_env || t < 0 || t >= a.buf.t_steps) {
    cnt[RLVLA_CNT_OOB] += 1;
    return c;
  }
  if (v < 0 || v > a.cur_version) {
    cnt[RLVLA_CNT_BAD_VERSION] += 1;
    return c;
  }
  c.slot = int64_t(e) * a.buf.t_steps + t;
  c.key = (uint64_t(uint32_t(v)) << kVersionShift) | (a.seq_base + uint64_t(i));
  unsigned long long old = atomicMax(reinterpret_cast<unsigned long long*>(a.buf.slot_key + c.slot),
                                     static_cast<unsigned long long>(c.key));
  if (old_out) *old_out = old;
  if (old != 0ull) cnt[RLVLA_CNT_DUP] += 1;
  else cnt[RLVLA_CNT_WRITTEN] += 1;
  c.valid = 1;
  return c;
}

// claim_head in two halves: the range / version checks (record-only) and the atomic
__device__ __forceinline__ Claim check_head(const ScatterArgs& a, int i, RecHead h, long long cnt[4]) {
  Claim c{0, 0, 0};
  if (h.e < 0 || h.e >= a.buf.n_env || h.t < 0 || h.t >= a.buf.t_steps) {
    cnt[RLVLA_CNT_OOB] += 1;
    return c;
  }
  if (h.v < 0 || h.v > a.cur_version) {
    cnt[RLVLA_CNT_BAD_VERSION] += 1;
    return c;
  }
  c.slot = int64_t(h.e) * a.buf.t_steps + h.t;
  c.key = (uint64_t(uint32_t(h.v)) << kVersionShift) | (a.seq_base + uint64_t(i));
  c.valid = 1;
  return c;
}
__device__ __forceinline__ unsigned long long claim_slot(const ScatterArgs& a, const Claim& c,
                                                         long long cnt[4]) {
  const unsigned long long old = atomicMax(reinterpret_cast<unsigned long long*>(a.buf.slot_key + c.slot),
                                           static_cast<unsigned long long>(c.key));
  cnt[old != 0ull ? RLVLA_CNT_DUP : RLVLA_CNT_WRITTEN] += 1;
  return old;
}

__device__ __forceinline__ Claim claim_one(const ScatterArgs& a, int i, long long cnt[4]) {
  return claim_head(a, i, load_head(a, i), cnt, nullptr);
}

// warp-cooperative payload copy of record i into slot (winner only)
__device__ __forceinline__ void write_payload(const ScatterArgs& a, int i, int64_t slot, int lane) {
  const int A = a.buf.a_tok;
  if (lane == 0) {
    a.buf.reward[slot] = a.rec.reward[i];
    a.buf.done[slot] = a.rec.done[i];
    a.buf.value[slot] = a.rec.value[i];
    a.buf.version[slot] = a.rec.version[i];
  }
  const int32_t* st = a.rec.tokens + int64_t(i) * A;
  const float* sl = a.rec.logp_behav + int64_t(i) * A;
  int32_t* dt = a.buf.tokens + slot * A;
  float* dl = a.buf.logp_behav + slot * A;
  for (int j = lane; j < A; j += 32) {
    dt[j] = st[j];
    dl[j] = sl[j];
  }
}

__device__ __forceinline__ void block_add_counters(long long cnt[4], int64_t* counters) {
  __shared__ long long red[32][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 4; ++k) cnt[k] = warp_sum_ll(cnt[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 4; ++k) red[warp][k] = cnt[k];
  __syncthreads();
  if (threadIdx.x < 4) {
    long long s = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    if (s) atomicAdd(reinterpret_cast<unsigned long long*>(counters + threadIdx.x),
                     static_cast<unsigned long long>(s));
  }
}

// M <= 1024: claim + write in one CTA. Everything that depends only on the records — each
// record's head (env, step, version) and header (reward, done, value), the first payload
// elements — is loaded before griddepcontrol.wait, so after it the critical path is the claim
// (one atomic round trip), the key re-read (one round trip) and the stores. The counters go
// through warp redux + one shared atomic per warp and leave as 4 REDs right after the claims
// (per-thread 64-bit shared atomics on one address serialise: 4.2 us per call). The payload copy is element-parallel over all (record, token) pairs, 16-byte
// quads when A % 4 == 0 and the arrays are 16-byte aligned.
#ifndef RLVLA_SCATTER_STOP
#define RLVLA_SCATTER_STOP 0  // latency breakdown (A/B only): 1 return after the PDL wait, 2 after the claims
#endif
#ifndef RLVLA_SCATTER_SCAN_MAX
#define RLVLA_SCATTER_SCAN_MAX 256  // calls of up to this many records decide winners by the scan
#endif
__global__ void __launch_bounds__(1024) scatter_fused_kernel(ScatterArgs a) {
  __shared__ long long s_slot[1024];  // the record's slot (-1: invalid), then its winner slot
  __shared__ unsigned long long s_key[1024];
  __shared__ unsigned s_cnt[4];
  const int i = threadIdx.x;
  const int M = a.rec.n_rec;
  const int A = a.buf.a_tok;
  const int n = M * A;
  const int32_t* __restrict__ src_t = a.rec.tokens;
  const float* __restrict__ src_l = a.rec.logp_behav;
  const bool vec = (A & 3) == 0 &&
                   ((reinterpret_cast<uintptr_t>(src_t) | reinterpret_cast<uintptr_t>(src_l) |
                     reinterpret_cast<uintptr_t>(a.buf.tokens) |
                     reinterpret_cast<uintptr_t>(a.buf.logp_behav)) & 15) == 0;
  const int nq = vec ? n >> 2 : n;  // copy units: quads or elements
  const int QA = A >> 2;
  if (i < 4) s_cnt[i] = 0u;
  // Programmatic dependent launch: let the next arrival chunk's kernel start launching now;
  // it waits (griddepcontrol.wait) before touching the buffer, so chunk order is kept.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  RecHead h{0, 0, 0};
  float rw = 0.f, vl = 0.f;
  uint8_t dn = 0;
  if (i < M) {
    h = load_head(a, i);
    rw = a.rec.reward[i];
    dn = a.rec.done[i];
    vl = a.rec.value[i];
  }
  int4 tq[2], lq[2];  // vec: this thread's first two quads of tokens / logp_behav
  int32_t tv[4];      // scalar: its first four elements
  float lv[4];
  if (vec) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = u * int(blockDim.x) + i;
      if (j < nq) {
        tq[u] = __ldg(reinterpret_cast<const int4*>(src_t) + j);
        lq[u] = __ldg(reinterpret_cast<const int4*>(src_l) + j);
      }
    }
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = u * int(blockDim.x) + i;
      if (j < n) {
        tv[u] = __ldg(src_t + j);
        lv[u] = __ldg(src_l + j);
      }
    }
  }
  // Small calls: whether a later record of this call supersedes this one (same slot, larger
  // key) depends only on the records, so it is settled here, before the wait — overlapping the
  // previous chunk's kernel — and the claim's returned key then decides the winner without
  // re-reading the slot: win <=> valid, not superseded, and old < key (chunks are ordered, so
  // `old` is the pre-call key or a smaller key of this call).
  const bool scan = M <= RLVLA_SCATTER_SCAN_MAX;
  long long cnt[4] = {0, 0, 0, 0};
  Claim c{0, 0, 0};
  if (i < M) c = check_head(a, i, h, cnt);
  if (scan && i < M) {
    s_slot[i] = c.valid ? c.slot : -1;
    s_key[i] = c.key;
  }
  __syncthreads();  // s_cnt zeroed, the call's (slot, key) table written
  bool superseded = false;
  if (scan && c.valid)
    for (int j = 0; j < M; ++j)
      if (s_slot[j] == c.slot && s_key[j] > c.key) {
        superseded = true;
        break;
      }
  // the records are inputs; the buffer may still be written by the previous chunk's kernel
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if RLVLA_SCATTER_STOP == 1
  return;
#endif
  unsigned long long old = 0ull;
  if (c.valid) old = claim_slot(a, c, cnt);
  // warp totals by redux.sync, one 32-bit shared atomic per warp and counter (M <= 1024)
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const unsigned w = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(cnt[k]));
    if ((i & 31) == 0 && w) atomicAdd(&s_cnt[k], w);
  }
  __syncthreads();  // all claims (device-scope atomics) and counts of this CTA are done
#if RLVLA_SCATTER_STOP == 2
  return;
#endif
  if (i < 4 && s_cnt[i])
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + i), static_cast<unsigned long long>(s_cnt[i]));
  if (i < M) {
    const bool win =
        c.valid && (scan ? !superseded && old < c.key
                         : __ldcg(reinterpret_cast<const unsigned long long*>(a.buf.slot_key + c.slot)) == c.key);
    s_slot[i] = win ? c.slot : -1;
    if (win) {
      a.buf.reward[c.slot] = rw;
      a.buf.done[c.slot] = dn;
      a.buf.value[c.slot] = vl;
      a.buf.version[c.slot] = h.v;
    }
  }
  __syncthreads();
  if (vec) {
    int4* dst_t = reinterpret_cast<int4*>(a.buf.tokens);
    int4* dst_l = reinterpret_cast<int4*>(a.buf.logp_behav);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = u * int(blockDim.x) + i;
      if (j < nq) {
        const int r = j / QA;
        const long long slot = s_slot[r];
        if (slot >= 0) {
          const long long d = slot * QA + (j - r * QA);
          dst_t[d] = tq[u];
          dst_l[d] = lq[u];
        }
      }
    }
    for (int j = 2 * int(blockDim.x) + i; j < nq; j += int(blockDim.x)) {  // M A > 8 blockDim
      const int r = j / QA;
      const long long slot = s_slot[r];
      if (slot >= 0) {
        const long long d = slot * QA + (j - r * QA);
        dst_t[d] = __ldg(reinterpret_cast<const int4*>(src_t) + j);
        dst_l[d] = __ldg(reinterpret_cast<const int4*>(src_l) + j);
      }
    }
    return;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = u * int(blockDim.x) + i;
    if (j < n) {
      const int r = j / A;
      const long long slot = s_slot[r];
      if (slot >= 0) {
        const long long d = slot * A + (j - r * A);
        a.buf.tokens[d] = tv[u];
        a.buf.logp_behav[d] = lv[u];
      }
    }
  }
  // remaining elements (M * A > 4 * blockDim): loads batched before stores
  for (int base = 4 * int(blockDim.x); base < n; base += 4 * int(blockDim.x)) {
    long long dst[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = base + u * int(blockDim.x) + i;
      dst[u] = -1;
      if (j < n) {
        const int r = j / A;
        const long long slot = s_slot[r];
        if (slot >= 0) {
          dst[u] = slot * A + (j - r * A);
          tv[u] = __ldg(src_t + j);
          lv[u] = __ldg(src_l + j);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (dst[u] >= 0) {
        a.buf.tokens[dst[u]] = tv[u];
        a.buf.logp_behav[dst[u]] = lv[u];
      }
  }
}

__global__ void __launch_bounds__(256) scatter_claim_kernel(ScatterArgs a) {
  long long cnt[4] = {0, 0, 0, 0};
  const int M = a.rec.n_rec;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x)
    (void)claim_one(a, i, cnt);
  block_add_counters(cnt, a.counters);
}

__global__ void __launch_bounds__(256) scatter_write_kernel(ScatterArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = gw; r < a.rec.n_rec; r += nw) {
    const int e = a.rec.env_id[r], t = a.rec.step[r], v = a.rec.version[r];
    if (e < 0 || e >= a.buf.n_env || t < 0 || t >= a.buf.t_steps || v < 0 || v > a.cur_version)
      continue;
    const int64_t slot = int64_t(e) * a.buf.t_steps + t;
    const uint64_t key = (uint64_t(uint32_t(v)) << kVersionShift) | (a.seq_base + uint64_t(r));
    if (__ldcg(reinterpret_cast<const unsigned long long*>(a.buf.slot_key + slot)) == key)
      write_payload(a, r, slot, lane);
  }
}

}  // namespace

cudaError_t launch_scatter(const ScatterArgs& a, cudaStream_t s) {
  const int M = a.rec.n_rec;
  if (M <= 0) return cudaSuccess;
  if (M <= 1024) {
    const int64_t work = int64_t(M) * a.buf.a_tok;
    int threads = int((work + RLVLA_SCATTER_EPT - 1) / RLVLA_SCATTER_EPT + 31) / 32 * 32;
    const int need = ((M + 31) / 32) * 32;
    if (threads < need) threads = need;
    if (threads < 128) threads = 128;
    if (threads > 1024) threads = 1024;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(threads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = RLVLA_SCATTER_PDL ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, scatter_fused_kernel, a);
  }
  const int sms = device_info().sm_count;
  int blocks = (M + 255) / 256;
  if (blocks > 8 * sms) blocks = 8 * sms;
  scatter_claim_kernel<<<blocks, 256, 0, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int wblocks = (M + 7) / 8;
  if (wblocks > 16 * sms) wblocks = 16 * sms;
  scatter_write_kernel<<<wblocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace rlvla
