// batcher.cu — NEXT-3: the Dynamic Batching Scheduler of Eq. (1) on the device
// (§3.2; reading R24 = SPEC.md S:161-180).
//
// State (rlvla_batch_queue): a FIFO ring of pending (env, enqueue_time) in arrival order,
// a pending flag per env, and int64 head / tail / anchor / batch count. Both kernels read
// the state once at entry and only the LAST CTA to finish writes it back (done counter in
// the workspace control words), so every CTA sees the same pre-call state without a grid
// barrier:
//   batch_offer_kernel  one 1024-thread CTA per <= 1024 requests decides acceptance
//                       (range, enqueue_time <= now, not pending, first of its env in the
//                       call) and the FIFO positions (ballot prefix sum); with obs_src the
//                       grid (one CTA per SM) copies the accepted observations into their
//                       env slots (obs_fifo = 0) or their FIFO rows (obs_fifo = 1); the
//                       last CTA appends to the ring.
//   batch_poll_kernel   every CTA evaluates Eq. (1) from the same state; a poll that does
//                       not fire returns at once. Otherwise the b = min(p, B_max) oldest
//                       observations are gathered into the batch (FIFO rows: already in
//                       place, only a wrap is mirrored past n_env), the concatenated rows
//                       split evenly over one CTA per SM (128-bit loads/stores: one read
//                       + one write of b * obs_bytes, HBM-bound); the last CTA pops the
//                       ring. (Measured and rejected: TMA bulk copies through an SMEM ring,
//                       256-thread CTAs, 8 or 16 loads in flight per thread — equal or slower.)
#include "internal.cuh"

namespace rlvla {
namespace {

#ifndef RLVLA_POLL_THREADS
#define RLVLA_POLL_THREADS 1024  // threads per poll CTA; the grid keeps 1024 threads per SM
#endif
constexpr int kPollThreads = RLVLA_POLL_THREADS;
constexpr int kPollCtasPerSm = 1024 / kPollThreads;

#ifndef RLVLA_COPY_DEPTH
#define RLVLA_COPY_DEPTH 4  // 16-byte loads in flight per thread (A/B: 4 < 8 < 16 in time)
#endif

// copy n16 16-byte words with the whole CTA, RLVLA_COPY_DEPTH words in flight per thread
__device__ __forceinline__ void cta_copy16(uint4* d4, const uint4* s4, int64_t n16) {
  constexpr int U = RLVLA_COPY_DEPTH;
  const int64_t bd = blockDim.x;
  for (int64_t k = threadIdx.x; k < n16; k += U * bd) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u * bd < n16) v[u] = ldg_stream(s4 + k + u * bd);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u * bd < n16) d4[k + u * bd] = v[u];
  }
}

// Row copy dst_row(i) <- src_row(i), i < nrows, rows of ob16 16-byte words, spread evenly
// over the grid: CTA c takes words [c P, (c+1) P) of the concatenated rows (one pass,
// every SM busy; a range crosses at most a few row boundaries).
template <typename Dst, typename Src>
__device__ __forceinline__ void grid_copy_rows(int nrows, int64_t ob16, Dst dst_row, Src src_row) {
  const int64_t total = int64_t(nrows) * ob16;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t lo = int64_t(blockIdx.x) * per;
  const int64_t hi = lo + per < total ? lo + per : total;
  for (int64_t x = lo; x < hi;) {
    const int64_t row = x / ob16;
    const int64_t off = x - row * ob16;
    const int64_t end = (row + 1) * ob16 < hi ? (row + 1) * ob16 : hi;
    cta_copy16(dst_row(int(row)) + off, src_row(int(row)) + off, end - x);
    x = end;
  }
}

__device__ __forceinline__ bool cta_is_last(unsigned* ctrl_word) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) am_last = atomicAdd(ctrl_word, 1u) == gridDim.x - 1;
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

__global__ void __launch_bounds__(kMaxOffer) batch_offer_kernel(BatchOfferArgs a) {
  __shared__ int s_cand[kMaxOffer];  // env of a candidate request, else -1
  __shared__ int s_idx[kMaxOffer];   // FIFO position among accepted -> request index
  __shared__ int s_warp[kMaxOffer / 32];
  __shared__ int s_nacc;
  const int i = threadIdx.x, lane = i & 31, w = i >> 5;
  // 0 OOB, 1 FUTURE, 2 DUP, 3 ACCEPTED, -1 no request
  int code = -1, e = -1;
  int64_t t = 0;
  // programmatic dependent launch: the next call may start launching now; this one reads
  // its own inputs, then waits for the previous call (it may have changed the queue)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (i < a.n) {
    e = a.env_id[i];
    t = a.enqueue_time[i];
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // queue state and counters: only this kernel's last CTA writes them, so every CTA may
  // read them now, in parallel with the pending-flag loads below
  __shared__ int64_t s_state[2], s_cnt[4];
  if (i < 2) s_state[i] = a.q.state[i];
  else if (i < 6) s_cnt[i - 2] = a.counters[i - 2];
  if (i < a.n) {
    if (e < 0 || e >= a.q.n_env) code = 0;
    else if (t > a.now) code = 1;
    else if (a.q.pending[e]) code = 2;
    else code = 4;  // candidate: accepted iff it is the first candidate of its env
  }
  s_cand[i] = code == 4 ? e : -1;
  __syncthreads();
  if (code == 4) {
    bool first = true;
    for (int j = 0; j < i && first; ++j) first = s_cand[j] != e;
    code = first ? 3 : 2;
  }
  // FIFO positions of the accepted requests: ballot + warp-prefix over 32 warps
  const bool acc = code == 3;
  const unsigned bal = __ballot_sync(0xffffffffu, acc);
  const int wpre = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) s_warp[w] = __popc(bal);
  __syncthreads();
  if (w == 0) {
    const int v = s_warp[lane];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    s_warp[lane] = incl - v;
    if (lane == 31) s_nacc = incl;
  }
  __syncthreads();
  const int pos = s_warp[w] + wpre;
  if (acc) s_idx[pos] = i;
  __syncthreads();
  const int nacc = s_nacc;
  const int64_t ob = a.q.obs_bytes;
  if (a.obs_src != nullptr && ob > 0) {
    const int64_t ob16 = ob >> 4;
    uint4* slots = reinterpret_cast<uint4*>(a.q.obs);
    const uint4* src = reinterpret_cast<const uint4*>(a.obs_src);
    if (a.q.obs_fifo) {
      // FIFO rows: request k of this call lands at ring position tail + k
      const int64_t tail = s_state[1];
      const int cap = a.q.n_env;
      grid_copy_rows(
          nacc, ob16, [&](int k) { return slots + ((tail + k) % cap) * ob16; },
          [&](int k) { return src + int64_t(s_idx[k]) * ob16; });
    } else {
      grid_copy_rows(
          nacc, ob16, [&](int k) { return slots + int64_t(s_cand[s_idx[k]]) * ob16; },
          [&](int k) { return src + int64_t(s_idx[k]) * ob16; });
    }
  }
  const int n_oob = __syncthreads_count(code == 0);
  const int n_fut = __syncthreads_count(code == 1);
  const int n_dup = __syncthreads_count(code == 2);
  if (gridDim.x > 1 && !cta_is_last(a.ws.ctrl + CTRL_BOFFER)) return;
  const int64_t head = s_state[0], tail = s_state[1];
  if (acc) {
    const int64_t slot = (tail + pos) % a.q.n_env;
    a.q.ring_env[slot] = e;
    a.q.ring_time[slot] = t;
    a.q.pending[e] = 1;
  }
  if (i == 0) {
    if (nacc > 0 && tail == head) a.q.state[2] = a.now;  // the queue was empty: anchor
    a.q.state[1] = tail + nacc;
    a.counters[RLVLA_BCNT_OOB] = s_cnt[RLVLA_BCNT_OOB] + n_oob;
    a.counters[RLVLA_BCNT_FUTURE] = s_cnt[RLVLA_BCNT_FUTURE] + n_fut;
    a.counters[RLVLA_BCNT_DUP] = s_cnt[RLVLA_BCNT_DUP] + n_dup;
    a.counters[RLVLA_BCNT_ACCEPTED] = s_cnt[RLVLA_BCNT_ACCEPTED] + nacc;
    a.ws.ctrl[CTRL_BOFFER] = 0u;
  }
}

__global__ void __launch_bounds__(kPollThreads) batch_poll_kernel(BatchPollArgs a) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous call's queue updates
  const int64_t head = a.q.state[0], tail = a.q.state[1], anchor = a.q.state[2];
  const int64_t nbatches = a.q.state[3];
  const int64_t p = tail - head;
  // Eq. (1): (Batch Size >= B_max) or (Wait Time >= T_max); an empty queue never fires
  const bool fire = p >= a.b_max || (p >= 1 && a.now - anchor >= a.t_max);
  const int b = fire ? int(p < a.b_max ? p : a.b_max) : 0;
  if (b == 0) {  // no trigger: the state is unchanged, only the batch size is reported
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.out_n = 0;
    return;
  }
  const int cap = a.q.n_env;
  const int64_t ob = a.q.obs_bytes;
  __shared__ int s_env[kPollThreads];  // envs of the batch (b <= cap; staged when b fits)
  const bool staged = b <= kPollThreads;
  if (staged) {
    for (int k = threadIdx.x; k < b; k += blockDim.x) s_env[k] = a.q.ring_env[(head + k) % cap];
    __syncthreads();
  }
  const int64_t row0 = head % cap;  // FIFO rows: the batch starts here
  if (a.q.obs_fifo && ob > 0 && row0 + b > cap) {
    // the batch wraps: mirror its first rows past n_env so rows [row0, row0 + b) are contiguous
    const int64_t ob16 = ob >> 4;
    uint4* rows = reinterpret_cast<uint4*>(a.q.obs);
    grid_copy_rows(
        int(row0 + b - cap), ob16, [&](int k) { return rows + (int64_t(cap) + k) * ob16; },
        [&](int k) { return rows + int64_t(k) * ob16; });
  }
  if (a.out_obs != nullptr && ob > 0) {
    const int64_t ob16 = ob >> 4;
    const uint4* slots = reinterpret_cast<const uint4*>(a.q.obs);
    uint4* out = reinterpret_cast<uint4*>(a.out_obs);
    auto dst = [&](int k) { return out + int64_t(k) * ob16; };
    auto src = [&](int k) {
      if (a.q.obs_fifo) return slots + ((head + k) % cap) * ob16;
      const int env = staged ? s_env[k] : a.q.ring_env[(head + k) % cap];
      return slots + int64_t(env) * ob16;
    };
    grid_copy_rows(b, ob16, dst, src);
  }
  if (blockIdx.x == 0)
    for (int k = threadIdx.x; k < b; k += blockDim.x) {
      const int64_t slot = (head + k) % cap;
      a.out_env[k] = a.q.ring_env[slot];
      a.out_time[k] = a.q.ring_time[slot];
    }
  if (gridDim.x > 1 && !cta_is_last(a.ws.ctrl + CTRL_BPOLL)) return;
  __syncthreads();
  for (int k = threadIdx.x; k < b; k += blockDim.x)
    a.q.pending[staged ? s_env[k] : a.q.ring_env[(head + k) % cap]] = 0;
  if (threadIdx.x == 0) {
    if (b > 0) {
      a.q.state[0] = head + b;
      if (p - b > 0) a.q.state[2] = a.now;  // requests remain: re-anchor at the poll time
      a.q.state[3] = nbatches + 1;
      a.q.state[4] = row0;
    }
    *a.out_n = b;
    a.ws.ctrl[CTRL_BPOLL] = 0u;
  }
}

int copy_grid(int64_t rows, int64_t obs_bytes, int ctas_per_sm) {
  // 1024 threads per SM once there are at least 64 KB per SM to move
  const int64_t ctas = (rows * obs_bytes * ctas_per_sm + 65535) / 65536;
  const int64_t cap = int64_t(device_info().sm_count) * ctas_per_sm;
  return int(ctas < 1 ? 1 : (ctas > cap ? cap : ctas));
}

// launch with programmatic stream serialization (PDL): a tick's offer and poll launches
// overlap the previous kernel's tail; each kernel's griddepcontrol.wait keeps the order
template <typename Args>
cudaError_t launch_pdl(void (*kernel)(Args), int grid, int threads, const Args& a, cudaStream_t s,
                       size_t smem = 0) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, a);
}

}  // namespace

cudaError_t launch_batch_offer(const BatchOfferArgs& a, cudaStream_t s) {
  const int grid = (a.obs_src != nullptr && a.q.obs_bytes > 0) ? copy_grid(a.n, a.q.obs_bytes, 1) : 1;
  return launch_pdl(batch_offer_kernel, grid, kMaxOffer, a, s);
}

cudaError_t launch_batch_poll(const BatchPollArgs& a, cudaStream_t s) {
  const int64_t rows = a.b_max < a.q.n_env ? a.b_max : a.q.n_env;
  const bool copies = a.q.obs_bytes > 0 && (a.out_obs != nullptr || a.q.obs_fifo);
  const int grid = copies ? copy_grid(rows, a.q.obs_bytes, kPollCtasPerSm) : 1;
  return launch_pdl(batch_poll_kernel, grid, kPollThreads, a, s);
}

}  // namespace rlvla
