// api.cu — the extern "C" boundary (include/rlvla.h): argument validation, dispatch to the
// kernels, and the cross-rank exchanges C1 (advantage statistics), C2 (GRPO returns) and C3
// (loss statistics): inside the kernels over IPC-mapped NVLink mailboxes (set up here at
// communicator init), else NCCL collectives on the caller's stream.
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <mutex>
#include <atomic>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

namespace {
// NVTX range around each entry point (header-only NVTX3: free when no tool is attached), so
// an nsys timeline groups the kernels and collectives of a call under its ABI name
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

struct rlvla_comm_s {
  ncclComm_t comm = nullptr;  // NULL for a P2P-only communicator (rlvla_comm_init_p2p)
  int nranks;
  int rank;
  // in-kernel NVLink reduction (P2PDesc): own mailbox, peers' mailboxes mapped by CUDA IPC
  bool p2p = false;
  uint8_t* mbox = nullptr;
  uint8_t* peer[rlvla::kP2PMaxRanks] = {};
  unsigned long long* seq = nullptr;
};

namespace rlvla {

const DeviceInfo& device_info() {
  static std::mutex mu;
  static DeviceInfo cache[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    static DeviceInfo none;
    return none;
  }
  std::lock_guard<std::mutex> lk(mu);
  DeviceInfo& d = cache[dev];
  if (d.device != dev) {
    cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    d.device = dev;
  }
  return d;
}

namespace {
std::atomic<int> g_reserved_sms{0};
}
int persistent_sms() {
  const int n = device_info().sm_count - g_reserved_sms.load(std::memory_order_relaxed);
  return n < 1 ? 1 : n;
}

bool sync_check_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RLVLA_SYNC_CHECK");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

}  // namespace rlvla

using namespace rlvla;

namespace {

constexpr size_t kAlignWs = 256;

size_t ws_bytes_for(int32_t n_env_global) {
  const size_t r = (size_t(n_env_global > 0 ? n_env_global : 1) * sizeof(float) + kAlignWs - 1) /
                   kAlignWs * kAlignWs;
  return kCtrlBytes + kPartialBytes + r;
}

// RLVLA_DEBUG=1 prints the CUDA error behind an RLVLA_ERR_CUDA to stderr
rlvla_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return RLVLA_OK;
  (void)cudaGetLastError();  // do not leave a (non-sticky) error for the next caller
  const char* d = std::getenv("RLVLA_DEBUG");
  if (d && d[0] == '1') std::fprintf(stderr, "[rlvla] CUDA error %d: %s\n", int(e), cudaGetErrorString(e));
  return RLVLA_ERR_CUDA;
}

bool device_ready() { return device_info().sm_count > 0; }

rlvla_status check_buffer(const rlvla_traj_buffer* b) {
  if (!b) return RLVLA_ERR_INVALID_ARG;
  if (b->n_env <= 0 || b->t_steps <= 0 || b->a_tok <= 0) return RLVLA_ERR_INVALID_ARG;
  if (!b->slot_key || !b->reward || !b->done || !b->value || !b->version || !b->tokens ||
      !b->logp_behav)
    return RLVLA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(b->slot_key) % 8) return RLVLA_ERR_INVALID_ARG;
  return RLVLA_OK;
}

// rows == 0 (a rank or micro-batch without rows) allows NULL per-row / per-step arrays
rlvla_status check_ppo_args(const rlvla_ppo_args* f, int64_t rows) {
  if (rows > 0 && (!f->logp_behav || !f->adv || !f->version || !f->slot_key)) return RLVLA_ERR_INVALID_ARG;
  if (f->a_tok <= 0 || f->max_staleness < 0) return RLVLA_ERR_INVALID_ARG;
  if (!(f->eps_low >= 0.f) || !(f->eps_high >= 0.f) || f->eps_low >= 1.f) return RLVLA_ERR_INVALID_ARG;
  if (!(f->tok_denominator > 0.0) && !f->adv_stats && f->ratio_level == 0) return RLVLA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(f->slot_key) % 8) return RLVLA_ERR_INVALID_ARG;
  if (f->accumulate != 0 && f->accumulate != 1) return RLVLA_ERR_INVALID_ARG;
  if (f->ratio_level != 0 && f->ratio_level != 1) return RLVLA_ERR_INVALID_ARG;
  if (!(f->dual_clip <= 0.f || f->dual_clip > 1.f)) return RLVLA_ERR_INVALID_ARG;
  if (f->kl_coef != 0.f && !f->logp_ref && rows > 0) return RLVLA_ERR_INVALID_ARG;
  if (!(f->ent_coef == f->ent_coef) || !(f->kl_coef == f->kl_coef)) return RLVLA_ERR_INVALID_ARG;
  // chunk ratio with the call's own step count: micro-batches would each normalise by their
  // own count, so accumulate needs N_steps up front (explicit or from rlvla_advantages)
  if (f->ratio_level == 1 && !(f->tok_denominator > 0.0) && !f->adv_stats && f->accumulate)
    return RLVLA_ERR_INVALID_ARG;
  return RLVLA_OK;
}

bool multi_rank(rlvla_comm c) { return c && c->nranks > 1; }

// the in-kernel reduction descriptor for a call that reduces its loss statistics over `c`
P2PDesc p2p_desc(rlvla_comm c, int ch) {
  P2PDesc d;
  if (!c || !c->p2p || c->nranks <= 1) return d;
  d.nranks = c->nranks;
  d.rank = c->rank;
  d.ch = ch;
  for (int r = 0; r < c->nranks; ++r) d.mbox[r] = c->peer[r];
  d.seq = c->seq;
  return d;
}
bool uses_p2p(rlvla_comm c) { return c && c->p2p && c->nranks > 1; }

rlvla_status allreduce_stats(double* p, int n, rlvla_comm c, cudaStream_t s) {
  if (!c || c->nranks <= 1) return RLVLA_OK;
  if (!c->comm) return RLVLA_ERR_UNSUPPORTED;  // P2P-only communicator: no NCCL fallback
  return ncclAllReduce(p, p, size_t(n), ncclDouble, ncclSum, c->comm, s) == ncclSuccess
             ? RLVLA_OK
             : RLVLA_ERR_NCCL;
}

rlvla_status sync_check_stats(const double* stats, int slot, cudaStream_t s) {
  if (!sync_check_enabled() || !stats) return RLVLA_OK;
  double v = 0;
  if (cudaMemcpyAsync(&v, stats + slot, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return RLVLA_ERR_CUDA;
  return v != 0.0 ? RLVLA_ERR_DATA : RLVLA_OK;
}

// Loss statistics of a call with no rows on this rank (logits / flow paths): one CTA of the
// token-level S4 kernel over zero rows writes the call's totals (zeros, or the running
// totals with accumulate) and joins C3 on the same channel as the computing kernels.
rlvla_status stats_only_call(const rlvla_ppo_args& f, double* stats, void* workspace,
                             rlvla_comm comm, cudaStream_t s) {
  PpoArgs a{};
  a.rows = 0;
  a.f = f;
  a.f.ratio_level = 0;
  a.stats = stats;
  a.ws = carve(workspace);
  const bool p2p = uses_p2p(comm);
  if (p2p) a.ws.p2p = p2p_desc(comm, P2P_CH_LOSS);
  rlvla_status st = cuda_status(launch_ppo_loss(a, s));
  if (st != RLVLA_OK || p2p) return st;
  return allreduce_stats(stats + RLVLA_STAT_LOSS, RLVLA_STAT_DENOM - RLVLA_STAT_LOSS, comm, s);
}

}  // namespace

extern "C" {

RLVLA_API int32_t rlvla_abi_version(void) { return RLVLA_ABI_VERSION; }

RLVLA_API int32_t rlvla_set_reserved_sms(int32_t n) {
  if (n < 0) n = 0;
  return g_reserved_sms.exchange(n);
}

RLVLA_API const char* rlvla_status_string(rlvla_status s) {
  switch (s) {
    case RLVLA_OK: return "ok";
    case RLVLA_ERR_INVALID_ARG: return "invalid argument";
    case RLVLA_ERR_UNSUPPORTED: return "unsupported configuration";
    case RLVLA_ERR_CUDA: return "CUDA error";
    case RLVLA_ERR_NCCL: return "NCCL error";
    case RLVLA_ERR_DATA: return "data error counted on device (RLVLA_SYNC_CHECK)";
    default: return "unknown status";
  }
}

RLVLA_API int32_t rlvla_nccl_version(void) {
  int v = 0;
  if (ncclGetVersion(&v) != ncclSuccess) return 0;
  return v;
}

RLVLA_API size_t rlvla_workspace_bytes(int64_t rows, int32_t n_env_global, int32_t t_steps) {
  (void)rows;
  (void)t_steps;
  return ws_bytes_for(n_env_global);
}

RLVLA_API rlvla_status rlvla_scatter_steps(const rlvla_traj_buffer* buf,
                                           const rlvla_step_batch* rec, int32_t cur_version,
                                           uint64_t seq_base, int64_t* counters, void* stream) {
  NvtxRange nvtx_range("rlvla_scatter_steps");
  rlvla_status st = check_buffer(buf);
  if (st != RLVLA_OK) return st;
  if (!rec || rec->n_rec < 0 || !counters) return RLVLA_ERR_INVALID_ARG;
  if (cur_version < 0 || cur_version >= (1 << 23)) return RLVLA_ERR_INVALID_ARG;
  if (seq_base < 1 || seq_base + uint64_t(rec->n_rec) >= (uint64_t(1) << 40)) return RLVLA_ERR_INVALID_ARG;
  if (rec->n_rec == 0) return RLVLA_OK;
  if (!rec->env_id || !rec->step || !rec->version || !rec->reward || !rec->done || !rec->value ||
      !rec->tokens || !rec->logp_behav)
    return RLVLA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(counters) % 8) return RLVLA_ERR_INVALID_ARG;
  if (!device_ready()) return RLVLA_ERR_CUDA;
  ScatterArgs a{*buf, *rec, cur_version, seq_base, counters};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = cuda_status(launch_scatter(a, s));
  if (st != RLVLA_OK || !sync_check_enabled()) return st;
  int64_t c[4];
  if (cudaMemcpyAsync(c, counters, sizeof(c), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return RLVLA_ERR_CUDA;
  return (c[RLVLA_CNT_OOB] || c[RLVLA_CNT_BAD_VERSION]) ? RLVLA_ERR_DATA : RLVLA_OK;
}

RLVLA_API rlvla_status rlvla_advantages(const rlvla_traj_buffer* buf, const float* last_value,
                                        const rlvla_adv_params* p, float* adv, float* ret,
                                        double* stats, void* workspace, size_t ws_bytes,
                                        rlvla_comm comm, void* stream) {
  NvtxRange nvtx_range("rlvla_advantages");
  rlvla_status st = check_buffer(buf);
  if (st != RLVLA_OK) return st;
  if (!p || !adv || !stats || !workspace) return RLVLA_ERR_INVALID_ARG;
  if (p->mode != RLVLA_ADV_GAE && p->mode != RLVLA_ADV_GRPO) return RLVLA_ERR_INVALID_ARG;
  if (p->mode == RLVLA_ADV_GAE && !ret) return RLVLA_ERR_INVALID_ARG;
  if (p->max_staleness < 0) return RLVLA_ERR_INVALID_ARG;
  const int nranks = comm ? comm->nranks : 1;
  const int rank = comm ? comm->rank : 0;
  if (p->n_env_global != buf->n_env * nranks || p->env_offset != rank * buf->n_env)
    return RLVLA_ERR_INVALID_ARG;
  if (p->mode == RLVLA_ADV_GRPO && !p->group_id && p->group_size <= 0) return RLVLA_ERR_INVALID_ARG;
  if (p->mode == RLVLA_ADV_GRPO && !(p->grpo_eps >= 0.f)) return RLVLA_ERR_INVALID_ARG;
  if (ws_bytes < ws_bytes_for(p->n_env_global)) return RLVLA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(workspace) % kAlignWs || reinterpret_cast<uintptr_t>(stats) % 8)
    return RLVLA_ERR_INVALID_ARG;
  if (!device_ready()) return RLVLA_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  AdvArgs a{*buf, last_value, *p, adv, ret, stats, carve(workspace)};
  // C1 (+ C2) inside the pass-1 kernel over NVLink when the mailbox can hold the returns
  const bool p2p = uses_p2p(comm) && p->n_env_global <= kP2PMaxEnvGlobal;
  if (!p2p && multi_rank(comm) && !comm->comm) return RLVLA_ERR_UNSUPPORTED;
  if (p2p) a.ws.p2p = p2p_desc(comm, P2P_CH_ADV);
  st = cuda_status(launch_adv_pass1(a, s));
  if (st != RLVLA_OK) return st;
  if (!p2p && comm && comm->nranks > 1) {
    if (!comm->comm) return RLVLA_ERR_UNSUPPORTED;  // P2P-only communicator, mailbox too small
    if (ncclGroupStart() != ncclSuccess) return RLVLA_ERR_NCCL;
    ncclResult_t r1 = ncclAllReduce(stats, stats, 6, ncclDouble, ncclSum, comm->comm, s);
    ncclResult_t r4 = ncclAllReduce(stats + RLVLA_STAT_N_LOSS_STEPS, stats + RLVLA_STAT_N_LOSS_STEPS, 1,
                                    ncclDouble, ncclSum, comm->comm, s);
    ncclResult_t r2 = ncclSuccess;
    if (p->mode == RLVLA_ADV_GRPO) {
      float* rg = a.ws.r_global;
      r2 = ncclAllGather(rg + size_t(rank) * buf->n_env, rg, size_t(buf->n_env), ncclFloat,
                         comm->comm, s);
    }
    ncclResult_t r3 = ncclGroupEnd();
    if (r1 != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess || r4 != ncclSuccess)
      return RLVLA_ERR_NCCL;
  }
  st = cuda_status(launch_adv_pass2(a, s));
  if (st != RLVLA_OK) return st;
  return sync_check_stats(stats, RLVLA_STAT_N_BAD_STEPS, s);
}

RLVLA_API rlvla_status rlvla_logprob_fwd_bwd(const rlvla_logits* x, const int32_t* target,
                                             float* logp, float* lse, const float* grad_logp,
                                             const rlvla_ppo_args* fused, void* dlogits,
                                             double* stats, void* workspace, size_t ws_bytes,
                                             rlvla_comm comm, void* stream) {
  NvtxRange nvtx_range("rlvla_logprob_fwd_bwd");
  if (!x || ((!x->ptr || !target) && x->rows != 0)) return RLVLA_ERR_INVALID_ARG;
  if (x->dtype != RLVLA_F32 && x->dtype != RLVLA_BF16) return RLVLA_ERR_INVALID_ARG;
  if (x->rows < 0 || x->vocab < 1 || x->ld < x->vocab) return RLVLA_ERR_INVALID_ARG;
  if (fused && grad_logp) return RLVLA_ERR_INVALID_ARG;
  if (grad_logp) {
    if ((!lse || !dlogits) && x->rows != 0) return RLVLA_ERR_INVALID_ARG;
  } else if (!logp && x->rows != 0) {
    return RLVLA_ERR_INVALID_ARG;
  }
  if (fused) {
    rlvla_status st = check_ppo_args(fused, x->rows);
    if (st != RLVLA_OK) return st;
    if (x->rows % fused->a_tok) return RLVLA_ERR_INVALID_ARG;
    if (fused->ratio_level != 0) return RLVLA_ERR_UNSUPPORTED;  // chunk ratio: rlvla_ppo_loss
  }
  if (stats && !grad_logp) {
    if (!workspace || ws_bytes < ws_bytes_for(1) || reinterpret_cast<uintptr_t>(workspace) % kAlignWs)
      return RLVLA_ERR_INVALID_ARG;
  }
  const bool want_stats = stats && !grad_logp;
  if (x->rows == 0 && !want_stats) return RLVLA_OK;
  if (!device_ready()) return RLVLA_ERR_CUDA;
  if (want_stats && multi_rank(comm) && !uses_p2p(comm) && !comm->comm) return RLVLA_ERR_UNSUPPORTED;
  if (x->rows == 0) {
    // no rows on this rank: write this call's (zero or accumulated) statistics and take part
    // in C3 like the ranks that have rows
    rlvla_ppo_args f0{};
    if (fused) f0 = *fused;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rlvla_status st = stats_only_call(f0, stats, workspace, comm, s);
    if (st != RLVLA_OK) return st;
    return sync_check_stats(stats, RLVLA_STAT_N_BAD_TOK, s);
  }
  LpArgs a{};
  a.x = *x;
  a.target = target;
  a.logp = logp;
  a.lse = lse;
  a.grad_logp = grad_logp;
  a.fused = fused != nullptr;
  if (fused) a.f = *fused;
  a.dlogits = dlogits;
  a.stats = grad_logp ? nullptr : stats;
  if (workspace) a.ws = carve(workspace);
  const bool p2p = a.stats && uses_p2p(comm);
  if (p2p) a.ws.p2p = p2p_desc(comm, P2P_CH_LOSS);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  rlvla_status st = cuda_status(launch_logprob(a, s));
  if (st != RLVLA_OK) return st;
  if (a.stats) {
    if (!p2p) st = allreduce_stats(stats + RLVLA_STAT_LOSS, RLVLA_STAT_DENOM - RLVLA_STAT_LOSS, comm, s);
    if (st != RLVLA_OK) return st;
    return sync_check_stats(stats, RLVLA_STAT_N_BAD_TOK, s);
  }
  return RLVLA_OK;
}

RLVLA_API rlvla_status rlvla_ppo_loss(const float* logp, int64_t rows, const int32_t* target,
                                      const rlvla_ppo_args* f, float* grad_logp, float* loss_tok,
                                      double* stats, void* workspace, size_t ws_bytes,
                                      rlvla_comm comm, void* stream) {
  NvtxRange nvtx_range("rlvla_ppo_loss");
  if (!f || rows < 0 || ((!logp || !grad_logp) && rows != 0)) return RLVLA_ERR_INVALID_ARG;
  rlvla_status st = check_ppo_args(f, rows);
  if (st != RLVLA_OK) return st;
  if (rows % f->a_tok) return RLVLA_ERR_INVALID_ARG;
  if (f->ent_coef != 0.f) return RLVLA_ERR_UNSUPPORTED;  // the entropy bonus needs the logits
  if (f->ratio_level == 1 && f->kl_coef != 0.f) return RLVLA_ERR_UNSUPPORTED;  // per-token KL vs per-step mean: no reading
  if ((stats || f->ratio_level == 1) &&
      (!workspace || ws_bytes < ws_bytes_for(1) || reinterpret_cast<uintptr_t>(workspace) % kAlignWs))
    return RLVLA_ERR_INVALID_ARG;
  // chunk ratio with the call's own step count over several ranks: the count is reduced
  // through `stats`, so they are required
  const bool implicit_chunk = f->ratio_level == 1 && !(f->tok_denominator > 0.0) && !f->adv_stats;
  if (implicit_chunk && multi_rank(comm) && !stats) return RLVLA_ERR_INVALID_ARG;
  if (rows == 0 && !stats) return RLVLA_OK;
  if (!device_ready()) return RLVLA_ERR_CUDA;
  if (stats && multi_rank(comm) && !uses_p2p(comm) && !comm->comm) return RLVLA_ERR_UNSUPPORTED;
  PpoArgs a{};
  a.logp = logp;
  a.rows = rows;
  a.target = target;
  a.f = *f;
  a.grad_logp = grad_logp;
  a.loss_tok = loss_tok;
  a.stats = stats;
  if (workspace) a.ws = carve(workspace);
  // C3 in-kernel over NVLink (token- and chunk-level paths)
  const bool p2p = stats && uses_p2p(comm);
  if (p2p) a.ws.p2p = p2p_desc(comm, P2P_CH_LOSS);
  // NCCL fallback with the chunk path's own step count: raw sums and counts are allreduced
  // (slots 6..18), then the scale kernel normalises with the global count
  a.defer = implicit_chunk && stats && multi_rank(comm) && !p2p;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = cuda_status(launch_ppo_loss(a, s));
  if (st != RLVLA_OK) return st;
  if (a.defer) {
    st = allreduce_stats(stats + RLVLA_STAT_LOSS, RLVLA_STAT_DENOM + 1 - RLVLA_STAT_LOSS, comm, s);
    if (st != RLVLA_OK) return st;
    st = cuda_status(launch_ppo_chunk_scale(a, s));
    if (st != RLVLA_OK) return st;
    return sync_check_stats(stats, RLVLA_STAT_N_BAD_TOK, s);
  }
  if (stats) {
    if (!p2p) st = allreduce_stats(stats + RLVLA_STAT_LOSS, RLVLA_STAT_DENOM - RLVLA_STAT_LOSS, comm, s);
    if (st != RLVLA_OK) return st;
    return sync_check_stats(stats, RLVLA_STAT_N_BAD_TOK, s);
  }
  return RLVLA_OK;
}

RLVLA_API rlvla_status rlvla_value_loss(const float* v_new, const float* v_old, const float* ret,
                                        const uint64_t* slot_key, const int32_t* version,
                                        int64_t n_steps, int32_t cur_version,
                                        int32_t max_staleness, float clip_eps,
                                        double denominator, float* grad_v, float* loss_step,
                                        double* stats, void* workspace, size_t ws_bytes,
                                        rlvla_comm comm, void* stream) {
  NvtxRange nvtx_range("rlvla_value_loss");
  if (n_steps < 0 || max_staleness < 0) return RLVLA_ERR_INVALID_ARG;
  if (n_steps > 0 && (!v_new || !ret || !slot_key || !version || !grad_v)) return RLVLA_ERR_INVALID_ARG;
  if (clip_eps > 0.f && !v_old && n_steps > 0) return RLVLA_ERR_INVALID_ARG;
  if (!(clip_eps == clip_eps)) return RLVLA_ERR_INVALID_ARG;
  if (!workspace || ws_bytes < ws_bytes_for(1) || reinterpret_cast<uintptr_t>(workspace) % kAlignWs)
    return RLVLA_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(slot_key) % 8 || (stats && reinterpret_cast<uintptr_t>(stats) % 8))
    return RLVLA_ERR_INVALID_ARG;
  const bool implicit = !(denominator > 0.0);
  // the call's own N_v over several ranks is reduced through `stats`
  if (implicit && multi_rank(comm) && !stats) return RLVLA_ERR_INVALID_ARG;
  if (n_steps == 0 && !stats) return RLVLA_OK;
  if (!device_ready()) return RLVLA_ERR_CUDA;
  if (stats && multi_rank(comm) && !uses_p2p(comm) && !comm->comm) return RLVLA_ERR_UNSUPPORTED;
  ValueArgs a{v_new, v_old, ret, slot_key, version, n_steps, cur_version, max_staleness, clip_eps,
              denominator, grad_v, loss_step, stats, carve(workspace), 0};
  const bool p2p = stats && uses_p2p(comm);
  if (p2p) a.ws.p2p = p2p_desc(comm, P2P_CH_VALUE);
  a.defer = implicit && stats && multi_rank(comm) && !p2p;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  rlvla_status st = cuda_status(launch_value_loss(a, s));
  if (st != RLVLA_OK || !stats || p2p) return st;
  st = allreduce_stats(stats + RLVLA_STAT_VALUE_LOSS, RLVLA_STAT_VALUE_DENOM - RLVLA_STAT_VALUE_LOSS,
                       comm, s);
  if (st != RLVLA_OK || !a.defer) return st;
  return cuda_status(launch_value_scale(a, s));
}

namespace {
bool misaligned(const void* p, uintptr_t a) { return reinterpret_cast<uintptr_t>(p) % a != 0; }

rlvla_status check_queue(const rlvla_batch_queue* q) {
  if (!q || q->n_env < 1 || !q->ring_env || !q->ring_time || !q->pending || !q->state)
    return RLVLA_ERR_INVALID_ARG;
  if (q->obs_bytes < 0 || q->obs_bytes % 16 || (q->obs_bytes > 0 && (!q->obs || misaligned(q->obs, 16))))
    return RLVLA_ERR_INVALID_ARG;
  if (misaligned(q->state, 8) || misaligned(q->ring_time, 8) || misaligned(q->ring_env, 4))
    return RLVLA_ERR_INVALID_ARG;
  if (q->obs_fifo != 0 && q->obs_fifo != 1) return RLVLA_ERR_INVALID_ARG;
  if (q->obs_fifo && (q->max_batch < 1 || q->max_batch > q->n_env)) return RLVLA_ERR_INVALID_ARG;
  return RLVLA_OK;
}

rlvla_status check_ws(const void* workspace, size_t ws_bytes) {
  if (!workspace || ws_bytes < ws_bytes_for(1) || misaligned(workspace, kAlignWs))
    return RLVLA_ERR_INVALID_ARG;
  return RLVLA_OK;
}
}  // namespace

RLVLA_API rlvla_status rlvla_batch_offer(const rlvla_batch_queue* q, const int32_t* env_id,
                                         const int64_t* enqueue_time, int32_t n, int64_t now,
                                         const void* obs_src, int64_t* counters,
                                         void* workspace, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_range("rlvla_batch_offer");
  rlvla_status st = check_queue(q);
  if (st != RLVLA_OK) return st;
  if ((st = check_ws(workspace, ws_bytes)) != RLVLA_OK) return st;
  if (n < 0 || n > kMaxOffer || now < 0 || !counters || misaligned(counters, 8))
    return RLVLA_ERR_INVALID_ARG;
  if (n > 0 && (!env_id || !enqueue_time || misaligned(enqueue_time, 8))) return RLVLA_ERR_INVALID_ARG;
  if (obs_src && misaligned(obs_src, 16)) return RLVLA_ERR_INVALID_ARG;
  if (q->obs_fifo && q->obs_bytes > 0 && n > 0 && !obs_src) return RLVLA_ERR_INVALID_ARG;
  if (n == 0) return RLVLA_OK;
  if (!device_ready()) return RLVLA_ERR_CUDA;
  BatchOfferArgs a{*q, env_id, enqueue_time, n, now, static_cast<const uint8_t*>(obs_src),
                   counters, carve(workspace)};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = cuda_status(launch_batch_offer(a, s));
  if (st != RLVLA_OK || !sync_check_enabled()) return st;
  int64_t c[4];
  if (cudaMemcpyAsync(c, counters, sizeof(c), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return RLVLA_ERR_CUDA;
  return (c[RLVLA_BCNT_OOB] || c[RLVLA_BCNT_FUTURE]) ? RLVLA_ERR_DATA : RLVLA_OK;
}

RLVLA_API rlvla_status rlvla_batch_poll(const rlvla_batch_queue* q, int64_t now, int32_t b_max,
                                        int64_t t_max, int32_t* out_env, int64_t* out_time,
                                        void* out_obs, int32_t* out_n, void* workspace,
                                        size_t ws_bytes, void* stream) {
  NvtxRange nvtx_range("rlvla_batch_poll");
  rlvla_status st = check_queue(q);
  if (st != RLVLA_OK) return st;
  if ((st = check_ws(workspace, ws_bytes)) != RLVLA_OK) return st;
  if (b_max < 1 || t_max < 0 || now < 0 || !out_env || !out_time || !out_n)
    return RLVLA_ERR_INVALID_ARG;
  if (q->obs_fifo && b_max > q->max_batch) return RLVLA_ERR_INVALID_ARG;
  if (misaligned(out_time, 8) || misaligned(out_env, 4) || misaligned(out_n, 4) ||
      (out_obs && misaligned(out_obs, 16)))
    return RLVLA_ERR_INVALID_ARG;
  if (!device_ready()) return RLVLA_ERR_CUDA;
  BatchPollArgs a{*q, now, b_max, t_max, out_env, out_time, static_cast<uint8_t*>(out_obs), out_n,
                  carve(workspace)};
  return cuda_status(launch_batch_poll(a, static_cast<cudaStream_t>(stream)));
}

RLVLA_API rlvla_status rlvla_flow_logprob(const rlvla_gauss_chain* c, float* logp,
                                          const float* grad_logp, const rlvla_ppo_args* fused,
                                          void* dmu, float* dlog_std, double* stats,
                                          void* workspace, size_t ws_bytes, rlvla_comm comm,
                                          void* stream) {
  NvtxRange nvtx_range("rlvla_flow_logprob");
  if (!c || c->rows < 0 || c->n_steps < 1 || c->dim < 1 || ((!c->mu || !c->x) && c->rows != 0))
    return RLVLA_ERR_INVALID_ARG;
  if (int64_t(c->n_steps) * c->dim > kFlowMaxElems) return RLVLA_ERR_INVALID_ARG;
  if (c->mu_dtype != RLVLA_F32 && c->mu_dtype != RLVLA_BF16) return RLVLA_ERR_INVALID_ARG;
  if (!c->log_std && !c->sigma_k && c->rows != 0) return RLVLA_ERR_INVALID_ARG;
  if (dlog_std && !c->log_std) return RLVLA_ERR_INVALID_ARG;  // no learned ln sigma to differentiate
  if (grad_logp && fused) return RLVLA_ERR_INVALID_ARG;
  if (!grad_logp && !logp && c->rows != 0) return RLVLA_ERR_INVALID_ARG;
  if (!grad_logp && !fused && (dmu || dlog_std)) return RLVLA_ERR_INVALID_ARG;  // nothing to differentiate
  if (grad_logp && !dmu && !dlog_std && c->rows != 0) return RLVLA_ERR_INVALID_ARG;
  if (misaligned(c->mu, c->mu_dtype == RLVLA_BF16 ? 2 : 4) || misaligned(c->x, 4) ||
      (stats && misaligned(stats, 8)))
    return RLVLA_ERR_INVALID_ARG;
  if (fused) {
    rlvla_status st = check_ppo_args(fused, c->rows);
    if (st != RLVLA_OK) return st;
    if (fused->a_tok != 1 || fused->ratio_level != 0) return RLVLA_ERR_INVALID_ARG;
  }
  if (stats || fused) {
    if (!workspace || ws_bytes < ws_bytes_for(1) || misaligned(workspace, kAlignWs))
      return RLVLA_ERR_INVALID_ARG;
  }
  const bool want_stats = stats && !grad_logp;
  if (c->rows == 0 && !want_stats) return RLVLA_OK;
  if (!device_ready()) return RLVLA_ERR_CUDA;
  if (want_stats && multi_rank(comm) && !uses_p2p(comm) && !comm->comm) return RLVLA_ERR_UNSUPPORTED;
  if (c->rows == 0) {  // no rows on this rank: zero / accumulated statistics, C3 as the others
    rlvla_ppo_args f0{};
    if (fused) f0 = *fused;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rlvla_status st = stats_only_call(f0, stats, workspace, comm, s);
    if (st != RLVLA_OK) return st;
    return sync_check_stats(stats, RLVLA_STAT_N_BAD_TOK, s);
  }
  FlowArgs a{};
  a.c = *c;
  a.logp = logp;
  a.grad_logp = grad_logp;
  a.fused = fused != nullptr;
  if (fused) a.f = *fused;
  a.dmu = dmu;
  a.dlog_std = dlog_std;
  a.stats = grad_logp ? nullptr : stats;
  if (workspace) a.ws = carve(workspace);
  const bool p2p = a.stats && uses_p2p(comm);
  if (p2p) a.ws.p2p = p2p_desc(comm, P2P_CH_LOSS);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  rlvla_status st = cuda_status(launch_flow(a, s));
  if (st != RLVLA_OK || !a.stats) return st;
  if (!p2p) st = allreduce_stats(stats + RLVLA_STAT_LOSS, RLVLA_STAT_DENOM - RLVLA_STAT_LOSS, comm, s);
  if (st != RLVLA_OK) return st;
  if (sync_check_enabled()) return sync_check_stats(stats, RLVLA_STAT_N_BAD_TOK, s);
  return RLVLA_OK;
}

RLVLA_API rlvla_status rlvla_comm_unique_id(void* out) {
  if (!out) return RLVLA_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return RLVLA_ERR_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return RLVLA_OK;
}

namespace {
static_assert(sizeof(cudaIpcMemHandle_t) == RLVLA_P2P_HANDLE_BYTES, "IPC handle size");

// this rank's mailbox and call counters, and the IPC handle of the mailbox (no collective)
bool alloc_mailbox(rlvla_comm c, cudaIpcMemHandle_t* h) {
  bool ok = cudaMalloc(&c->mbox, kP2PMboxBytes) == cudaSuccess &&
            cudaMemset(c->mbox, 0, kP2PMboxBytes) == cudaSuccess &&
            cudaMalloc(&c->seq, kP2PChannels * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMemset(c->seq, 0, kP2PChannels * sizeof(unsigned long long)) == cudaSuccess &&
            cudaIpcGetMemHandle(h, c->mbox) == cudaSuccess;
  (void)cudaGetLastError();
  return ok;
}

void close_peers(rlvla_comm c) {
  for (int r = 0; r < c->nranks; ++r)
    if (r != c->rank && c->peer[r]) cudaIpcCloseMemHandle(c->peer[r]);
  for (auto& q : c->peer) q = nullptr;
  (void)cudaGetLastError();
}

// map every peer's mailbox (all: [nranks] handles in rank order); on failure none stays open
bool open_peers(rlvla_comm c, const cudaIpcMemHandle_t* all) {
  bool ok = true;
  for (int r = 0; ok && r < c->nranks; ++r) {
    if (r == c->rank) {
      c->peer[r] = c->mbox;
      continue;
    }
    void* p = nullptr;
    ok = cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    c->peer[r] = ok ? static_cast<uint8_t*>(p) : nullptr;
  }
  if (!ok) close_peers(c);
  (void)cudaGetLastError();
  return ok;
}

// one record per rank in the NCCL handle exchange: the handle and whether the rank has one
struct HandleRec {
  cudaIpcMemHandle_t h;
  int32_t ok;
  int32_t pad[15];
};
size_t stage_bytes(int nranks) { return sizeof(HandleRec) * size_t(nranks + 1) + sizeof(int); }

// Mailboxes for the in-kernel NVLink reduction over an NCCL communicator: the handles are
// allgathered over it and opened (peer mappings). `stage` is device memory allocated before
// the communicator existed, so every rank enters the same two collectives (the allgather,
// then a min-vote) whatever its local result; a rank that failed to allocate or map makes
// every rank keep the NCCL collectives. RLVLA_P2P=0 disables it (on every rank).
void setup_p2p(rlvla_comm c, uint8_t* stage) {
  const char* env = std::getenv("RLVLA_P2P");
  if (c->nranks <= 1 || c->nranks > kP2PMaxRanks || (env && env[0] == '0')) return;
  HandleRec mine{};
  mine.ok = alloc_mailbox(c, &mine.h) ? 1 : 0;
  const size_t rb = sizeof(HandleRec);
  uint8_t* recv = stage;
  uint8_t* send = stage + size_t(c->nranks) * rb;
  int* vote = reinterpret_cast<int*>(stage + size_t(c->nranks + 1) * rb);
  if (cudaMemcpy(send, &mine, rb, cudaMemcpyHostToDevice) != cudaSuccess) mine.ok = 0;
  std::vector<HandleRec> all(size_t(c->nranks));
  bool ok = ncclAllGather(send, recv, rb, ncclChar, c->comm, nullptr) == ncclSuccess &&
            cudaDeviceSynchronize() == cudaSuccess &&
            cudaMemcpy(all.data(), recv, rb * size_t(c->nranks), cudaMemcpyDeviceToHost) == cudaSuccess;
  for (int r = 0; ok && r < c->nranks; ++r) ok = all[size_t(r)].ok == 1;
  if (ok) {
    std::vector<cudaIpcMemHandle_t> h(size_t(c->nranks));
    for (int r = 0; r < c->nranks; ++r) h[size_t(r)] = all[size_t(r)].h;
    ok = open_peers(c, h.data());
  }
  // every rank must agree: a rank that failed makes all of them use NCCL
  int flag = ok ? 1 : 0;
  const bool voted = cudaMemcpy(vote, &flag, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess;
  if (ncclAllReduce(vote, vote, 1, ncclInt, ncclMin, c->comm, nullptr) != ncclSuccess ||
      cudaDeviceSynchronize() != cudaSuccess || !voted ||
      cudaMemcpy(&flag, vote, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    flag = 0;
  (void)cudaGetLastError();
  c->p2p = flag == 1;
  if (!c->p2p) close_peers(c);
}
}  // namespace

RLVLA_API int32_t rlvla_comm_p2p_enabled(rlvla_comm c) { return (c && c->p2p) ? 1 : 0; }

RLVLA_API rlvla_status rlvla_comm_init(const void* id, int32_t nranks, int32_t rank,
                                       rlvla_comm* out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return RLVLA_ERR_INVALID_ARG;
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  // the handle-exchange staging buffer exists before the communicator does: a rank that
  // cannot allocate it fails here, like a failed NCCL init, not inside a collective
  uint8_t* stage = nullptr;
  if (nranks > 1 && cudaMalloc(&stage, stage_bytes(nranks)) != cudaSuccess) {
    (void)cudaGetLastError();
    return RLVLA_ERR_CUDA;
  }
  rlvla_comm c = new rlvla_comm_s{};
  c->nranks = nranks;
  c->rank = rank;
  if (ncclCommInitRank(&c->comm, nranks, uid, rank) != ncclSuccess) {
    if (stage) cudaFree(stage);
    delete c;
    return RLVLA_ERR_NCCL;
  }
  if (stage) {
    setup_p2p(c, stage);  // best effort: without it the collectives stay on NCCL
    cudaFree(stage);
  }
  *out = c;
  return RLVLA_OK;
}

RLVLA_API rlvla_status rlvla_comm_init_p2p(int32_t nranks, int32_t rank, void* out_handle,
                                           rlvla_comm* out) {
  if (!out_handle || !out || nranks < 1 || nranks > kP2PMaxRanks || rank < 0 || rank >= nranks)
    return RLVLA_ERR_INVALID_ARG;
  if (!device_ready()) return RLVLA_ERR_CUDA;
  rlvla_comm c = new rlvla_comm_s{};
  c->nranks = nranks;
  c->rank = rank;
  cudaIpcMemHandle_t h{};
  if (nranks > 1 && !alloc_mailbox(c, &h)) {
    if (c->mbox) cudaFree(c->mbox);
    if (c->seq) cudaFree(c->seq);
    delete c;
    return RLVLA_ERR_CUDA;
  }
  std::memcpy(out_handle, &h, sizeof(h));
  *out = c;
  return RLVLA_OK;
}

RLVLA_API rlvla_status rlvla_comm_connect_p2p(rlvla_comm c, const void* all_handles) {
  if (!c || !all_handles || c->comm) return RLVLA_ERR_INVALID_ARG;
  if (c->nranks <= 1) return RLVLA_OK;
  if (c->p2p) return RLVLA_ERR_INVALID_ARG;  // already connected
  std::vector<cudaIpcMemHandle_t> h(size_t(c->nranks));
  std::memcpy(h.data(), all_handles, sizeof(cudaIpcMemHandle_t) * size_t(c->nranks));
  if (!open_peers(c, h.data())) return RLVLA_ERR_CUDA;
  c->p2p = true;
  return RLVLA_OK;
}

RLVLA_API rlvla_status rlvla_comm_destroy(rlvla_comm c) {
  if (!c) return RLVLA_OK;
  close_peers(c);
  if (c->mbox) cudaFree(c->mbox);
  if (c->seq) cudaFree(c->seq);
  const ncclResult_t r = c->comm ? ncclCommDestroy(c->comm) : ncclSuccess;
  delete c;
  return r == ncclSuccess ? RLVLA_OK : RLVLA_ERR_NCCL;
}

}  // extern "C"
