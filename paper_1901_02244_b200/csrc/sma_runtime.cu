// sma_runtime.cu -- libsma's C ABI (include/sma.h): handle, buffers, streams,
// events, NCCL communicator / P2P / NVLS z-sync setup, CUDA graphs, learners.
// (Error messages, the NCCL binding and the pure bookkeeping functions live in
// sma_host.cu.)
//
// One round (sma_step) is one iteration of Alg. 1.  The
// runtime replaces Crossbow's task manager/scheduler with a
// static contiguous layout: the r local replicas live in ONE allocation
// W[r][d_pad] and are advanced by ONE batched kernel instead
// of r learner streams; the global synchronisation task
// is NCCL reduce-scatter -> shard update -> all-gather on
// the caller's stream (Mode A) or on a second stream overlapping the next
// replica kernel (Mode B).
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <future>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/sma.h"
#include "sma_host.h"
#include "sma_internal.h"

using namespace sma;

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(_e == cudaErrorMemoryAllocation ? SMA_ERR_OOM : SMA_ERR_CUDA,           \
                  "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

// NVTX ranges (header-only NVTX3: free unless a profiler such as nsys injects
// itself) around the host-side enqueue of every phase of a round.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

#define STATUS_TRY(expr)              \
  do {                                \
    sma_status _s = (expr);           \
    if (_s != SMA_OK) return _s;      \
  } while (0)

#define NCCL_TRY(expr)                                                                  \
  do {                                                                                  \
    ncclResult_t _r = (expr);                                                           \
    if (_r != ncclSuccess)                                                              \
      return fail(SMA_ERR_NCCL, "%s failed: %s", #expr, g_nccl.GetErrorString(_r));     \
  } while (0)

// ------------------------------------------------------------------ handle
struct sma_handle {
  sma_config cfg{};
  int dev = 0, num_sms = 148;
  int64_t d_pad = 0, n4 = 0, shard_off = 0, shard_len = 0;
  int r = 0, j0 = 0;
  bool collective = false, overlap = false, matc = false, tma = false, timing = false,
       graphs = false, check = false;
  float alpha = 0, gamma = 0, mu = 0;
  // Section 3.3 two-level rule (SMA_FLAG_HIERARCHICAL, R20): alpha is alpha_l;
  // U is this GPU's reference model u_g (ranks >= 1 of the collective path; on
  // rank 0 the reference model is z itself)
  bool hier = false;
  float alpha_g = 0;
  float* U = nullptr;      // [d_pad]

  float* W = nullptr;      // [r][d_pad]
  float* zbuf = nullptr;   // [2][d_pad]
  float* P = nullptr;      // [d_pad] per-GPU partial (collective, Mode A)
  float* S = nullptr;      // [shard] reduce-scatter result
  float* Q = nullptr;      // [2][d_pad] (Mode B)
  float* C = nullptr;      // [r][d_pad] (MATERIALIZE_C)
  float* G = nullptr;      // [r][d_pad] internal gradient buffers (lazy)
  int* nonfinite = nullptr;
  int cur = 0, qi = 0;
  bool q_dirty = true;

  const float* gptr[SMA_MAX_LOCAL_REPLICAS] = {};
  uint64_t ver = 1;  // bumps when anything baked into a graph changes

  // pipelined host intake and asynchronous read-back (sma_stage_grads_host,
  // sma_get_central_async): two internal gradient sets G2[2][r][d_pad] filled on
  // sH2D, z copied out on sD2H; events order each against the rounds
  float* G2 = nullptr;
  cudaStream_t sH2D = nullptr, sD2H = nullptr;
  cudaEvent_t evStaged[2] = {}, evUsed[2] = {}, evZread[2] = {}, evAsync = nullptr;
  bool used_rec[2] = {false, false}, zread_pending[2] = {false, false};
  bool async_pending = false, h2d_pending = false;
  int cur_set = -1;        // the gradient set the registrations point into (-1: none)
  bool stage_wait = false; // the next round must wait for evStaged[cur_set]

  ncclComm_t comm = nullptr;
  // collective buffers from ncclMemAlloc (NVLS-capable) and their registrations
  std::vector<void*> nccl_allocs, nccl_regs;
  int sync_sms = 16;  // SMs left to the overlapped z-sync in Mode B (SMA_SYNC_SMS)
  // NEXT-1 multicast z-sync
  bool nvls = false;
  NvlsRegion nv;
  size_t nv_off_part = 0, nv_off_z = 0;
  unsigned* nv_ctl = nullptr;  // [0..1] expect, [2] done counter (local memory)
  // P2P z-sync (CUDA IPC)
  bool p2p = false, p2p_connected = false;
  bool push = false;            // SMA_FLAG_P2P_PUSH
  float* push_scratch = nullptr;  // [d_pad] Mode B prologue staging (push mode)
  char* p2p_region = nullptr;
  size_t p2p_off_part = 0, p2p_off_z = 0;
  std::vector<char*> p2p_base;  // per rank, as mapped in this process
  unsigned* p2p_ctl = nullptr;
  cudaStream_t sB = nullptr, sIO = nullptr;
  cudaEvent_t evFork = nullptr, evJoin = nullptr, evDone = nullptr;
  bool any_work = false;

  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  uint64_t gver[2] = {0, 0};

  // SMA_FLAG_TIMING: (start, stop) event pairs per phase (SMA_PHASE_*)
  std::vector<cudaEvent_t> tev[SMA_NUM_PHASES];
  size_t tused[SMA_NUM_PHASES] = {};
  int64_t launches = 0;

  // learner
  bool learner = false;
  int kind = 0, in_dim = 0, hidden = 0, classes = 0, batch = 0;
  float2* mlp_A1 = nullptr;  // MLP scratch, sized for SMA_MAX_LOCAL_REPLICAS learners
  float* mlp_DA = nullptr;
  float* mlp_E = nullptr;
  float* mlp_PL = nullptr;     // fused MLP round: partial logits [2][num_sms][16][32], b2 [2][num_sms][32]
  unsigned* mlp_bar = nullptr; // fused MLP round: flag lines [3 num_sms][32]
  unsigned mlp_epoch = 0;      // fused MLP round: launches so far (the flags' epoch)
  const float* X = nullptr;
  const int32_t* y = nullptr;
  int64_t n_samples = 0;
  uint64_t batch_seed = 0;
  int32_t* perm_dev[2] = {nullptr, nullptr};
  int64_t perm_epoch[2] = {-1, -1};
  int32_t* perm_host[2] = {nullptr, nullptr};  // pinned staging, one per device buffer
  cudaEvent_t perm_ev[2] = {nullptr, nullptr};  // the upload from perm_host[i] completed
  bool perm_ev_used[2] = {false, false};
  // the next epoch's permutation, computed on a host worker thread while the
  // current epoch's rounds run (into perm_host[(e + 1) & 1])
  std::future<void> perm_next;
  int64_t perm_next_epoch = -1;

  float* z() const { return zbuf + (int64_t)cur * d_pad; }
  float* zprev() const { return zbuf + (int64_t)(1 - cur) * d_pad; }
};

namespace {
struct DeviceGuard {
  int old = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&old) != cudaSuccess) old = -1;
    if (old != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int now = -1;
    if (old >= 0 && cudaGetDevice(&now) == cudaSuccess && now != old) cudaSetDevice(old);
  }
};

bool finite_f(float v) { return std::isfinite(v); }

sma_status local_slot(const sma_handle* h, int32_t j, int* slot) {
  if (j < 0 || j >= h->cfg.k) return fail(SMA_ERR_INVALID_ARG, "replica %d outside [0,%d)", j, h->cfg.k);
  if (j < h->j0 || j >= h->j0 + h->r)
    return fail(SMA_ERR_NOT_LOCAL, "replica %d lives on another rank (local [%d,%d))", j, h->j0,
                h->j0 + h->r);
  *slot = j - h->j0;
  return SMA_OK;
}

void free_all(sma_handle* h) {
  DeviceGuard g(h->dev);
  if (h->any_work) cudaDeviceSynchronize();
  for (int i = 0; i < 2; ++i)
    if (h->gexec[i]) cudaGraphExecDestroy(h->gexec[i]);
  if (h->p2p) {
    for (int g = 0; g < (int)h->p2p_base.size(); ++g)
      if (g != h->cfg.rank && h->p2p_base[g]) cudaIpcCloseMemHandle(h->p2p_base[g]);
    cudaFree(h->p2p_region);
    cudaFree(h->p2p_ctl);
    h->zbuf = nullptr;
    h->P = nullptr;
    h->Q = nullptr;
  }
  if (h->nvls) nvls_teardown(&h->nv);
  cudaFree(h->nv_ctl);
  if (h->nvls) {  // these live in the NVLS region, not in cudaMalloc memory
    h->zbuf = nullptr;
    h->P = nullptr;
    h->Q = nullptr;
  }
  if (h->comm) {
    for (void* r : h->nccl_regs)
      if (g_nccl.CommDeregister) g_nccl.CommDeregister(h->comm, r);
  }
  for (void* p : h->nccl_allocs) {
    if (p == h->zbuf) h->zbuf = nullptr;
    if (p == h->P) h->P = nullptr;
    if (p == h->S) h->S = nullptr;
    if (p == h->Q) h->Q = nullptr;
    if (g_nccl.MemFree) g_nccl.MemFree(p);
  }
  if (h->comm) g_nccl.CommDestroy(h->comm);
  for (auto& v : h->tev)
    for (cudaEvent_t e : v) cudaEventDestroy(e);
  if (h->evFork) cudaEventDestroy(h->evFork);
  if (h->evJoin) cudaEventDestroy(h->evJoin);
  if (h->evDone) cudaEventDestroy(h->evDone);
  if (h->sB) cudaStreamDestroy(h->sB);
  if (h->sIO) cudaStreamDestroy(h->sIO);
  if (h->sH2D) cudaStreamDestroy(h->sH2D);
  if (h->sD2H) cudaStreamDestroy(h->sD2H);
  for (int i = 0; i < 2; ++i) {
    if (h->evStaged[i]) cudaEventDestroy(h->evStaged[i]);
    if (h->evUsed[i]) cudaEventDestroy(h->evUsed[i]);
    if (h->evZread[i]) cudaEventDestroy(h->evZread[i]);
  }
  if (h->evAsync) cudaEventDestroy(h->evAsync);
  cudaFree(h->G2);
  cudaFree(h->W);
  cudaFree(h->zbuf);
  cudaFree(h->P);
  cudaFree(h->S);
  cudaFree(h->Q);
  cudaFree(h->C);
  cudaFree(h->G);
  cudaFree(h->U);
  cudaFree(h->push_scratch);
  cudaFree(h->nonfinite);
  for (int i = 0; i < 2; ++i) cudaFree(h->perm_dev[i]);
  cudaFree(h->mlp_A1);
  cudaFree(h->mlp_DA);
  cudaFree(h->mlp_E);
  cudaFree(h->mlp_PL);
  cudaFree(h->mlp_bar);
  if (h->perm_next.valid()) h->perm_next.wait();
  for (int i = 0; i < 2; ++i) {
    if (h->perm_host[i]) cudaFreeHost(h->perm_host[i]);
    if (h->perm_ev[i]) cudaEventDestroy(h->perm_ev[i]);
  }
  delete h;
}

sma_status ensure_G(sma_handle* h) {
  if (h->G) return SMA_OK;
  CUDA_TRY(cudaMalloc(&h->G, sizeof(float) * (size_t)h->r * h->d_pad));
  CUDA_TRY(cudaMemset(h->G, 0, sizeof(float) * (size_t)h->r * h->d_pad));
  return SMA_OK;
}

void set_gptr(sma_handle* h, int slot, const float* p) {
  if (h->gptr[slot] != p) {
    h->gptr[slot] = p;
    ++h->ver;
  }
}

// A registration from any path but sma_stage_grads_host leaves the staged set.
void leave_staged_set(sma_handle* h) {
  h->cur_set = -1;
  h->stage_wait = false;
}

sma_status mark_done(sma_handle* h, cudaStream_t s) {
  CUDA_TRY(cudaEventRecord(h->evDone, s));
  h->any_work = true;
  return SMA_OK;
}

// Wait for everything the handle enqueued, on the host (rounds, staged
// host-to-device copies, asynchronous read-backs).
sma_status sync_handle(sma_handle* h) {
  if (h->any_work) CUDA_TRY(cudaEventSynchronize(h->evDone));
  if (h->h2d_pending) {
    CUDA_TRY(cudaStreamSynchronize(h->sH2D));
    h->h2d_pending = false;
  }
  if (h->async_pending) {
    CUDA_TRY(cudaEventSynchronize(h->evAsync));
    h->async_pending = false;
  }
  return SMA_OK;
}

// Cross-stream ordering of a round enqueued on s with the pipelined intake and
// read-back: wait for the staged gradient copies it reads, and -- if it writes
// the z_prev half (writes_z) -- for an asynchronous read-back of the z value
// that half still holds; afterwards, mark the gradient set as read by s.
sma_status pre_round(sma_handle* h, cudaStream_t s, bool writes_z) {
  if (h->stage_wait) {
    CUDA_TRY(cudaStreamWaitEvent(s, h->evStaged[h->cur_set], 0));
    h->stage_wait = false;
  }
  const int b = 1 - h->cur;
  if (writes_z && h->zread_pending[b]) {
    CUDA_TRY(cudaStreamWaitEvent(s, h->evZread[b], 0));
    h->zread_pending[b] = false;
  }
  return SMA_OK;
}
sma_status post_round(sma_handle* h, cudaStream_t s) {
  if (h->cur_set >= 0) {
    CUDA_TRY(cudaEventRecord(h->evUsed[h->cur_set], s));
    h->used_rec[h->cur_set] = true;
  }
  return SMA_OK;
}

sma_status check_nonfinite(sma_handle* h) {
  if (!h->check) return SMA_OK;
  int flag = 0;
  CUDA_TRY(cudaMemcpy(&flag, h->nonfinite, sizeof(int), cudaMemcpyDeviceToHost));
  if (flag) return fail(SMA_ERR_NONFINITE, "a non-finite value was produced by an SMA round");
  return SMA_OK;
}

// Next (start, stop) event pair of `phase` (nullptr unless SMA_FLAG_TIMING).
sma_status timer_pair(sma_handle* h, int phase, cudaEvent_t** out) {
  *out = nullptr;
  if (!h->timing) return SMA_OK;
  auto& v = h->tev[phase];
  size_t& used = h->tused[phase];
  while (used + 2 > v.size()) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    v.push_back(e);
  }
  *out = &v[used];
  used += 2;
  return SMA_OK;
}

// SMA_FLAG_P2P_PUSH: the partial destined for local buffer `out` goes, shard by
// shard, into slot `rank` of the same buffer on every rank (same region offsets).
void fill_push(const sma_handle* h, const float* out, ReplicaArgs* a) {
  const size_t off = (size_t)(reinterpret_cast<const char*>(out) - h->p2p_region);
  for (int g = 0; g < h->cfg.world; ++g) a->push.p[g] = reinterpret_cast<float*>(h->p2p_base[g] + off);
  a->push_n = h->cfg.world;
  a->push_rank = h->cfg.rank;
  a->push_shard = h->shard_len;
}

sma_status replica_launch(sma_handle* h, int mode, float* out, cudaStream_t s, int sms = 0) {
  NvtxRange nvtx("sma.replica_kernel");
  if (sms <= 0) sms = h->num_sms;
  ReplicaArgs a{};
  a.W = h->W;
  a.ld = h->d_pad;
  a.r = h->r;
  for (int i = 0; i < h->r; ++i) a.g.p[i] = h->gptr[i];
  a.d = h->cfg.d;
  a.n4 = h->n4;
  a.z = h->z();
  a.zprev_next = h->zprev();
  a.out = out;
  a.C = h->matc ? h->C : nullptr;
  a.alpha = h->alpha;
  a.gamma = h->gamma;
  a.mu = h->mu;
  a.nonfinite = h->check ? h->nonfinite : nullptr;
  a.U = h->U;
  a.alpha_g = h->alpha_g;
  if (h->push && out) fill_push(h, out, &a);
  cudaEvent_t* tp = nullptr;
  STATUS_TRY(timer_pair(h, SMA_PHASE_REPLICA, &tp));
  if (tp) CUDA_TRY(cudaEventRecord(tp[0], s));
  // a reference model u_g is updated even on a GPU without learners
  if (h->r > 0 || mode == kHierA || mode == kHierB) {
    CUDA_TRY(launch_replica_step(mode, h->tma, a, sms, s));
    ++h->launches;
    if (h->matc) {
      CUDA_TRY(launch_reduce_corrections(mode, a, sms, s));
      ++h->launches;
    }
  } else if (mode == kFused) {
    CUDA_TRY(launch_replica_step(mode, false, a, sms, s));  // z <- z + mu (z - z_prev)
    ++h->launches;
  } else if (h->push) {  // no local learners: push a zero partial
    CUDA_TRY(cudaMemsetAsync(h->push_scratch, 0, sizeof(float) * h->d_pad, s));
    ReplicaArgs z{};
    z.n4 = h->n4;
    fill_push(h, out, &z);
    CUDA_TRY(launch_push_partial(h->push_scratch, z, h->num_sms, s));
    ++h->launches;
  } else {
    CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(float) * h->d_pad, s));
  }
  if (tp) CUDA_TRY(cudaEventRecord(tp[1], s));
  return SMA_OK;
}

// Mode B shard update z' = (z + alpha_s S) + coef_b (z - z_prev): flat Alg. 1
// emits Q = sum_j (w_j' - z) unscaled (alpha_s = alpha, coef_b = mu - alpha k);
// the two-level rule emits pre-scaled partials (alpha_s = 1; coef_b in mode_b_coef).
float zsync_alpha(const sma_handle* h) { return h->hier ? 1.f : h->alpha; }
float mode_b_coef(const sma_handle* h) {
  if (!h->hier) return h->mu - h->alpha * (float)h->cfg.k;
  int32_t f0 = 0, r0 = 0;
  sma_plan_local_replicas(h->cfg.k, h->cfg.world, 0, &f0, &r0);
  // z^{i+1} = z^i + sum_g E_g - (alpha_l r_0 + alpha_g (n-1)) delta + mu delta
  return h->mu - (h->alpha * (float)r0 + h->alpha_g * (float)(h->cfg.world - 1));
}

// a6-a8 on stream s: reduce-scatter the per-GPU partial, update this GPU's
// shard of z in place into the z_prev half, all-gather z.  Each phase is
// bracketed by timing events with SMA_FLAG_TIMING.
sma_status enqueue_zsync(sma_handle* h, int mode, const float* partial, float coef_b,
                         cudaStream_t s) {
  NvtxRange nvtx(h->p2p ? "sma.zsync_p2p" : h->nvls ? "sma.zsync_nvls" : "sma.zsync_nccl");
  const size_t cnt = (size_t)h->shard_len;
  cudaEvent_t* tp = nullptr;
  if (h->p2p) {  // a6-a8 in one kernel over IPC-mapped peer memory
    P2PArgs a{};
    for (int g = 0; g < h->cfg.world; ++g) a.base[g] = h->p2p_base[g];
    a.off_flags = 0;
    a.off_part = reinterpret_cast<const char*>(partial) - h->p2p_region;
    a.off_z = reinterpret_cast<const char*>(h->z()) - h->p2p_region;
    a.off_zprev = reinterpret_cast<const char*>(h->zprev()) - h->p2p_region;
    a.off4 = h->shard_off / 4;
    a.len4 = h->shard_len / 4;
    a.alpha = zsync_alpha(h);
    a.mu = h->mu;
    a.coef_b = coef_b;
    a.n = h->cfg.world;
    a.rank = h->cfg.rank;
    a.ctl = h->p2p_ctl;
    a.nonfinite = h->check ? h->nonfinite : nullptr;
    a.push = h->push ? 1 : 0;
    // SMA_P2P_EMULATE_N=N (measurement only; ignored unless world == 1): see sma_p2p.cu
    static const int emu_n = [] {
      const char* e = getenv("SMA_P2P_EMULATE_N");
      const int v = e ? atoi(e) : 0;
      return v >= 2 && v <= kMaxP2PRanks ? v : 0;
    }();
    a.emu_n = h->cfg.world == 1 ? emu_n : 0;
    STATUS_TRY(timer_pair(h, SMA_PHASE_FUSED_ZSYNC, &tp));
    if (tp) CUDA_TRY(cudaEventRecord(tp[0], s));
    // persistent grid: SMA_P2P_CTAS_PER_SM x #SMs CTAs (default 4); in Mode B
    // they share the SMs with the concurrent replica kernel
    static const int per_sm = [] {
      const char* e = getenv("SMA_P2P_CTAS_PER_SM");
      const int v = e ? atoi(e) : 4;
      return v >= 1 && v <= 8 ? v : 4;
    }();
    // SMA_P2P_CTAS (experiments): an absolute cap on the grid, e.g. the few SMs
    // that saturate NVLink while the concurrent replica kernel keeps the rest
    static const int cap = [] {
      const char* e = getenv("SMA_P2P_CTAS");
      return e ? atoi(e) : 0;
    }();
    CUDA_TRY(launch_zsync_p2p(mode, a, cap > 0 ? cap : per_sm * h->num_sms, s));  // Mode B: high-priority stream
    if (tp) CUDA_TRY(cudaEventRecord(tp[1], s));
    return SMA_OK;
  }
  if (h->nvls) {  // a6-a8 in one multicast kernel
    NvlsArgs a{};
    const size_t part_off = (size_t)(reinterpret_cast<const char*>(partial) -
                                     reinterpret_cast<const char*>(h->nv.uc));
    a.part_mc = reinterpret_cast<const float*>(h->nv.mcva + part_off);
    a.znext_mc = reinterpret_cast<float*>(h->nv.mcva + h->nv_off_z) + (int64_t)(1 - h->cur) * h->d_pad;
    a.z = h->z();
    a.zprev = h->zprev();
    a.off4 = h->shard_off / 4;
    a.len4 = h->shard_len / 4;
    a.alpha = zsync_alpha(h);
    a.mu = h->mu;
    a.coef_b = coef_b;
    a.flag_uc = reinterpret_cast<unsigned*>(h->nv.uc);
    a.flag_mc = reinterpret_cast<unsigned*>(h->nv.mcva);
    a.expect = h->nv_ctl;
    a.done_ctr = h->nv_ctl + 2;
    a.n = h->cfg.world;
    a.nonfinite = h->check ? h->nonfinite : nullptr;
    STATUS_TRY(timer_pair(h, SMA_PHASE_NVLS_ZSYNC, &tp));
    if (tp) CUDA_TRY(cudaEventRecord(tp[0], s));
    CUDA_TRY(launch_zsync_nvls(mode, a, h->overlap ? (h->sync_sms > 0 ? h->sync_sms : 1) : h->num_sms, s));
    if (tp) CUDA_TRY(cudaEventRecord(tp[1], s));
    return SMA_OK;
  }
  STATUS_TRY(timer_pair(h, SMA_PHASE_REDUCE_SCATTER, &tp));
  if (tp) CUDA_TRY(cudaEventRecord(tp[0], s));
  NCCL_TRY(g_nccl.ReduceScatter(partial, h->S, cnt, ncclFloat32, ncclSum, h->comm, s));
  if (tp) CUDA_TRY(cudaEventRecord(tp[1], s));
  STATUS_TRY(timer_pair(h, SMA_PHASE_SHARD_UPDATE, &tp));
  if (tp) CUDA_TRY(cudaEventRecord(tp[0], s));
  CUDA_TRY(launch_zsync(mode, h->S, h->z() + h->shard_off, h->zprev() + h->shard_off,
                        h->shard_len / 4, zsync_alpha(h), h->mu, coef_b,
                        h->check ? h->nonfinite : nullptr, h->num_sms, s));
  if (tp) CUDA_TRY(cudaEventRecord(tp[1], s));
  STATUS_TRY(timer_pair(h, SMA_PHASE_ALL_GATHER, &tp));
  if (tp) CUDA_TRY(cudaEventRecord(tp[0], s));
  NCCL_TRY(g_nccl.AllGather(h->zprev() + h->shard_off, h->zprev(), cnt, ncclFloat32, h->comm, s));
  if (tp) CUDA_TRY(cudaEventRecord(tp[1], s));
  return SMA_OK;
}

// Mode B prologue: Q^i of the current state into Q[qi] --
// or, with SMA_FLAG_P2P_PUSH, into the scratch buffer and from there into
// slot `rank` of every owner's Q[qi].
sma_status enqueue_q_prologue(sma_handle* h, cudaStream_t s) {
  const float scale = !h->hier ? 1.f : (h->U ? h->alpha_g : h->alpha);
  float* q = h->Q + (int64_t)h->qi * h->d_pad;
  CUDA_TRY(launch_q_prologue(h->W, h->d_pad, h->r, h->zprev(), h->push ? h->push_scratch : q, h->n4,
                             h->U, scale, h->num_sms, s));
  ++h->launches;
  if (h->push) {
    ReplicaArgs a{};
    a.n4 = h->n4;
    fill_push(h, q, &a);
    CUDA_TRY(launch_push_partial(h->push_scratch, a, h->num_sms, s));
    ++h->launches;
  }
  h->q_dirty = false;
  return SMA_OK;
}

// The body of one round, enqueued on stream s (capturable without a learner).
// `learner` (optional) enqueues this round's learner gradients (a2') on s
// before the replica kernel; in Mode B it is enqueued AFTER the z-sync fork, so
// the global synchronisation runs concurrently with the learning tasks -- the
// paper's overlap of GlobalSync with Learning (fig:dependencies f).
using LearnerFn = std::function<sma_status(cudaStream_t)>;
sma_status enqueue_round(sma_handle* h, cudaStream_t s, const LearnerFn* learner = nullptr) {
  if (learner && !(h->collective && h->overlap)) STATUS_TRY((*learner)(s));
  if (!h->collective) {  // n == 1: a3-a7 fused in one kernel
    STATUS_TRY(replica_launch(h, kFused, nullptr, s));
  } else if (!h->overlap) {  // Mode A: paper order (fig:dependencies d/e)
    STATUS_TRY(replica_launch(h, h->U ? kHierA : kPartialA, h->P, s));
    STATUS_TRY(enqueue_zsync(h, kPartialA, h->P, 0.f, s));
    h->launches += 1;  // zsync (NCCL's own kernels are not counted)
  } else {  // Mode B: z-sync(i) on sB  ||  replica kernel(i) on s
    float* Qcur = h->Q + (int64_t)h->qi * h->d_pad;
    float* Qnext = h->Q + (int64_t)(1 - h->qi) * h->d_pad;
    const float coef_b = mode_b_coef(h);
    const int rmode = !h->hier ? kPartialB : (h->U ? kHierB : kHierB0);
    CUDA_TRY(cudaEventRecord(h->evFork, s));
    CUDA_TRY(cudaStreamWaitEvent(h->sB, h->evFork, 0));
    STATUS_TRY(enqueue_zsync(h, kPartialB, Qcur, coef_b, h->sB));
    CUDA_TRY(cudaEventRecord(h->evJoin, h->sB));
    if (learner) STATUS_TRY((*learner)(s));   // Learning(i) || GlobalSync(i)
    STATUS_TRY(replica_launch(h, rmode, Qnext, s, h->num_sms - h->sync_sms));
    CUDA_TRY(cudaStreamWaitEvent(s, h->evJoin, 0));
    h->launches += 1;  // zsync
  }
  return SMA_OK;
}

void advance(sma_handle* h) {
  h->cur ^= 1;
  if (h->overlap) h->qi ^= 1;
}

sma_status alloc_zero(float** p, size_t n) {
  CUDA_TRY(cudaMalloc(p, sizeof(float) * n));
  CUDA_TRY(cudaMemset(*p, 0, sizeof(float) * n));
  return SMA_OK;
}

// Collective buffer: ncclMemAlloc + ncclCommRegister when available (and
// SMA_NCCL_MEMALLOC != 0), else cudaMalloc.  Zero-filled.
sma_status alloc_coll(sma_handle* h, float** p, size_t n) {
  const char* e = getenv("SMA_NCCL_MEMALLOC");
  // a 1-rank communicator gains nothing from registration (no NVLS team)
  const bool use = h->cfg.world > 1 && g_nccl.MemAlloc && g_nccl.MemFree && !(e && e[0] == '0');
  if (!use) return alloc_zero(p, n);
  void* q = nullptr;
  if (g_nccl.MemAlloc(&q, sizeof(float) * n) != ncclSuccess || !q) {
    cudaGetLastError();            // NCCL could not provide NVLS-capable memory:
    return alloc_zero(p, n);       // plain device memory works for every algorithm
  }
  h->nccl_allocs.push_back(q);
  *p = static_cast<float*>(q);
  CUDA_TRY(cudaMemset(q, 0, sizeof(float) * n));
  if (g_nccl.CommRegister) {
    void* reg = nullptr;
    if (g_nccl.CommRegister(h->comm, q, sizeof(float) * n, &reg) == ncclSuccess && reg)
      h->nccl_regs.push_back(reg);
  }
  return SMA_OK;
}

sma_status create_impl(const sma_config* cfg, const float* w0, sma_handle* h) {
  h->cfg = *cfg;
  h->dev = cfg->device;
  h->alpha = cfg->alpha;
  h->gamma = cfg->gamma;
  h->mu = cfg->mu;
  const uint32_t f = cfg->flags;
  h->collective = cfg->world > 1 || (f & SMA_FLAG_FORCE_COLLECTIVE);
  h->overlap = h->collective && (f & SMA_FLAG_OVERLAP);
  h->matc = (f & SMA_FLAG_MATERIALIZE_C) != 0;
  if ((f & SMA_FLAG_KERNEL_TMA) && (f & SMA_FLAG_KERNEL_LDG))
    return fail(SMA_ERR_INVALID_ARG, "SMA_FLAG_KERNEL_TMA and SMA_FLAG_KERNEL_LDG are exclusive");
  h->timing = (f & SMA_FLAG_TIMING) != 0;
  h->graphs = (f & SMA_FLAG_CUDA_GRAPH) != 0;  // used only while timing is off
  h->check = (f & SMA_FLAG_CHECK_FINITE) != 0;
  h->nvls = (f & SMA_FLAG_NVLS_ZSYNC) != 0;
  h->p2p = (f & SMA_FLAG_P2P_ZSYNC) != 0;
  if (h->p2p && h->nvls)
    return fail(SMA_ERR_INVALID_ARG, "SMA_FLAG_P2P_ZSYNC and SMA_FLAG_NVLS_ZSYNC are exclusive");
  if (h->p2p && !h->collective)
    return fail(SMA_ERR_INVALID_ARG, "SMA_FLAG_P2P_ZSYNC needs world > 1 or SMA_FLAG_FORCE_COLLECTIVE");
  h->push = (f & SMA_FLAG_P2P_PUSH) != 0;
  if (h->push && (!h->p2p || h->matc || (f & SMA_FLAG_KERNEL_TMA)))
    return fail(SMA_ERR_INVALID_ARG,
                "SMA_FLAG_P2P_PUSH needs SMA_FLAG_P2P_ZSYNC and excludes MATERIALIZE_C / KERNEL_TMA");
  if (h->p2p && cfg->world > kMaxP2PRanks)
    return fail(SMA_ERR_INVALID_ARG, "SMA_FLAG_P2P_ZSYNC supports at most %d ranks", kMaxP2PRanks);
  if (h->nvls && !h->collective)
    return fail(SMA_ERR_INVALID_ARG, "SMA_FLAG_NVLS_ZSYNC needs world > 1 or SMA_FLAG_FORCE_COLLECTIVE");
  h->d_pad = sma_plan_d_pad(cfg->d, cfg->world);
  h->n4 = h->d_pad / 4;
  STATUS_TRY(sma_plan_local_replicas(cfg->k, cfg->world, cfg->rank, &h->j0, &h->r));
  STATUS_TRY(sma_plan_shard_range(cfg->d, cfg->world, cfg->rank, &h->shard_off, &h->shard_len));
  // Kernel policy: the direct-load kernel on a full grid is the fastest at every
  // measured size (profiles/r01_ldg_variants.jsonl); the TMA ring on request.
  h->tma = (f & SMA_FLAG_KERNEL_TMA) != 0;
  if (h->r > SMA_MAX_LOCAL_REPLICAS)
    return fail(SMA_ERR_INVALID_ARG, "%d replicas on rank %d exceeds SMA_MAX_LOCAL_REPLICAS=%d",
                h->r, cfg->rank, SMA_MAX_LOCAL_REPLICAS);
  if (h->matc && h->overlap)
    return fail(SMA_ERR_INVALID_ARG, "SMA_FLAG_MATERIALIZE_C is not combined with SMA_FLAG_OVERLAP");
  h->hier = (f & SMA_FLAG_HIERARCHICAL) != 0;
  if (h->hier && (h->matc || h->tma))
    return fail(SMA_ERR_INVALID_ARG,
                "SMA_FLAG_HIERARCHICAL is not combined with SMA_FLAG_MATERIALIZE_C or SMA_FLAG_KERNEL_TMA");
  // R20 default: z's total pull alpha_l r + alpha_g (n-1) = 1 at alpha_l = 1/(2r)
  h->alpha_g = 1.f / (2.f * (float)(cfg->world > 1 ? cfg->world - 1 : 1));

  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (cfg->device < 0 || cfg->device >= ndev)
    return fail(SMA_ERR_INVALID_ARG, "device %d not present (%d devices)", cfg->device, ndev);
  DeviceGuard guard(h->dev);
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, h->dev));
  if (prop.major < 10)
    return fail(SMA_ERR_CUDA, "device %d is sm_%d%d; libsma is built for sm_100a only", h->dev,
                prop.major, prop.minor);
  h->num_sms = prop.multiProcessorCount;

  {  // the z-sync stream gets the highest priority, so in Mode B the CTA
     // scheduler dispatches NCCL's / the shard update's CTAs ahead of the
     // (full-grid) replica kernel's remaining CTAs instead of after them
    int least = 0, greatest = 0;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CUDA_TRY(cudaStreamCreateWithPriority(&h->sB, cudaStreamNonBlocking, greatest));
  }
  CUDA_TRY(cudaStreamCreateWithFlags(&h->sIO, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&h->evFork, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&h->evJoin, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&h->evDone, cudaEventDisableTiming));
  const size_t dp = (size_t)h->d_pad;
  if (h->collective && !h->p2p) {  // the communicator first: the collective buffers come from NCCL
    if (!nccl_load()) return fail(SMA_ERR_NCCL, "cannot load NCCL: %s", g_nccl.why.c_str());
    ncclUniqueId id;
    if (cfg->world > 1) {
      memcpy(&id, cfg->nccl_id, sizeof id);
    } else {
      NCCL_TRY(g_nccl.GetUniqueId(&id));
    }
    NCCL_TRY(g_nccl.CommInitRank(&h->comm, cfg->world, id, cfg->rank));
    if (const char* e = getenv("SMA_SYNC_SMS")) h->sync_sms = atoi(e);
    if (h->sync_sms < 0) h->sync_sms = 0;
    if (h->sync_sms > h->num_sms - 1) h->sync_sms = h->num_sms - 1;
  }
  STATUS_TRY(alloc_zero(&h->W, dp * (h->r > 0 ? h->r : 1)));
  if (h->p2p) {
    // [flags (4 KB) | P, or Q[2] | z[2]] in one IPC-exportable allocation
    h->p2p_off_part = 4096;
    h->p2p_off_z = h->p2p_off_part + sizeof(float) * dp * (h->overlap ? 2 : 1);
    const size_t bytes = h->p2p_off_z + sizeof(float) * 2 * dp;
    CUDA_TRY(cudaMalloc(&h->p2p_region, bytes));
    CUDA_TRY(cudaMemset(h->p2p_region, 0, bytes));
    h->zbuf = reinterpret_cast<float*>(h->p2p_region + h->p2p_off_z);
    if (h->overlap)
      h->Q = reinterpret_cast<float*>(h->p2p_region + h->p2p_off_part);
    else
      h->P = reinterpret_cast<float*>(h->p2p_region + h->p2p_off_part);
    CUDA_TRY(cudaMalloc(&h->p2p_ctl, 4 * sizeof(unsigned)));
    CUDA_TRY(cudaMemset(h->p2p_ctl, 0, 4 * sizeof(unsigned)));
    h->p2p_base.assign(cfg->world, nullptr);
    h->p2p_base[cfg->rank] = h->p2p_region;
    if (h->push) STATUS_TRY(alloc_zero(&h->push_scratch, dp));
    h->p2p_connected = cfg->world == 1;  // a single rank maps only itself
  } else if (h->nvls) {
    // [flags (4 KB) | P, or Q[2] | z[2]] bound to one multicast object per rank
    h->nv_off_part = 4096;
    h->nv_off_z = h->nv_off_part + sizeof(float) * dp * (h->overlap ? 2 : 1);
    const size_t bytes = h->nv_off_z + sizeof(float) * 2 * dp;
    std::string key;
    {
      uint64_t x = 1469598103934665603ull;  // FNV-1a of the NCCL id: rendezvous name
      const unsigned char* b = reinterpret_cast<const unsigned char*>(cfg->nccl_id);
      if (cfg->world > 1)
        for (int i = 0; i < SMA_NCCL_ID_BYTES; ++i) x = (x ^ b[i]) * 1099511628211ull;
      else
        x ^= (uint64_t)getpid() << 20 ^ (uint64_t)(uintptr_t)h;
      char buf[32];
      snprintf(buf, sizeof buf, "%016llx", (unsigned long long)x);
      key = buf;
    }
    int* bar = nullptr;
    CUDA_TRY(cudaMalloc(&bar, sizeof(int) * cfg->world));
    auto barrier = [&](std::string* err) -> bool {
      if (cfg->world == 1) return true;
      if (g_nccl.AllReduce(bar, bar, 1, ncclInt32, ncclSum, h->comm, h->sIO) != ncclSuccess ||
          cudaStreamSynchronize(h->sIO) != cudaSuccess) {
        *err = "NCCL barrier failed";
        return false;
      }
      return true;
    };
    std::string err;
    const bool ok = nvls_setup(&h->nv, h->dev, cfg->rank, cfg->world, bytes, key, barrier, &err);
    cudaFree(bar);
    if (!ok) return fail(SMA_ERR_CUDA, "NVLS z-sync setup: %s", err.c_str());
    h->zbuf = reinterpret_cast<float*>(h->nv.uc + h->nv_off_z);
    if (h->overlap)
      h->Q = reinterpret_cast<float*>(h->nv.uc + h->nv_off_part);
    else
      h->P = reinterpret_cast<float*>(h->nv.uc + h->nv_off_part);
    CUDA_TRY(cudaMalloc(&h->nv_ctl, 4 * sizeof(unsigned)));
    CUDA_TRY(cudaMemset(h->nv_ctl, 0, 4 * sizeof(unsigned)));
  } else if (h->collective) {
    // z (the all-gather target), the partial(s) and the reduce-scatter output
    // are NCCL-allocated and registered, so NCCL can use zero-copy NVLS
    // (in-switch reduction / multicast) on NVSwitch systems.
    STATUS_TRY(alloc_coll(h, &h->zbuf, 2 * dp));
    STATUS_TRY(alloc_coll(h, &h->S, (size_t)h->shard_len));
    if (h->overlap)
      STATUS_TRY(alloc_coll(h, &h->Q, 2 * dp));
    else
      STATUS_TRY(alloc_coll(h, &h->P, dp));
  } else {
    STATUS_TRY(alloc_zero(&h->zbuf, 2 * dp));
  }
  if (h->matc) STATUS_TRY(alloc_zero(&h->C, dp * (h->r > 0 ? h->r : 1)));
  if (h->hier && h->collective && cfg->rank > 0) STATUS_TRY(alloc_zero(&h->U, dp));
  CUDA_TRY(cudaMalloc(&h->nonfinite, sizeof(int)));
  CUDA_TRY(cudaMemset(h->nonfinite, 0, sizeof(int)));

  // Alg. 1 line 1-2 (R2) and R3: z = z_prev = w_j = w0; padding stays 0.
  CUDA_TRY(cudaMemcpy(h->zbuf, w0, sizeof(float) * cfg->d, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(h->zbuf + dp, h->zbuf, sizeof(float) * dp, cudaMemcpyDeviceToDevice));
  if (h->r > 0) CUDA_TRY(launch_broadcast_rows(h->W, h->d_pad, h->r, h->zbuf, h->n4, h->num_sms, 0));
  if (h->U)  // R20: every reference model starts as the initial model
    CUDA_TRY(cudaMemcpy(h->U, h->zbuf, sizeof(float) * dp, cudaMemcpyDeviceToDevice));
  CUDA_TRY(cudaDeviceSynchronize());

  return SMA_OK;
}
}  // namespace

// ======================================================================= ABI
extern "C" {

int sma_abi_version(void) { return SMA_ABI_VERSION; }

sma_status sma_nccl_unique_id(void* out) {
  if (!out) return fail(SMA_ERR_INVALID_ARG, "NULL output");
  if (!nccl_load()) return fail(SMA_ERR_NCCL, "cannot load NCCL: %s", g_nccl.why.c_str());
  ncclUniqueId id;
  NCCL_TRY(g_nccl.GetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return SMA_OK;
}

sma_status sma_create(const sma_config* cfg, const float* w0_host, sma_handle** out) {
  if (!out) return fail(SMA_ERR_INVALID_ARG, "NULL out");
  *out = nullptr;
  if (!cfg || !w0_host) return fail(SMA_ERR_INVALID_ARG, "NULL config or w0");
  if (cfg->d < 1) return fail(SMA_ERR_INVALID_ARG, "d must be >= 1 (got %lld)", (long long)cfg->d);
  if (cfg->k < 1) return fail(SMA_ERR_INVALID_ARG, "k must be >= 1 (got %d)", cfg->k);
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world)
    return fail(SMA_ERR_INVALID_ARG, "bad rank/world %d/%d", cfg->rank, cfg->world);
  if (!finite_f(cfg->alpha) || !finite_f(cfg->gamma) || !finite_f(cfg->mu))
    return fail(SMA_ERR_INVALID_ARG, "non-finite hyper-parameter");
  if (cfg->world > 1 && !cfg->nccl_id && !(cfg->flags & SMA_FLAG_P2P_ZSYNC))
    return fail(SMA_ERR_INVALID_ARG, "world > 1 requires nccl_id (or SMA_FLAG_P2P_ZSYNC)");
  sma_handle* h = new sma_handle();
  sma_status st = create_impl(cfg, w0_host, h);
  if (st != SMA_OK) {
    const std::string msg = sma_last_error();  // free_all must not overwrite the cause
    free_all(h);
    fail(st, "%s", msg.c_str());
    return st;
  }
  *out = h;
  return SMA_OK;
}

void sma_destroy(sma_handle* h) {
  if (h) free_all(h);
}

sma_status sma_set_learner_grads(sma_handle* h, int32_t j, const float* g_dev) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  int slot;
  STATUS_TRY(local_slot(h, j, &slot));
  if (!g_dev || (reinterpret_cast<uintptr_t>(g_dev) & 15u))
    return fail(SMA_ERR_INVALID_ARG, "gradient pointer must be non-NULL and 16-byte aligned");
  set_gptr(h, slot, g_dev);
  leave_staged_set(h);
  return SMA_OK;
}

sma_status sma_set_learner_grads_host(sma_handle* h, int32_t j, const float* g_host, void* stream) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  int slot;
  STATUS_TRY(local_slot(h, j, &slot));
  if (!g_host) return fail(SMA_ERR_INVALID_ARG, "NULL gradient");
  DeviceGuard guard(h->dev);
  STATUS_TRY(ensure_G(h));
  cudaStream_t s = (cudaStream_t)stream;
  float* dst = h->G + (int64_t)slot * h->d_pad;
  CUDA_TRY(cudaMemcpyAsync(dst, g_host, sizeof(float) * h->cfg.d, cudaMemcpyHostToDevice, s));
  set_gptr(h, slot, dst);
  leave_staged_set(h);
  return mark_done(h, s);
}

sma_status sma_stage_grads_host(sma_handle* h, int32_t set, const float* const* g_host) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (set != 0 && set != 1) return fail(SMA_ERR_INVALID_ARG, "gradient set %d (0 or 1)", set);
  if (!g_host && h->r > 0) return fail(SMA_ERR_INVALID_ARG, "NULL pointer array");
  for (int i = 0; i < h->r; ++i)
    if (!g_host[i]) return fail(SMA_ERR_INVALID_ARG, "NULL gradient of local learner %d", i);
  if (h->r == 0) return SMA_OK;
  DeviceGuard guard(h->dev);
  const size_t dp = (size_t)h->d_pad;
  if (!h->G2) {
    CUDA_TRY(cudaMalloc(&h->G2, sizeof(float) * 2 * dp * (size_t)h->r));
    CUDA_TRY(cudaMemset(h->G2, 0, sizeof(float) * 2 * dp * (size_t)h->r));  // padding stays 0
  }
  if (!h->sH2D) CUDA_TRY(cudaStreamCreateWithFlags(&h->sH2D, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    if (!h->evStaged[i]) CUDA_TRY(cudaEventCreateWithFlags(&h->evStaged[i], cudaEventDisableTiming));
    if (!h->evUsed[i]) CUDA_TRY(cudaEventCreateWithFlags(&h->evUsed[i], cudaEventDisableTiming));
  }
  // the set is free again once the last round that read it has run
  if (h->used_rec[set]) CUDA_TRY(cudaStreamWaitEvent(h->sH2D, h->evUsed[set], 0));
  float* base = h->G2 + (size_t)set * dp * (size_t)h->r;
  for (int i = 0; i < h->r; ++i) {
    CUDA_TRY(cudaMemcpyAsync(base + (size_t)i * dp, g_host[i], sizeof(float) * h->cfg.d,
                             cudaMemcpyHostToDevice, h->sH2D));
    set_gptr(h, i, base + (size_t)i * dp);
  }
  CUDA_TRY(cudaEventRecord(h->evStaged[set], h->sH2D));
  h->cur_set = set;
  h->stage_wait = true;
  h->h2d_pending = true;
  return SMA_OK;
}

sma_status sma_get_central_async(sma_handle* h, float* z_host) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (!z_host) return fail(SMA_ERR_INVALID_ARG, "NULL output");
  DeviceGuard guard(h->dev);
  if (!h->sD2H) CUDA_TRY(cudaStreamCreateWithFlags(&h->sD2H, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i)
    if (!h->evZread[i]) CUDA_TRY(cudaEventCreateWithFlags(&h->evZread[i], cudaEventDisableTiming));
  if (!h->evAsync) CUDA_TRY(cudaEventCreateWithFlags(&h->evAsync, cudaEventDisableTiming));
  if (h->any_work) CUDA_TRY(cudaStreamWaitEvent(h->sD2H, h->evDone, 0));
  CUDA_TRY(cudaMemcpyAsync(z_host, h->z(), sizeof(float) * h->cfg.d, cudaMemcpyDeviceToHost, h->sD2H));
  CUDA_TRY(cudaEventRecord(h->evZread[h->cur], h->sD2H));
  h->zread_pending[h->cur] = true;
  CUDA_TRY(cudaEventRecord(h->evAsync, h->sD2H));
  h->async_pending = true;
  return SMA_OK;
}

sma_status sma_synchronize(sma_handle* h) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  DeviceGuard guard(h->dev);
  STATUS_TRY(sync_handle(h));
  return check_nonfinite(h);
}

sma_status sma_synth_grads(sma_handle* h, int64_t round, uint64_t seed, void* stream) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (round < 0) return fail(SMA_ERR_INVALID_ARG, "round < 0");
  if (h->r == 0) return SMA_OK;
  DeviceGuard guard(h->dev);
  STATUS_TRY(ensure_G(h));
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(launch_synth_grads(h->G, h->d_pad, h->r, h->j0, h->cfg.k, h->cfg.d, round, seed,
                              h->num_sms, s));
  ++h->launches;
  for (int i = 0; i < h->r; ++i) set_gptr(h, i, h->G + (int64_t)i * h->d_pad);
  leave_staged_set(h);
  return mark_done(h, s);
}

sma_status sma_step(sma_handle* h, void* stream) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  NvtxRange nvtx("sma_step");
  if (h->p2p && !h->p2p_connected)
    return fail(SMA_ERR_STATE, "SMA_FLAG_P2P_ZSYNC: call sma_p2p_connect on every rank first");
  for (int i = 0; i < h->r; ++i)
    if (!h->gptr[i])
      return fail(SMA_ERR_GRADS_MISSING, "learner %d has no registered gradient", h->j0 + i);
  DeviceGuard guard(h->dev);
  cudaStream_t s = (cudaStream_t)stream;
  STATUS_TRY(pre_round(h, s, true));
  if (h->overlap && h->q_dirty) STATUS_TRY(enqueue_q_prologue(h, s));
  if (h->graphs && !h->timing && s != nullptr) {
    const int key = h->cur;
    if (!h->gexec[key] || h->gver[key] != h->ver) {
      const int64_t launches0 = h->launches;
      cudaGraph_t graph = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      sma_status st = enqueue_round(h, s);
      cudaError_t ce = cudaStreamEndCapture(s, &graph);
      h->launches = launches0;
      if (st != SMA_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
      }
      if (ce != cudaSuccess)
        return fail(SMA_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
      if (h->gexec[key]) {
        cudaGraphExecDestroy(h->gexec[key]);
        h->gexec[key] = nullptr;
      }
      ce = cudaGraphInstantiate(&h->gexec[key], graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess)
        return fail(SMA_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
      h->gver[key] = h->ver;
    }
    CUDA_TRY(cudaGraphLaunch(h->gexec[key], s));
    h->launches += (h->collective ? 2 : 1) + (h->matc ? 1 : 0);
  } else {
    STATUS_TRY(enqueue_round(h, s));
  }
  STATUS_TRY(post_round(h, s));
  advance(h);
  return mark_done(h, s);
}

sma_status sma_step_local(sma_handle* h, void* stream) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  NvtxRange nvtx("sma_step_local");
  for (int i = 0; i < h->r; ++i)
    if (!h->gptr[i])
      return fail(SMA_ERR_GRADS_MISSING, "learner %d has no registered gradient", h->j0 + i);
  if (h->r == 0) return SMA_OK;
  DeviceGuard guard(h->dev);
  cudaStream_t s = (cudaStream_t)stream;
  STATUS_TRY(pre_round(h, s, false));
  ReplicaArgs a{};
  a.W = h->W;
  a.ld = h->d_pad;
  a.r = h->r;
  for (int i = 0; i < h->r; ++i) a.g.p[i] = h->gptr[i];
  a.d = h->cfg.d;
  a.n4 = h->n4;
  a.gamma = h->gamma;
  a.nonfinite = h->check ? h->nonfinite : nullptr;
  cudaEvent_t* tp = nullptr;
  STATUS_TRY(timer_pair(h, SMA_PHASE_REPLICA, &tp));
  if (tp) CUDA_TRY(cudaEventRecord(tp[0], s));
  CUDA_TRY(launch_replica_step(kLocal, false, a, h->num_sms, s));
  if (tp) CUDA_TRY(cudaEventRecord(tp[1], s));
  STATUS_TRY(post_round(h, s));
  ++h->launches;
  h->q_dirty = true;  // Mode B: Q^i = sum_j (w_j - z_prev) must be recomputed
  return mark_done(h, s);
}

sma_status sma_set_local_replicas(sma_handle* h, int32_t l_new, void* stream) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (l_new < 0 || l_new > SMA_MAX_LOCAL_REPLICAS)
    return fail(SMA_ERR_INVALID_ARG, "l_new=%d outside [0, %d]", l_new, SMA_MAX_LOCAL_REPLICAS);
  if (!h->collective && l_new == 0)
    return fail(SMA_ERR_INVALID_ARG, "a single-GPU handle needs at least one replica");
  if (h->learner && (int64_t)l_new * h->cfg.world * h->batch > h->n_samples)
    return fail(SMA_ERR_INVALID_ARG,
                "l_new=%d: %d learners x batch %d exceed the attached learner's %lld samples",
                l_new, l_new * h->cfg.world, h->batch, (long long)h->n_samples);
  DeviceGuard guard(h->dev);
  cudaStream_t s = (cudaStream_t)stream;
  STATUS_TRY(sync_handle(h));
  CUDA_TRY(cudaStreamSynchronize(s));
  const size_t dp = (size_t)h->d_pad;
  const int keep = h->r < l_new ? h->r : l_new;
  float* W2 = nullptr;
  STATUS_TRY(alloc_zero(&W2, dp * (l_new > 0 ? l_new : 1)));
  if (keep > 0)
    CUDA_TRY(cudaMemcpyAsync(W2, h->W, sizeof(float) * dp * keep, cudaMemcpyDeviceToDevice, s));
  if (l_new > keep)  // added learners start from the current central model
    CUDA_TRY(launch_broadcast_rows(W2 + dp * keep, h->d_pad, l_new - keep, h->z(), h->n4,
                                   h->num_sms, s));
  float* G2 = nullptr;
  float* C2 = nullptr;
  float* S2 = nullptr;  // the two staged gradient sets, [2][l_new][d_pad]
  if (h->G2) {
    STATUS_TRY(alloc_zero(&S2, 2 * dp * (l_new > 0 ? l_new : 1)));
    for (int set = 0; set < 2 && keep > 0; ++set)
      CUDA_TRY(cudaMemcpyAsync(S2 + (size_t)set * dp * l_new, h->G2 + (size_t)set * dp * h->r,
                               sizeof(float) * dp * keep, cudaMemcpyDeviceToDevice, s));
  }
  if (h->G) {
    STATUS_TRY(alloc_zero(&G2, dp * (l_new > 0 ? l_new : 1)));
    if (keep > 0)
      CUDA_TRY(cudaMemcpyAsync(G2, h->G, sizeof(float) * dp * keep, cudaMemcpyDeviceToDevice, s));
  }
  if (h->matc) STATUS_TRY(alloc_zero(&C2, dp * (l_new > 0 ? l_new : 1)));
  CUDA_TRY(cudaStreamSynchronize(s));
  // re-point registrations: internal buffers move, borrowed pointers stay
  const float* gp[SMA_MAX_LOCAL_REPLICAS] = {};
  for (int i = 0; i < keep; ++i) {
    const float* old = h->gptr[i];
    if (h->G && old >= h->G && old < h->G + dp * h->r)
      gp[i] = G2 + (old - h->G);
    else if (h->G2 && old >= h->G2 && old < h->G2 + 2 * dp * h->r) {
      const size_t off = (size_t)(old - h->G2), set = off / (dp * h->r);
      gp[i] = S2 + set * dp * l_new + (off - set * dp * h->r);
    } else
      gp[i] = old;
  }
  if (h->G2) {
    cudaFree(h->G2);
    h->G2 = S2;
    h->used_rec[0] = h->used_rec[1] = false;  // the copy above synchronised the stream
  }
  if (l_new > keep) leave_staged_set(h);  // added learners need a fresh registration
  cudaFree(h->W);
  h->W = W2;
  if (h->G) {
    cudaFree(h->G);
    h->G = G2;
  }
  if (h->matc) {
    cudaFree(h->C);
    h->C = C2;
  }
  for (int i = 0; i < SMA_MAX_LOCAL_REPLICAS; ++i) h->gptr[i] = gp[i];
  h->r = l_new;
  h->cfg.k = l_new * h->cfg.world;
  h->j0 = h->cfg.rank * l_new;
  h->q_dirty = true;
  ++h->ver;
  return mark_done(h, s);
}

static sma_status copy_out(sma_handle* h, const float* src, float* out, int out_is_device) {
  if (!out) return fail(SMA_ERR_INVALID_ARG, "NULL output");
  DeviceGuard guard(h->dev);
  STATUS_TRY(sync_handle(h));
  CUDA_TRY(cudaMemcpyAsync(out, src, sizeof(float) * h->cfg.d,
                           out_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->sIO));
  CUDA_TRY(cudaStreamSynchronize(h->sIO));
  return check_nonfinite(h);
}

sma_status sma_get_central(sma_handle* h, float* z_out, int out_is_device) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  return copy_out(h, h->z(), z_out, out_is_device);
}

sma_status sma_get_central_prev(sma_handle* h, float* out, int out_is_device) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  return copy_out(h, h->zprev(), out, out_is_device);
}

sma_status sma_get_replica(sma_handle* h, int32_t j, float* out, int out_is_device) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  int slot;
  STATUS_TRY(local_slot(h, j, &slot));
  return copy_out(h, h->W + (int64_t)slot * h->d_pad, out, out_is_device);
}

static sma_status copy_in(sma_handle* h, float* dst, const float* src, int in_is_device) {
  CUDA_TRY(cudaMemcpyAsync(dst, src, sizeof(float) * h->cfg.d,
                           in_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->sIO));
  return SMA_OK;
}

sma_status sma_set_replica(sma_handle* h, int32_t j, const float* w, int in_is_device) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  int slot;
  STATUS_TRY(local_slot(h, j, &slot));
  if (!w) return fail(SMA_ERR_INVALID_ARG, "NULL input");
  DeviceGuard guard(h->dev);
  STATUS_TRY(sync_handle(h));
  STATUS_TRY(copy_in(h, h->W + (int64_t)slot * h->d_pad, w, in_is_device));
  CUDA_TRY(cudaStreamSynchronize(h->sIO));
  h->q_dirty = true;
  return SMA_OK;
}

sma_status sma_set_central(sma_handle* h, const float* z, const float* z_prev, int in_is_device) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (!z || !z_prev) return fail(SMA_ERR_INVALID_ARG, "NULL input");
  DeviceGuard guard(h->dev);
  STATUS_TRY(sync_handle(h));
  STATUS_TRY(copy_in(h, h->z(), z, in_is_device));
  STATUS_TRY(copy_in(h, h->zprev(), z_prev, in_is_device));
  CUDA_TRY(cudaStreamSynchronize(h->sIO));
  h->q_dirty = true;
  return SMA_OK;
}

sma_status sma_replica_device_ptr(sma_handle* h, int32_t j, const float** w_dev) {
  if (!h || !w_dev) return fail(SMA_ERR_INVALID_ARG, "NULL argument");
  int slot;
  STATUS_TRY(local_slot(h, j, &slot));
  *w_dev = h->W + (int64_t)slot * h->d_pad;
  return SMA_OK;
}

sma_status sma_central_device_ptr(sma_handle* h, const float** z_dev) {
  if (!h || !z_dev) return fail(SMA_ERR_INVALID_ARG, "NULL argument");
  *z_dev = h->z();
  return SMA_OK;
}

sma_status sma_restart(sma_handle* h, void* stream) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  DeviceGuard guard(h->dev);
  cudaStream_t s = (cudaStream_t)stream;
  // Alg. 1 again with w0 := z; z_prev := z.
  CUDA_TRY(cudaMemcpyAsync(h->zprev(), h->z(), sizeof(float) * h->d_pad, cudaMemcpyDeviceToDevice, s));
  if (h->r > 0) {
    CUDA_TRY(launch_broadcast_rows(h->W, h->d_pad, h->r, h->z(), h->n4, h->num_sms, s));
    ++h->launches;
  }
  if (h->U)  // R20: the reference models restart from z as well
    CUDA_TRY(cudaMemcpyAsync(h->U, h->z(), sizeof(float) * h->d_pad, cudaMemcpyDeviceToDevice, s));
  h->q_dirty = true;
  return mark_done(h, s);
}

sma_status sma_set_alpha_global(sma_handle* h, float alpha_g) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (!h->hier) return fail(SMA_ERR_STATE, "not a SMA_FLAG_HIERARCHICAL handle");
  if (!finite_f(alpha_g)) return fail(SMA_ERR_INVALID_ARG, "non-finite alpha_g");
  h->alpha_g = alpha_g;
  h->q_dirty = true;  // Mode B: the pre-scaled partials change with alpha_g
  ++h->ver;
  return SMA_OK;
}

sma_status sma_get_reference(sma_handle* h, float* out, int out_is_device) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (!h->hier) return fail(SMA_ERR_STATE, "not a SMA_FLAG_HIERARCHICAL handle");
  return copy_out(h, h->U ? h->U : h->z(), out, out_is_device);
}

sma_status sma_set_reference(sma_handle* h, const float* u, int in_is_device) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (!h->hier) return fail(SMA_ERR_STATE, "not a SMA_FLAG_HIERARCHICAL handle");
  if (!h->U)
    return fail(SMA_ERR_STATE, "rank %d's reference model is z (use sma_set_central)", h->cfg.rank);
  if (!u) return fail(SMA_ERR_INVALID_ARG, "NULL input");
  DeviceGuard guard(h->dev);
  STATUS_TRY(sync_handle(h));
  STATUS_TRY(copy_in(h, h->U, u, in_is_device));
  CUDA_TRY(cudaStreamSynchronize(h->sIO));
  h->q_dirty = true;
  return SMA_OK;
}

sma_status sma_set_hparams(sma_handle* h, float alpha, float gamma, float mu) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (!finite_f(alpha) || !finite_f(gamma) || !finite_f(mu))
    return fail(SMA_ERR_INVALID_ARG, "non-finite hyper-parameter");
  h->alpha = alpha;
  h->gamma = gamma;
  h->mu = mu;
  if (h->hier) h->q_dirty = true;  // Mode B partials are pre-scaled by alpha_l (R20)
  ++h->ver;
  return SMA_OK;
}

sma_status sma_check_finite(sma_handle* h, int* flag) {
  if (!h || !flag) return fail(SMA_ERR_INVALID_ARG, "NULL argument");
  DeviceGuard guard(h->dev);
  STATUS_TRY(sync_handle(h));
  CUDA_TRY(cudaMemcpy(flag, h->nonfinite, sizeof(int), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemset(h->nonfinite, 0, sizeof(int)));
  return SMA_OK;
}

sma_status sma_learner_attach(sma_handle* h, int32_t kind, int32_t in_dim, int32_t hidden,
                              int32_t classes, int32_t batch, const float* X_dev,
                              const int32_t* y_dev, int64_t n_samples, uint64_t batch_seed) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (kind != 0 && kind != 1)
    return fail(SMA_ERR_INVALID_ARG, "learner kind %d not available (0 softmax, 1 mlp)", kind);
  if (in_dim < 1 || classes < 2 || classes > 32 || batch < 1 || batch > 64 || !X_dev || !y_dev ||
      (kind == 1 && (hidden < 1 || hidden > 4096)))
    return fail(SMA_ERR_INVALID_ARG, "bad learner arguments");
  const int64_t dl = kind == 0 ? (int64_t)classes * in_dim + classes
                               : (int64_t)hidden * in_dim + hidden + (int64_t)classes * hidden + classes;
  if (dl != h->cfg.d)
    return fail(SMA_ERR_INVALID_ARG, "d=%lld does not match the learner's %lld parameters",
                (long long)h->cfg.d, (long long)dl);
  if (n_samples < (int64_t)h->cfg.k * batch || n_samples > INT32_MAX)
    return fail(SMA_ERR_INVALID_ARG, "n_samples must be in [k*batch, 2^31)");
  // dynamic shared memory of every learner kernel (sma_kernels.cu, sma_learner_mlp.cu):
  // softmax logits + dW slice; MLP layer 1 (batch rows + up to 16 W1 rows), logits
  // (h row + W2 + b2), head (h, W2, e, staged a1 as float2)
  size_t smem_need = 0;
  if (kind == 0) {
    smem_need = sizeof(float) * ((size_t)in_dim + (size_t)batch * (64 + classes));
  } else {
    const size_t hd = (size_t)hidden, b = (size_t)batch, c = (size_t)classes;
    const size_t sm1 = sizeof(float) * ((b + 16) * (size_t)in_dim);
    const size_t smL = sizeof(float) * (hd + c * hd + c);
    const size_t sm2 = sizeof(float) * (b * hd + c * hd + b * c) + 16 + sizeof(float) * 2 * b * hd;
    smem_need = sm1 > smL ? sm1 : smL;
    if (sm2 > smem_need) smem_need = sm2;
  }
  if (smem_need > 200 * 1024)
    return fail(SMA_ERR_INVALID_ARG,
                "learner shapes need %zu B of shared memory in one kernel (limit 200 KB)", smem_need);
  DeviceGuard guard(h->dev);
  STATUS_TRY(sync_handle(h));
  for (int i = 0; i < 2; ++i) {
    cudaFree(h->perm_dev[i]);
    h->perm_dev[i] = nullptr;
    h->perm_epoch[i] = -1;
    CUDA_TRY(cudaMalloc(&h->perm_dev[i], sizeof(int32_t) * (size_t)n_samples));
  }
  if (h->perm_next.valid()) h->perm_next.wait();
  h->perm_next_epoch = -1;
  for (int i = 0; i < 2; ++i) {
    if (h->perm_host[i]) cudaFreeHost(h->perm_host[i]);
    h->perm_host[i] = nullptr;
    CUDA_TRY(cudaMallocHost(&h->perm_host[i], sizeof(int32_t) * (size_t)n_samples));
    if (!h->perm_ev[i]) CUDA_TRY(cudaEventCreateWithFlags(&h->perm_ev[i], cudaEventDisableTiming));
    h->perm_ev_used[i] = false;
  }
  STATUS_TRY(ensure_G(h));
  {  // learner scratch, sized for SMA_MAX_LOCAL_REPLICAS learners (resize-safe)
    cudaFree(h->mlp_A1);
    cudaFree(h->mlp_DA);
    h->mlp_A1 = nullptr;
    h->mlp_DA = nullptr;
    const size_t n = (size_t)SMA_MAX_LOCAL_REPLICAS * batch * (kind == 1 ? hidden : classes);
    if (kind == 1) {
      CUDA_TRY(cudaMalloc(&h->mlp_A1, sizeof(float2) * n));
      cudaFree(h->mlp_E);
      h->mlp_E = nullptr;
      CUDA_TRY(cudaMalloc(&h->mlp_E, sizeof(float) * (size_t)SMA_MAX_LOCAL_REPLICAS * batch * classes));
      if (!h->mlp_PL)  // two round-parity sets of partial logits (one [16][32] tile per CTA),
                       // then two of b2 per learner ([32] each; r <= grid <= #SMs)
        CUDA_TRY(cudaMalloc(&h->mlp_PL, sizeof(float) * 2 * (size_t)h->num_sms * (16 * 32 + 32)));
      if (!h->mlp_bar) {  // three kinds of 128-byte flag lines, one per CTA (grid <= #SMs)
        const size_t nb = sizeof(unsigned) * 32 * 3 * (size_t)h->num_sms;
        CUDA_TRY(cudaMalloc(&h->mlp_bar, nb));
        CUDA_TRY(cudaMemset(h->mlp_bar, 0, nb));
      }
    }
    CUDA_TRY(cudaMalloc(&h->mlp_DA, sizeof(float) * n));
  }
  h->learner = true;
  h->kind = kind;
  h->hidden = hidden;
  h->in_dim = in_dim;
  h->classes = classes;
  h->batch = batch;
  h->X = X_dev;
  h->y = y_dev;
  h->n_samples = n_samples;
  h->batch_seed = batch_seed;
  return SMA_OK;
}

// The batch permutation of `round`'s epoch on the device (R10): built on the
// host and uploaded when the epoch changes, double-buffered by epoch parity on
// both sides, with no host synchronisation of the stream: the upload is
// stream-ordered after every earlier round of the handle (so after the last
// kernel that read this device buffer, two epochs ago), and the host only waits
// for the previous upload out of the same pinned buffer.
static sma_status learner_batch(sma_handle* h, int64_t round, cudaStream_t s, int* buf_out,
                         int64_t* pos0_out) {
  const int64_t E = h->n_samples / ((int64_t)h->cfg.k * h->batch);
  if (E < 1)  // as sma_plan_batch_indices: k learners need k * batch samples per round
    return fail(SMA_ERR_INVALID_ARG, "n_samples=%lld < k*batch=%lld: no full round per epoch",
                (long long)h->n_samples, (long long)h->cfg.k * h->batch);
  const int64_t e = round / E;
  const int buf = (int)(e & 1);
  if (h->perm_epoch[buf] != e) {
    if (h->perm_next.valid()) h->perm_next.wait();   // a prefetch may target this buffer
    if (h->perm_next_epoch != e) {                   // not prefetched: build it now
      if (h->perm_ev_used[buf]) CUDA_TRY(cudaEventSynchronize(h->perm_ev[buf]));
      plan_epoch_permutation(h->n_samples, h->batch_seed, e, h->perm_host[buf]);
    }
    if (h->any_work) CUDA_TRY(cudaStreamWaitEvent(s, h->evDone, 0));
    CUDA_TRY(cudaMemcpyAsync(h->perm_dev[buf], h->perm_host[buf], sizeof(int32_t) * h->n_samples,
                             cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaEventRecord(h->perm_ev[buf], s));
    h->perm_ev_used[buf] = true;
    h->perm_epoch[buf] = e;
    // prefetch epoch e + 1 on a host worker: it first waits for the upload of
    // epoch e - 1 out of the same pinned buffer, then overwrites it
    const int nb = buf ^ 1;
    int32_t* dst = h->perm_host[nb];
    cudaEvent_t prev = h->perm_ev_used[nb] ? h->perm_ev[nb] : nullptr;
    const int64_t N = h->n_samples;
    const uint64_t seed = h->batch_seed;
    h->perm_next_epoch = e + 1;
    h->perm_next = std::async(std::launch::async, [=] {
      if (prev) cudaEventSynchronize(prev);
      plan_epoch_permutation(N, seed, e + 1, dst);
    });
  }
  *buf_out = buf;
  *pos0_out = (round % E) * h->cfg.k * (int64_t)h->batch;
  return SMA_OK;
}

sma_status sma_learner_grads(sma_handle* h, int64_t round, void* stream) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  NvtxRange nvtx("sma_learner_grads");
  if (!h->learner) return fail(SMA_ERR_STATE, "no learner attached");
  if (round < 0) return fail(SMA_ERR_INVALID_ARG, "round < 0");
  if (h->r == 0) return SMA_OK;
  DeviceGuard guard(h->dev);
  cudaStream_t s = (cudaStream_t)stream;
  int buf = 0;
  int64_t pos0 = 0;
  STATUS_TRY(learner_batch(h, round, s, &buf, &pos0));
  if (h->kind == 0) {
    CUDA_TRY(launch_softmax_grad(h->X, h->y, h->perm_dev[buf], pos0, h->batch, h->in_dim,
                                 h->classes, h->W, h->d_pad, h->r, h->j0, h->mlp_DA, h->G, s));
    h->launches += 2;
  } else {
    ReplicaArgs a{};
    a.W = h->W;
    a.ld = h->d_pad;
    a.r = h->r;
    cudaError_t e = launch_mlp_round(h->X, h->y, h->perm_dev[buf], pos0, (int64_t)h->cfg.k * h->batch,
                                     1, h->batch, h->in_dim, h->hidden, h->classes, h->j0, h->mlp_PL,
                                     h->mlp_bar, h->mlp_epoch + 1, h->G, a, false, h->num_sms, s);
    if (e != cudaErrorNotSupported) ++h->mlp_epoch;
    if (e == cudaErrorNotSupported) {  // the five-kernel path
      CUDA_TRY(launch_mlp_grad(h->X, h->y, h->perm_dev[buf], pos0, h->batch, h->in_dim, h->hidden,
                               h->classes, h->W, h->d_pad, h->r, h->j0, h->mlp_A1, h->mlp_E,
                               h->mlp_DA, h->G, s));
      h->launches += 4;
    } else {
      CUDA_TRY(e);
      h->launches += 1;
    }
  }
  for (int i = 0; i < h->r; ++i) set_gptr(h, i, h->G + (int64_t)i * h->d_pad);
  leave_staged_set(h);
  return mark_done(h, s);
}

// The n = 1 learner round in one fused kernel applies: the MLP kernel
// (sma_learner_mlp_fused.cu) or the softmax cluster kernel
// (sma_learner_softmax_fused.cu).
static bool learner_fused_ok(const sma_handle* h) {
  return !h->collective && !h->matc && h->r > 0 && !(h->graphs && !h->timing) &&
         ((h->kind == 1 && mlp_fused_enabled()) || (h->kind == 0 && softmax_cluster_enabled()));
}

// Rounds [round0, round0 + count) of ONE epoch, with the learner in the loop,
// in one launch of the fused learner kernel (MLP, or the softmax cluster).
// *unsupported (nothing enqueued) when
// the kernel does not cover the shape or count.
static sma_status fused_learner_rounds(sma_handle* h, int64_t round0, int count, cudaStream_t s,
                                   bool* unsupported) {
  *unsupported = false;
  DeviceGuard guard(h->dev);
  int buf = 0;
  int64_t pos0 = 0;
  STATUS_TRY(learner_batch(h, round0, s, &buf, &pos0));
  ReplicaArgs a{};
  a.W = h->W;
  a.ld = h->d_pad;
  a.r = h->r;
  a.d = h->cfg.d;
  a.n4 = h->n4;
  a.z = h->z();
  a.zprev_next = h->zprev();
  a.alpha = h->alpha;
  a.gamma = h->gamma;
  a.mu = h->mu;
  a.nonfinite = h->check ? h->nonfinite : nullptr;
  STATUS_TRY(pre_round(h, s, true));
  if (count > 1 && h->zread_pending[h->cur]) {  // round 2 of the launch rewrites z[cur] too
    CUDA_TRY(cudaStreamWaitEvent(s, h->evZread[h->cur], 0));
    h->zread_pending[h->cur] = false;
  }
  cudaEvent_t* tp = nullptr;
  STATUS_TRY(timer_pair(h, SMA_PHASE_REPLICA, &tp));
  if (tp) CUDA_TRY(cudaEventRecord(tp[0], s));
  const cudaError_t e =
      h->kind == 0
          ? launch_softmax_cluster_rounds(h->X, h->y, h->perm_dev[buf], pos0,
                                          (int64_t)h->cfg.k * h->batch, count, h->batch, h->in_dim,
                                          h->classes, h->j0, h->G, a, s)
          : launch_mlp_round(h->X, h->y, h->perm_dev[buf], pos0, (int64_t)h->cfg.k * h->batch, count,
                             h->batch, h->in_dim, h->hidden, h->classes, h->j0, h->mlp_PL, h->mlp_bar,
                             h->mlp_epoch + 1, h->G, a, true, h->num_sms, s);
  if (e == cudaErrorNotSupported) {
    if (tp) h->tused[SMA_PHASE_REPLICA] -= 2;  // nothing launched: drop the event pair
    *unsupported = true;
    return SMA_OK;
  }
  CUDA_TRY(e);
  if (tp) CUDA_TRY(cudaEventRecord(tp[1], s));
  h->mlp_epoch += (unsigned)count;
  h->launches += 1;
  for (int i = 0; i < h->r; ++i) set_gptr(h, i, h->G + (int64_t)i * h->d_pad);
  leave_staged_set(h);
  for (int i = 0; i < count; ++i) advance(h);
  return mark_done(h, s);
}

sma_status sma_learner_steps(sma_handle* h, int64_t round0, int32_t count, void* stream) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  NvtxRange nvtx("sma_learner_steps");
  if (!h->learner) return fail(SMA_ERR_STATE, "no learner attached");
  if (round0 < 0 || count < 0) return fail(SMA_ERR_INVALID_ARG, "round0 < 0 or count < 0");
  int64_t i = round0;
  const int64_t end = round0 + count;
  const char* fe = getenv("SMA_LEARNER_FUSE");
  if (!(fe && fe[0] == '1') && learner_fused_ok(h)) {
    const int64_t E = h->n_samples / ((int64_t)h->cfg.k * h->batch);
    if (E < 1)
      return fail(SMA_ERR_INVALID_ARG, "n_samples=%lld < k*batch: no full round per epoch",
                  (long long)h->n_samples);
    while (i < end) {  // one launch per epoch segment (one permutation per launch)
      const int64_t n = std::min<int64_t>(end - i, E - i % E);
      bool unsupported = false;
      STATUS_TRY(fused_learner_rounds(h, i, (int)n, (cudaStream_t)stream, &unsupported));
      if (unsupported) break;
      i += n;
    }
  }
  for (; i < end; ++i) STATUS_TRY(sma_learner_step(h, i, stream));  // one round at a time
  return SMA_OK;
}

sma_status sma_learner_step(sma_handle* h, int64_t round, void* stream) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  NvtxRange nvtx("sma_learner_step");
  if (!h->learner) return fail(SMA_ERR_STATE, "no learner attached");
  if (round < 0) return fail(SMA_ERR_INVALID_ARG, "round < 0");
  const size_t fused_smem =
      (sizeof(float) * (32 + (size_t)h->classes) + sizeof(int)) * (size_t)h->r * h->batch;
  // The learner-fused softmax round (one kernel after the logits) is opt-in,
  // SMA_LEARNER_FUSE=1 (read per call): on B200 the unfused sequence (logits,
  // feature-sliced dW, the small-round replica kernel) measured faster, 58.8k vs
  // 54.1k C1 rounds/s -- the fused kernel's 26 CTAs serialise its update work.
  const char* fe = getenv("SMA_LEARNER_FUSE");
  const bool fuse_knob = fe && fe[0] == '1';
  const bool fusable = fuse_knob && h->kind == 0 && !h->collective && !h->matc && h->r > 0 &&
                       h->classes <= 16 && fused_smem <= 200 * 1024 && !(h->graphs && !h->timing);
  if (!fusable && h->collective && h->overlap && !(h->graphs && !h->timing)) {
    // Mode B: the z-sync of this round is forked first and overlaps the
    // learner kernels and the replica kernel
    NvtxRange nvtx2("sma_learner_step.overlap");
    if (h->p2p && !h->p2p_connected)
      return fail(SMA_ERR_STATE, "SMA_FLAG_P2P_ZSYNC: call sma_p2p_connect on every rank first");
    DeviceGuard guard(h->dev);
    cudaStream_t s = (cudaStream_t)stream;
    leave_staged_set(h);  // the learner writes the handle's own gradient buffers
    STATUS_TRY(pre_round(h, s, true));
    if (h->q_dirty) STATUS_TRY(enqueue_q_prologue(h, s));
    const LearnerFn fn = [&](cudaStream_t ls) { return sma_learner_grads(h, round, ls); };
    STATUS_TRY(enqueue_round(h, s, &fn));
    advance(h);
    return mark_done(h, s);
  }
  if (!fusable && learner_fused_ok(h)) {
    // n = 1 learner round: gradient of every local learner and the fused update
    // of the replicas and z in ONE kernel (sma_learner_mlp_fused.cu, or
    // sma_learner_softmax_fused.cu's cluster for the softmax learner)
    bool unsupported = false;
    STATUS_TRY(fused_learner_rounds(h, round, 1, (cudaStream_t)stream, &unsupported));
    if (!unsupported) return SMA_OK;
  }
  if (!fusable) {  // the same result through the two public calls
    STATUS_TRY(sma_learner_grads(h, round, stream));
    return sma_step(h, stream);
  }
  DeviceGuard guard(h->dev);
  cudaStream_t s = (cudaStream_t)stream;
  leave_staged_set(h);
  STATUS_TRY(pre_round(h, s, true));
  int buf = 0;
  int64_t pos0 = 0;
  STATUS_TRY(learner_batch(h, round, s, &buf, &pos0));
  ReplicaArgs a{};
  a.W = h->W;
  a.ld = h->d_pad;
  a.r = h->r;
  a.d = h->cfg.d;
  a.n4 = h->n4;
  a.z = h->z();
  a.zprev_next = h->zprev();
  a.alpha = h->alpha;
  a.gamma = h->gamma;
  a.mu = h->mu;
  a.nonfinite = h->check ? h->nonfinite : nullptr;
  cudaEvent_t* tp = nullptr;
  STATUS_TRY(timer_pair(h, SMA_PHASE_REPLICA, &tp));
  if (tp) CUDA_TRY(cudaEventRecord(tp[0], s));
  CUDA_TRY(launch_softmax_round(h->X, h->y, h->perm_dev[buf], pos0, h->batch, h->in_dim,
                                h->classes, h->j0, h->mlp_DA, h->G, a, s));
  if (tp) CUDA_TRY(cudaEventRecord(tp[1], s));
  h->launches += 2;
  for (int i = 0; i < h->r; ++i) set_gptr(h, i, h->G + (int64_t)i * h->d_pad);
  advance(h);
  return mark_done(h, s);
}

sma_status sma_p2p_handle(sma_handle* h, void* out) {
  if (!h || !out) return fail(SMA_ERR_INVALID_ARG, "NULL argument");
  if (!h->p2p) return fail(SMA_ERR_STATE, "not an SMA_FLAG_P2P_ZSYNC handle");
  DeviceGuard guard(h->dev);
  cudaIpcMemHandle_t ipc;
  CUDA_TRY(cudaIpcGetMemHandle(&ipc, h->p2p_region));
  static_assert(sizeof(ipc) == SMA_P2P_HANDLE_BYTES, "IPC handle size");
  memcpy(out, &ipc, sizeof ipc);
  return SMA_OK;
}

sma_status sma_p2p_connect(sma_handle* h, const void* handles) {
  if (!h || !handles) return fail(SMA_ERR_INVALID_ARG, "NULL argument");
  if (!h->p2p) return fail(SMA_ERR_STATE, "not an SMA_FLAG_P2P_ZSYNC handle");
  if (h->p2p_connected) return fail(SMA_ERR_STATE, "already connected");
  DeviceGuard guard(h->dev);
  const char* all = static_cast<const char*>(handles);
  for (int g = 0; g < h->cfg.world; ++g) {
    if (g == h->cfg.rank) continue;
    cudaIpcMemHandle_t ipc;
    memcpy(&ipc, all + (size_t)g * SMA_P2P_HANDLE_BYTES, sizeof ipc);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int q = 0; q < g; ++q)
        if (q != h->cfg.rank && h->p2p_base[q]) {
          cudaIpcCloseMemHandle(h->p2p_base[q]);
          h->p2p_base[q] = nullptr;
        }
      return fail(SMA_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d) failed: %s", g, cudaGetErrorString(e));
    }
    h->p2p_base[g] = static_cast<char*>(p);
  }
  h->p2p_connected = true;
  return SMA_OK;
}

sma_status sma_set_timing(sma_handle* h, int on) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  h->timing = on != 0;
  return SMA_OK;
}

sma_status sma_kernel_time(sma_handle* h, int32_t phase, double* total_ms, int64_t* launches,
                           int reset) {
  if (!h || !total_ms || !launches) return fail(SMA_ERR_INVALID_ARG, "NULL argument");
  if (phase < 0 || phase >= SMA_NUM_PHASES) return fail(SMA_ERR_INVALID_ARG, "bad phase %d", phase);
  DeviceGuard guard(h->dev);
  STATUS_TRY(sync_handle(h));
  double tot = 0;
  const auto& v = h->tev[phase];
  for (size_t i = 0; i + 1 < h->tused[phase]; i += 2) {
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, v[i], v[i + 1]));
    tot += ms;
  }
  *total_ms = tot;
  *launches = (int64_t)(h->tused[phase] / 2);
  if (reset) h->tused[phase] = 0;
  return SMA_OK;
}

int64_t sma_launch_count(const sma_handle* h) { return h ? h->launches : -1; }

sma_status sma_info(const sma_handle* h, int64_t* d_pad, int32_t* local_first, int32_t* local_count,
                    int64_t* shard_offset, int64_t* shard_length) {
  if (!h) return fail(SMA_ERR_INVALID_ARG, "NULL handle");
  if (d_pad) *d_pad = h->d_pad;
  if (local_first) *local_first = h->j0;
  if (local_count) *local_count = h->r;
  if (shard_offset) *shard_offset = h->shard_off;
  if (shard_length) *shard_length = h->shard_len;
  return SMA_OK;
}

}  // extern "C"
