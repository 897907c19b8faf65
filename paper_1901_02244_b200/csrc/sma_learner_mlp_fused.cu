// sma_learner_mlp_fused.cu -- the MLP learner's gradient (a2', Eq. 2 P:228-232,
// back-propagation) for all r local learners AND, for the n = 1 round,
// the SMA update of every replica and of z (a3-a7, Alg. 1 lines 9-13), in ONE
// kernel -- optionally for several consecutive rounds per launch
// (sma_learner_steps).
//
// Why: at the paper's small batches (b = 16) the learner is a chain of short
// dependent phases (layer 1 -> logits -> softmax -> head -> dW1 -> update).  As
// five kernels each boundary costs a drain + launch (PDL hides only part of it)
// and every phase re-stages its operands: 24 us per k = 4 round in round 1
// (DESIGN §13).  Here one CTA owns (learner j, a block of U hidden units): it
// keeps the batch rows, the block's W1 rows / W2 columns / b1 (its own learner's
// parameters -- it is their only writer, so across the rounds of one launch
// they stay in shared memory) and the z rows it needs, all staged by TMA bulk
// copies, and exchanges only the (b x classes) partial logits through L2.
// There is no grid-wide barrier: CTAs order themselves with per-CTA flag lines
// (partial logits written; z slice written; replicas stored), each waited on
// exactly where the data is consumed.  The round's z^{i+1} is computed from the
// PRE-update replicas by every CTA on a 1/grid slice of the vector (it needs no
// gradient), and each CTA updates its replica block where it computed the
// block's gradient.  See mlp_round_kernel below for the phase order.
//
// All CTAs must be co-resident (grid <= #SMs with one CTA per SM, checked by
// the launcher).  Summation orders are fixed, so results are deterministic;
// they differ from the five-kernel path only in fp32 rounding (different K
// order of the layer-1 dot and of the logits).  Shapes outside this kernel
// (b > 16, in_dim % 4, hidden not a multiple of U, too many CTAs, shared
// memory) return cudaErrorNotSupported and the caller uses the five-kernel path
// (one round at a time).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "sma_bulk.cuh"
#include "sma_dot2.cuh"
#include "sma_pdl.cuh"
#include "sma_softmax.cuh"
#include "sma_internal.h"

namespace sma {
namespace {
constexpr int kThr = 256;
constexpr int kWarps = kThr / 32;
// Phase 1 splits K into kSlices slices (partials summed in slice order): 12 is
// a multiple of the group-1 sizes 4 and 6, so the slices spread evenly, and a1's
// rounding does not depend on how many warps run phase 1.
constexpr int kSlices = 12;
constexpr int kRows = 16;        // batch rows per learner (b <= 16, zero-padded)
constexpr int kTR = 2;           // rows per lane in phase 1 (8 row groups)
constexpr int kUG = 4;           // unit groups per warp in phase 1

using dot2::f2;

// L2 only: data written by other CTAs of this kernel (the partial logits)
__device__ __forceinline__ float ld_cg(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Cross-CTA ordering without a shared counter or a full grid barrier (128
// atomics on one address serialise in the L2's atomic unit, ~27 cycles each,
// B300_MICROARCH "L2-atom multi-CTA"; a counter barrier measured ~2.5 us from
// the last arrival to the release).  Each CTA publishes the round's epoch
// (a host-side round counter, so flags only ever grow) in its own 128-byte
// line with a release store -- cumulative over the CTA's writes through the
// bar.sync before it -- and a consumer acquires exactly the lines it depends
// on, one thread per line, then bar.syncs.  Three split-phase points per round:
//   PL: the partial logits of CTA c are written (consumers: the CTAs of the
//       same learner, right after their own partials);
//   ZD: CTA c's slice of z^{i+1} is written, i.e. it has finished reading the
//       PRE-update replicas (consumers: every CTA, before its first replica
//       store -- long satisfied by then -- and before it stages z^{i+1});
//   P2: CTA c has stored its replica block of W^{i+1} (consumers: every CTA,
//       before its z slice of round i + 1, which reads every replica).
// `releaser`: the thread that issues the release store (it waits there for the
// CTA's outstanding stores), chosen off the next phase's critical path.
__device__ __forceinline__ void flag_arrive(unsigned* line, unsigned epoch, int releaser = 0) {
  __syncthreads();
  if ((int)threadIdx.x == releaser) st_release_gpu(line, epoch);
}
// Spin until *line >= epoch (acquire).
__device__ __forceinline__ void flag_poll(const unsigned* line, unsigned epoch) {
  const long long t0 = clock64();
  while ((int)(ld_acquire_gpu(line) - epoch) < 0)
    if (clock64() - t0 > 60000000000ll) __trap();  // ~30 s: a CTA never arrived
}
// Split cluster barrier (every thread of the cluster arrives, then waits):
// release / acquire at cluster scope, covering shared::cluster and global memory.
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Named barrier over the first / second warp group of the CTA.
__device__ __forceinline__ void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
struct MlpRoundArgs {
  const float* X;
  const int32_t* y;
  const int32_t* perm;    // this launch's epoch permutation
  int64_t pos0;           // perm position of learner 0, row 0 of the first round
  int64_t kb;             // perm positions per round (k * b)
  int count;              // rounds in this launch (UPDATE; 1 otherwise)
  int b, in_dim, hidden, classes, j0;
  int U, nblk;            // hidden units per CTA, CTAs per learner
  int nch;                // phase-1 chunks of CU = TU * kUG units (U / CU); > 1 only if count == 1
  int nx;                 // batch-row buffers: 2 = the next round's rows prefetched
  int nzb;                // z-row buffers of the W1 block: 0 (z read from L2), 1, or 2 (prefetched)
  int nzw;                // UPDATE: warps of group 2 (0 = it runs on all warps, after phase 1)
  int bexp;               // certainty threshold 2^bexp (R18; >= 6x the dot's error bound)
  float bscale;           // 2^bexp
  int cl;                 // UPDATE, cluster mode: the r CTAs of one unit block form a thread-block
                          // cluster (blockIdx.x = blk * r + j) and exchange z through it
  float* PL;              // [2][grid][kRows][classes] partial logits (round parity)
  float* B2;              // [2][r][32] b2^{i+1} of each learner, written by its block 0 (parity)
  float* G;               // gradients [r][ld]
  unsigned* bar;          // flag lines: kind q of CTA c at bar + 32 (q fstride + c)
  int fstride;            // flag lines per kind (>= grid)
  unsigned epoch;         // first round's number (host counter, increasing)
  unsigned long long* prof;  // SMA_MLP_PROF: per-phase cycle sums [grid][16] (or nullptr)
  int p2rel;              // P2 flag released by group 2 (SMA_MLP_P2REL, default 1)
  ReplicaArgs a;          // W, ld, r, z, zprev_next, alpha, gamma, mu, d, n4, nonfinite
};
enum { kFlagPL = 0, kFlagZD = 1, kFlagP2 = 2 };

// SMA_MLP_PROF: thread 0 (phase 1, phase 2) and the first z-slice thread
// accumulate clock64() cycles per phase boundary over every round of the
// launch; written to prof[CTA][16] at the end (see the launcher's report).
// sma_elem / central_elem of sma_kernels.cu.
__device__ __forceinline__ float elem_w(float w, float g, float z, float alpha, float gamma,
                                       float& c) {
  c = __fmul_rn(alpha, __fsub_rn(w, z));
  return __fsub_rn(__fmaf_rn(-gamma, g, w), c);
}
__device__ __forceinline__ float4 elem_w4(float4 w, float4 g, float4 z, float alpha, float gamma) {
  float c;
  w.x = elem_w(w.x, g.x, z.x, alpha, gamma, c);
  w.y = elem_w(w.y, g.y, z.y, alpha, gamma, c);
  w.z = elem_w(w.z, g.z, z.z, alpha, gamma, c);
  w.w = elem_w(w.w, g.w, z.w, alpha, gamma, c);
  return w;
}
__device__ __forceinline__ bool finite4(float4 v) {
  return isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
}
// L2 loads of data other CTAs of this kernel rewrite every round (both z
// halves, the replicas): never the read-only path, never a possibly stale L1 line.
__device__ __forceinline__ float4 ld_z4(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
// Generic-proxy writes of other CTAs (acquired through a flag) -> this
// thread's TMA reads of the same global memory.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// One CTA = (learner j, a block of U hidden units); `count` SMA rounds per
// launch.  Per round i (state W^i, z^i, z^{i-1}):
//   phase 1  a1 = W1 x + b1 for the block from shared memory (the block's W1
//            rows, W2 columns and b1 are staged by TMA once per launch and then
//            kept there: this CTA is their only writer), K split over the 8
//            warps with a fixed-order cross-warp sum; R18's certainty test +
//            Dot2 for the uncertain; h = relu(a1); partial logits -> L2, PL flag.
//   z slice  (UPDATE) after every CTA has stored W^i (P2 flags of round i-1):
//            z^{i+1} = (z^i + sum_j alpha (w_j^i - z^i)) + mu (z^i - z^{i-1}) on
//            this CTA's 1/grid of the vector (corrections in ascending j), into
//            the z^{i-1} half; ZD flag.
//   phase 2  after the PL flags of learner j: its partial logits (one TMA bulk
//            copy) summed in ascending block order, softmax - onehot (one warp
//            per row), da1 = (W2^T e)[a1 > 0], dW2 / db2 / db1 / dW1 -> G and,
//            UPDATE, after every ZD flag (nobody still reads W^i), the block's
//            w' = fma(-gamma, g, w) - alpha (w - z^i) -> global and shared
//            memory; P2 flag.  The z^{i+1} rows of the block for round i + 1 are
//            prefetched by TMA as soon as the ZD flags are in, and the next
//            round's batch rows at the start of the round.
// Every parameter of learner j belongs to exactly one unit block (W1 rows,
// b1, W2 columns; b2 to block 0), so the updates touch disjoint data.
// The arithmetic per element is replica_step_ldg<kFused>'s, so a round is
// bitwise the same as gradients-then-update with these gradients.
// FB, FC: the batch size and the class count as compile-time constants (16 and
// 10, the bench's shape: the per-row and per-class loops unroll fully) or 0
// (read from the arguments).
template <int TU, bool UPDATE, bool PROF, int FB, int FC, int FI = 0>
__global__ void __launch_bounds__(kThr, 2) mlp_round_kernel(const MlpRoundArgs m) {
  constexpr int CU = TU * kUG;  // units per phase-1 chunk (<= 32)
  extern __shared__ __align__(16) float sm[];
  const int in_dim = FI ? FI : m.in_dim, hidden = m.hidden, classes = FC ? FC : m.classes, b = FB ? FB : m.b,
            U = m.U;
  const int nch = m.nch, nblk = m.nblk;
  // rows padded to xld = in_dim + 4 floats: consecutive rows then start 20
  // banks apart (784 + 4 = 788 = 20 mod 32), so the 8 batch-row groups and the
  // 4 unit groups of a warp's 128-bit loads hit distinct banks (784 = 16 mod
  // 32 put rows t and t + 2 on the same banks)
  const int xld = in_dim + 4;
  const int npl = kRows * classes;                       // partial logits per CTA
  float* xs = sm;                                        // [nx][kRows][xld]
  float* w1s = xs + m.nx * kRows * xld;                  // [CU][xld] W1 rows (a chunk)
  float* zs = w1s + CU * xld;                            // [nzb][U][xld] z rows
  float* part = zs + m.nzb * U * xld;                    // [kSlices][kRows][CU]
  float* hs = part + kSlices * kRows * CU;               // [kRows][U] relu(a1)
  float* das = hs + kRows * U;                           // [kRows][U] da1
  float* lg = das + kRows * U;                           // [kRows][32] logits
  float* es = lg + kRows * 32;                           // [kRows][32] softmax - onehot
  float* xnb = es + kRows * 32;                          // [2][kRows] ||x_t|| (round parity)
  float* wn = xnb + 2 * kRows;                           // [CU] ||W1[u]||
  float* w2s = wn + CU;                                  // [32][U] W2 columns of the block
  float* b1s = w2s + 32 * U;                             // [U] b1 of the block
  float* zw2s = b1s + U;                                 // [2][32][U] z of the W2 columns
  float* zb1s = zw2s + 2 * 32 * U;                       // [2][U] z of b1
  float* plg = zb1s + 2 * U;                             // [nblk][npl] learner j's partial logits
  unsigned char* msk = reinterpret_cast<unsigned char*>(plg + nblk * npl);  // [kRows][U]
  __shared__ int rows[2][kRows], ys[2][kRows];
  __shared__ int n_unc;
  __shared__ short unc[kRows * 32];
  __shared__ float b2s[32];  // b2^i of learner j (read before any CTA may write b2^{i+1})
  __shared__ float zb2s[32];  // z^i of b2 (block 0's update)
  // [0], [1] batch-row buffers; [2] weight block; [3], [4] z block buffers; [5] partial logits
  __shared__ __align__(8) uint64_t mbar[6];

  // cluster mode: the r CTAs of unit block blk are one cluster (rank j)
  const int j = m.cl ? (int)(blockIdx.x % (unsigned)m.a.r) : (int)(blockIdx.x / nblk);
  const int blk = m.cl ? (int)(blockIdx.x / (unsigned)m.a.r) : (int)(blockIdx.x - j * nblk);
  const int cid = j * nblk + blk;  // learner-major CTA index (partial logits, their flags)
  const int u0 = blk * U;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const ReplicaArgs& a = m.a;
  const int64_t ob1 = (int64_t)hidden * in_dim, oW2 = ob1 + hidden, ob2 = oW2 + (int64_t)classes * hidden;
  float* W = a.W + (int64_t)j * a.ld;
  float* G = m.G + (int64_t)j * a.ld;
  const uint32_t rowb = 4u * (uint32_t)in_dim;
  unsigned* const fPL = m.bar + 32 * (kFlagPL * m.fstride);
  unsigned* const fZD = m.bar + 32 * (kFlagZD * m.fstride);
  unsigned* const fP2 = m.bar + 32 * (kFlagP2 * m.fstride);

  // rows / labels of round i's batch for this learner (threads < kRows)
  auto load_rows = [&](int i) {
    if (tid < kRows) {
      const int r = tid < b ? m.perm[m.pos0 + (int64_t)i * m.kb + (int64_t)(m.j0 + j) * b + tid] : 0;
      rows[i & 1][tid] = r;
      ys[i & 1][tid] = tid < b ? m.y[r] : 0;
    }
  };
  // one TMA bulk copy per batch row into buffer xb (warp 0; rows[i & 1] visible)
  auto issue_rows = [&](int i, int xb) {
    if (warp == 0) {
      if (lane == 0) bulk::expect_tx(&mbar[xb], rowb * (uint32_t)b);
      __syncwarp();
      if (lane < b) bulk::copy(xs + (xb * kRows + lane) * xld, m.X + (int64_t)rows[i & 1][lane] * in_dim, rowb, &mbar[xb]);
    }
  };
  // ||x_t|| of the rows at xr into out[kRows]: one warp per row (fixed order),
  // by the calling warps lw = 0 .. nwarps - 1
  auto x_norms = [&](const float* xr, float* out, int lw, int nwarps) {
    for (int t = lw; t < kRows; t += nwarps) {
      const float4* x4 = reinterpret_cast<const float4*>(xr + t * xld);
      float s = 0.f;
      for (int f = lane; f < (in_dim >> 2); f += 32) {
        const float4 v = x4[f];
        s = __fmaf_rn(v.x, v.x, s); s = __fmaf_rn(v.y, v.y, s);
        s = __fmaf_rn(v.z, v.z, s); s = __fmaf_rn(v.w, v.w, s);
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
      if (lane == 0) out[t] = sqrtf(s);
    }
  };
  // z^{i} of the block's W2 columns and b1 (+ W1 rows if staged) into buffer zb,
  // issued by the calling warp
  auto issue_z_warp = [&](const float* zsrc, int zb) {
    {
      if (lane == 0)
        bulk::expect_tx(&mbar[3 + zb], 4u * (uint32_t)(classes * U + U) + (m.nzb ? rowb * (uint32_t)U : 0u));
      __syncwarp();
      for (int c = lane; c < classes; c += 32)
        bulk::copy(zw2s + (zb * 32 + c) * U, zsrc + oW2 + (int64_t)c * hidden + u0, 4u * U, &mbar[3 + zb]);
      if (lane == 0) bulk::copy(zb1s + zb * U, zsrc + ob1 + u0, 4u * U, &mbar[3 + zb]);
      if (m.nzb)
        for (int t = lane; t < U; t += 32)
          bulk::copy(zs + ((m.nzb == 2 ? zb : 0) * U + t) * xld, zsrc + (int64_t)(u0 + t) * in_dim, rowb, &mbar[3 + zb]);
    }
  };

  // ---- prologue (X, perm, y are never written by a kernel: before the PDL wait)
  load_rows(0);
  if (tid == 0) {
    n_unc = 0;
    for (int q = 0; q < 6; ++q) bulk::bar_init(&mbar[q]);
  }
  __syncthreads();
  issue_rows(0, 0);
  for (int q = b * xld + tid; q < kRows * xld; q += kThr) {  // zero-padded batch rows (never copied)
    xs[q] = 0.f;
    if (m.nx == 2) xs[kRows * xld + q] = 0.f;
  }
  bulk::wait(&mbar[0], 0);
  __syncthreads();
  x_norms(xs, xnb, warp, kWarps);
  pdl::wait_and_release();  // the replicas and z were written by the previous launch
  // b2 of round 0 (later rounds: from block 0's copy in m.B2, see phase 2)
  if (tid < classes) b2s[tid] = ld_cg(W + ob2 + tid);

  // ---- the block's weights (kept for the whole launch) and round 0's z, by TMA
  if (warp == 0) {
    if (lane == 0) bulk::expect_tx(&mbar[2], rowb * CU + 4u * (uint32_t)(classes * U + U));
    __syncwarp();
    for (int t = lane; t < CU; t += 32) bulk::copy(w1s + t * xld, W + (int64_t)(u0 + t) * in_dim, rowb, &mbar[2]);
    for (int c = lane; c < classes; c += 32)
      bulk::copy(w2s + c * U, W + oW2 + (int64_t)c * hidden + u0, 4u * U, &mbar[2]);
    if (lane == 0) bulk::copy(b1s, W + ob1 + u0, 4u * U, &mbar[2]);
  }
  if (UPDATE && warp == 0) {
    issue_z_warp(a.z, 0);
    if (m.cl) issue_z_warp(a.zprev_next, 1);  // cluster mode: z^{-1} too (then z moves through DSMEM)
  }

  bool bad = false;
  const float fb = (float)b;
  const bool pow2 = (b & (b - 1)) == 0;
  const float inv_b = 1.f / fb;
  // UPDATE: warps [0, nw1) ("group 1") run phase 1 and the logits / softmax /
  // da1 chain of phase 2; the other nzw warps ("group 2") run, beside them,
  // everything that does not need the gradient: the next round's batch rows
  // (TMA + norms), the z slice, and the z^{i+1} block prefetch.  Each group
  // synchronises on its own named barrier; they join before the replica update.
  const int nzw = UPDATE ? m.nzw : 0;  // group-2 warps (0: none, group 2's work runs on all)
  const int nw1 = kWarps - nzw;
  const int nt1 = 32 * nw1;
  __shared__ unsigned long long pacc[16];  // (shared: no register pressure on the PROF build)
  if (PROF && tid < 16) pacc[tid] = 0;
  __syncthreads();
  long long tprev = PROF ? clock64() : 0;
  auto pmark = [&](int q) {  // SMA_MLP_PROF cycle accumulators (threads 0 and nt1)
    if (PROF && (tid == 0 || tid == nt1)) {
      const long long t = clock64();
      if ((tid == 0) == (q < 12)) pacc[q] += (unsigned long long)(t - tprev);
      tprev = t;
    }
  };
  for (int i = 0; i < m.count; ++i) {
    pmark(0);
    // G (the gradients the handle registers afterwards) is only observable
    // after the launch: write the last round's
    const bool wg = !UPDATE || i + 1 == m.count;
    const unsigned ep = m.epoch + (unsigned)i;
    const int xb = m.nx == 2 ? (i & 1) : 0;
    const float* xr = xs + xb * kRows * xld;
    const float* xnr = xnb + (i & 1) * kRows;                          // ||x_t|| of round i
    const float* zc = (i & 1) ? a.zprev_next : a.z;                    // z^i
    float* zo = (i & 1) ? const_cast<float*>(a.z) : a.zprev_next;      // z^{i-1}, receives z^{i+1}
    const int* yr = ys[i & 1];
    if (i > 0 && m.nx == 1) {  // this round's batch rows, staged now (no spare buffer)
      if (warp == 0) {
        load_rows(i);
        __syncwarp();  // rows[] is written and read by warp 0 only here
        issue_rows(i, 0);
      }
      bulk::wait(&mbar[0], i & 1);
      x_norms(xr, xnb + (i & 1) * kRows, warp, kWarps);
      __syncthreads();
    }
    pmark(1);

    if (warp < nw1) {  // group 1: phase 1 and the partial logits
      // ---- phase 1: a1 = W1 x + b1 for (16 rows x U units), chunk by chunk
      for (int ch = 0; ch < nch; ++ch) {
        if (i == 0) bulk::wait(&mbar[2], ch & 1);
        // K is always split into kSlices slices (summed in slice order below), each
        // group-1 warp taking slices warp, warp + nw1, ...: a1's rounding does not
        // depend on the group sizes, so one round per launch (2 group-2 warps)
        // and several (4) give the same bits
        for (int sl = warp; sl < kSlices; sl += nw1) {
          // 8 row groups x 4 unit groups; row group rg takes batch rows rg and
          // rg + 8: with the 788-float row stride (197 float4 = 5 mod 8 bank
          // groups) the 8 rows of one 128-bit load land on 8 distinct bank groups
          // (rows 2rg, 2rg + 1 had 2-way conflicts)
          const int rg = lane >> 2, ug = lane & 3;
          const int t0 = rg;
          const int n4k = in_dim >> 2;
          const int k4a = sl * n4k / kSlices, k4b = (sl + 1) * n4k / kSlices;
          float acc[kTR][TU];
  #pragma unroll
          for (int u = 0; u < TU; ++u) {
  #pragma unroll
            for (int q = 0; q < kTR; ++q) acc[q][u] = 0.f;
          }
          const float4* xr0 = reinterpret_cast<const float4*>(xr + t0 * xld);
          const float4* xr1 = reinterpret_cast<const float4*>(xr + (t0 + kRows / kTR) * xld);
  #pragma unroll 2
          for (int k4 = k4a; k4 < k4b; ++k4) {
            float4 wv[TU];
  #pragma unroll
            for (int u = 0; u < TU; ++u) wv[u] = reinterpret_cast<const float4*>(w1s + (ug + kUG * u) * xld)[k4];
            const float4 x0 = xr0[k4], x1 = xr1[k4];
  #pragma unroll
            for (int u = 0; u < TU; ++u) {
              acc[0][u] = __fmaf_rn(wv[u].x, x0.x, acc[0][u]);
              acc[0][u] = __fmaf_rn(wv[u].y, x0.y, acc[0][u]);
              acc[0][u] = __fmaf_rn(wv[u].z, x0.z, acc[0][u]);
              acc[0][u] = __fmaf_rn(wv[u].w, x0.w, acc[0][u]);
              acc[1][u] = __fmaf_rn(wv[u].x, x1.x, acc[1][u]);
              acc[1][u] = __fmaf_rn(wv[u].y, x1.y, acc[1][u]);
              acc[1][u] = __fmaf_rn(wv[u].z, x1.z, acc[1][u]);
              acc[1][u] = __fmaf_rn(wv[u].w, x1.w, acc[1][u]);
            }
          }
  #pragma unroll
          for (int u = 0; u < TU; ++u) {
            const int ul = ug + kUG * u;
  #pragma unroll
            for (int q = 0; q < kTR; ++q) part[(sl * kRows + t0 + q * (kRows / kTR)) * CU + ul] = acc[q][u];
          }
        }
        for (int ul = warp; ul < CU; ul += nw1) {  // ||W1[u]|| (one warp per unit, fixed order)
          const float4* w4 = reinterpret_cast<const float4*>(w1s + ul * xld);
          float sq = 0.f;
          for (int f = lane; f < (in_dim >> 2); f += 32) {
            const float4 v = w4[f];
            sq = __fmaf_rn(v.x, v.x, sq); sq = __fmaf_rn(v.y, v.y, sq);
            sq = __fmaf_rn(v.z, v.z, sq); sq = __fmaf_rn(v.w, v.w, sq);
          }
  #pragma unroll
          for (int off = 16; off >= 1; off >>= 1) sq = __fadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, off));
          if (lane == 0) wn[ul] = sqrtf(sq);
        }
        group_sync(1, nt1);
        const int uc = ch * CU;  // first unit of the chunk within the block
        for (int q = tid; q < kRows * CU; q += nt1) {  // cross-warp sum, bias, certainty test
          const int t = q / CU, ul = q - t * CU;
          float s = 0.f;
          for (int w = 0; w < kSlices; ++w) s = __fadd_rn(s, part[(w * kRows + t) * CU + ul]);
          const float bias = b1s[uc + ul];
          const float av = __fadd_rn(s, bias);
          // fl(a) sums at most n = 4 ceil(in_dim / (4 kSlices)) + kSlices + 1 terms
          // along any path (a slice's FMA chain, the slice partials, the bias), so
          // |fl(a) - a| <= gamma_n (sum |w x| + |b|) <= gamma_n (||w|| ||x|| + |b|)
          // (Cauchy-Schwarz); the launcher's threshold 2^bexp >= 6 gamma_n keeps a
          // 6x margin over it and over the norms' own rounding (in_dim = 784:
          // n = 81, 2^-15; round 1's 2^-12 sent ~8x more entries to the Dot2).
          const float bound = __fmul_rn(__fmaf_rn(wn[ul], xnr[t], fabsf(bias)), m.bscale);  // exact: 2^bexp
          const int o = t * U + uc + ul;
          if (t < b && fabsf(av) <= bound) {
            const int slot = atomicAdd(&n_unc, 1);
            unc[slot] = (short)q;
            hs[o] = 0.f;
            msk[o] = 0;
          } else {
            const bool on = av > 0.f;
            hs[o] = (on && t < b) ? av : 0.f;
            msk[o] = (on && t < b) ? 1 : 0;
          }
        }
        group_sync(1, nt1);
        for (int q0 = warp; q0 < n_unc; q0 += nw1) {  // R18: decide near a kink at ~2^-48
          const int q = unc[q0], t = q / CU, ul = q - t * CU;
          const float4* w4 = reinterpret_cast<const float4*>(w1s + ul * xld);
          const float4* x4 = reinterpret_cast<const float4*>(xr + t * xld);
          f2 acc = {0.f, 0.f};
          for (int f = lane; f < (in_dim >> 2); f += 32) {
            const float4 av = w4[f], cv = x4[f];
            dot2::dot2_step(acc, av.x, cv.x);
            dot2::dot2_step(acc, av.y, cv.y);
            dot2::dot2_step(acc, av.z, cv.z);
            dot2::dot2_step(acc, av.w, cv.w);
          }
          acc = dot2::f2_add(dot2::warp_sum(acc), f2{b1s[uc + ul], 0.f});
          if (lane == 0) {
            const bool on = dot2::positive(acc.hi, acc.lo);
            const int o = t * U + uc + ul;
            hs[o] = on ? __fadd_rn(acc.hi, acc.lo) : 0.f;
            msk[o] = on ? 1 : 0;
          }
        }
        group_sync(1, nt1);  // every thread is done with this chunk's W1 rows and the list
        if (tid == 0) n_unc = 0;
        if (ch + 1 < nch && warp == 0) {  // (count == 1 whenever nch > 1)
          if (lane == 0) bulk::expect_tx(&mbar[2], rowb * CU);
          __syncwarp();
          for (int t = lane; t < CU; t += 32)
            bulk::copy(w1s + t * xld, W + (int64_t)(u0 + uc + CU + t) * in_dim, rowb, &mbar[2]);
        }
      }
      pmark(2);
      // partial logits of this unit block
      float* PL = m.PL + ((int64_t)(i & 1) * gridDim.x + cid) * npl;
      for (int q = tid; q < npl; q += nt1) {
        const int t = q / classes, c = q - t * classes;
        float s = 0.f;
#pragma unroll 8
        for (int ul = 0; ul < U; ++ul) s = __fmaf_rn(w2s[c * U + ul], hs[t * U + ul], s);
        PL[q] = s;
      }
      group_sync(1, nt1);
      if (tid == 0) st_release_gpu(fPL + 32 * cid, ep);  // my partial logits are written
      pmark(3);
    }
    // group 2 (UPDATE): with nzw = 0 every warp runs it here, after its partial
    // logits, filling the wait for the other CTAs' partials
    if (UPDATE && (nzw == 0 || warp >= nw1)) {
      const int zt = nzw ? tid - nt1 : tid;        // this group's thread index
      const int nzt = nzw ? kThr - nt1 : kThr;     // and size
      const int zw = nzw ? warp - nw1 : warp;      // and warp index
      // next round's batch rows: indices, labels and the TMA into the spare
      // buffer now, the norms once they have landed (after the z slice)
      const bool pre = m.nx == 2 && i + 1 < m.count;
      if (pre && zw == 0) {
        if (lane < kRows) {
          const int r = lane < b ? m.perm[m.pos0 + (int64_t)(i + 1) * m.kb + (int64_t)(m.j0 + j) * b + lane] : 0;
          rows[(i + 1) & 1][lane] = r;
          ys[(i + 1) & 1][lane] = lane < b ? m.y[r] : 0;
        }
        __syncwarp();
        if (lane == 0) bulk::expect_tx(&mbar[(i + 1) & 1], rowb * (uint32_t)b);
        __syncwarp();
        if (lane < b)
          bulk::copy(xs + (((i + 1) & 1) * kRows + lane) * xld, m.X + (int64_t)rows[(i + 1) & 1][lane] * in_dim,
                     rowb, &mbar[(i + 1) & 1]);
      }
      if (m.cl) {
        // ---- z^{i+1} on this CTA's 1/r of the unit block, from the cluster
        // peers' pre-update replicas W^i read from THEIR shared memory (DSMEM):
        // the block's W1 rows, b1, W2 columns (and b2) live only in the cluster
        if (i > 0) cluster_wait();  // (P_{i-1}) every peer holds W^i
        pmark(12);
        if (i == 0) {  // z^0 and z^{-1} of the block (later rounds: DSMEM stores of the peers)
          bulk::wait(&mbar[3], 0);
          bulk::wait(&mbar[4], 0);
        }
        namespace cg = cooperative_groups;
        const cg::cluster_group clu = cg::this_cluster();
        const int r = a.r, zb = i & 1;
        const int n4 = in_dim >> 2, nI = U * n4;
        const int it1 = (j + 1) * nI / r;
        for (int it = j * nI / r + zt; it < it1; it += nzt) {
          const int ul = it / n4, f4 = it - ul * n4;
          const int64_t o = (int64_t)(u0 + ul) * in_dim + 4 * f4;
          // z^i and z^{i-1} of the block are both on chip (zs[i & 1], zs[(i + 1) & 1])
          const float4 z0 = reinterpret_cast<const float4*>(zs + (zb * U + ul) * xld)[f4];
          const float4 zp0 = reinterpret_cast<const float4*>(zs + ((zb ^ 1) * U + ul) * xld)[f4];
          float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
          for (int l = 0; l < r; ++l) {  // corrections added in ascending learner
            const float4 w = reinterpret_cast<const float4*>(clu.map_shared_rank(w1s, l) + ul * xld)[f4];
            s0.x = __fadd_rn(s0.x, __fmul_rn(a.alpha, __fsub_rn(w.x, z0.x)));
            s0.y = __fadd_rn(s0.y, __fmul_rn(a.alpha, __fsub_rn(w.y, z0.y)));
            s0.z = __fadd_rn(s0.z, __fmul_rn(a.alpha, __fsub_rn(w.z, z0.z)));
            s0.w = __fadd_rn(s0.w, __fmul_rn(a.alpha, __fsub_rn(w.w, z0.w)));
          }
          float4 zn;
          zn.x = __fadd_rn(__fadd_rn(z0.x, s0.x), __fmul_rn(a.mu, __fsub_rn(z0.x, zp0.x)));
          zn.y = __fadd_rn(__fadd_rn(z0.y, s0.y), __fmul_rn(a.mu, __fsub_rn(z0.y, zp0.y)));
          zn.z = __fadd_rn(__fadd_rn(z0.z, s0.z), __fmul_rn(a.mu, __fsub_rn(z0.z, zp0.z)));
          zn.w = __fadd_rn(__fadd_rn(z0.w, s0.w), __fmul_rn(a.mu, __fsub_rn(z0.w, zp0.w)));
          *reinterpret_cast<float4*>(zo + o) = zn;
          // z^{i+1} into every peer's zs[(i + 1) & 1] (where z^{i-1} was: each CTA
          // reads only its own part of it, which only it overwrites)
          for (int l = 0; l < r; ++l)
            reinterpret_cast<float4*>(clu.map_shared_rank(zs, l) + ((zb ^ 1) * U + ul) * xld)[f4] = zn;
          bad |= !finite4(zn);
        }
        if (j == 0) {  // the block's W2 columns, b1 (and, block 0, b2): cluster rank 0
          const int nw2 = classes * U, nsm = nw2 + U + (blk == 0 ? classes : 0);
          for (int q = zt; q < nsm; q += nzt) {
            int64_t o;
            float z0, zp0;
            const float* src;  // this parameter's slot in a peer's shared memory
            float* zdst;       // and where z^{i+1} goes in every peer's (nullptr: b2)
            int so;
            if (q < nw2) {
              const int c = q / U, ul = q - c * U;
              o = oW2 + (int64_t)c * hidden + u0 + ul;
              z0 = zw2s[zb * 32 * U + q];
              zp0 = zw2s[(zb ^ 1) * 32 * U + q];
              src = w2s; so = q;
              zdst = zw2s + (zb ^ 1) * 32 * U + q;
            } else if (q < nw2 + U) {
              const int ul = q - nw2;
              o = ob1 + u0 + ul;
              z0 = zb1s[zb * U + ul];
              zp0 = zb1s[(zb ^ 1) * U + ul];
              src = b1s; so = ul;
              zdst = zb1s + (zb ^ 1) * U + ul;
            } else {
              const int c = q - nw2 - U;
              o = ob2 + c;
              z0 = ld_cg(zc + o);
              zp0 = ld_cg(zo + o);
              src = b2s; so = c;
              zdst = nullptr;
            }
            float acc = 0.f;
            for (int l = 0; l < r; ++l)
              acc = __fadd_rn(acc, __fmul_rn(a.alpha, __fsub_rn(clu.map_shared_rank(src, l)[so], z0)));
            const float zn = __fadd_rn(__fadd_rn(z0, acc), __fmul_rn(a.mu, __fsub_rn(z0, zp0)));
            zo[o] = zn;
            if (zdst)
              for (int l = 0; l < r; ++l) *clu.map_shared_rank(zdst, l) = zn;
            bad |= !isfinite(zn);
          }
        }
        // z^i of b2 (block 0's update): written by cluster 0 in round i - 1
        if (blk == 0 && zt < classes) zb2s[zt] = ld_cg(zc + ob2 + zt);
        pmark(13);
        cluster_arrive();  // (Z_i) my part of z^{i+1} is stored; I have read the peers' W^i
        pmark(14);
      } else {
        // ---- z^{i+1} on this CTA's slice, from the pre-update replicas W^i
        if (i > 0) {  // every CTA has stored W^i
          for (int c = zt; c < (int)gridDim.x; c += nzt) flag_poll(fP2 + 32 * c, ep - 1u);
          group_sync(2, nzt);
        }
        pmark(12);
        // z^i of b2 (block 0's update): complete since round i - 1's ZD flags
        if (blk == 0 && zt < classes) zb2s[zt] = ld_cg(zc + ob2 + zt);
          const int64_t per = (a.n4 + gridDim.x - 1) / gridDim.x;
          const int64_t c_lo = (int64_t)blockIdx.x * per;
          const int64_t c_hi = c_lo + per < a.n4 ? c_lo + per : a.n4;
          // two columns per thread and iteration, every load of a replica group issued
          // before its arithmetic (the compiler cannot hoist loads across the stores)
          const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int64_t c4 = c_lo + zt; c4 < c_hi; c4 += 2 * nzt) {
            const bool two = c4 + nzt < c_hi;
            const int64_t p0 = c4 << 2, p1 = (c4 + nzt) << 2;
            const float4 z0 = ld_z4(zc + p0), zp0 = ld_z4(zo + p0);
            const float4 z1 = two ? ld_z4(zc + p1) : zero;
            const float4 zp1 = two ? ld_z4(zo + p1) : zero;
            float4 s0 = zero, s1 = zero;
            for (int jj = 0; jj < a.r; jj += 4) {
              float4 w0[4], w1[4];
    #pragma unroll
              for (int u = 0; u < 4; ++u) {
                w0[u] = jj + u < a.r ? ld_z4(a.W + (int64_t)(jj + u) * a.ld + p0) : zero;
                w1[u] = two && jj + u < a.r ? ld_z4(a.W + (int64_t)(jj + u) * a.ld + p1) : zero;
              }
    #pragma unroll
              for (int u = 0; u < 4; ++u) {  // corrections added in ascending j
                if (jj + u < a.r) {
                  s0.x = __fadd_rn(s0.x, __fmul_rn(a.alpha, __fsub_rn(w0[u].x, z0.x)));
                  s0.y = __fadd_rn(s0.y, __fmul_rn(a.alpha, __fsub_rn(w0[u].y, z0.y)));
                  s0.z = __fadd_rn(s0.z, __fmul_rn(a.alpha, __fsub_rn(w0[u].z, z0.z)));
                  s0.w = __fadd_rn(s0.w, __fmul_rn(a.alpha, __fsub_rn(w0[u].w, z0.w)));
                  s1.x = __fadd_rn(s1.x, __fmul_rn(a.alpha, __fsub_rn(w1[u].x, z1.x)));
                  s1.y = __fadd_rn(s1.y, __fmul_rn(a.alpha, __fsub_rn(w1[u].y, z1.y)));
                  s1.z = __fadd_rn(s1.z, __fmul_rn(a.alpha, __fsub_rn(w1[u].z, z1.z)));
                  s1.w = __fadd_rn(s1.w, __fmul_rn(a.alpha, __fsub_rn(w1[u].w, z1.w)));
                }
              }
            }
            float4 zn;
            zn.x = __fadd_rn(__fadd_rn(z0.x, s0.x), __fmul_rn(a.mu, __fsub_rn(z0.x, zp0.x)));
            zn.y = __fadd_rn(__fadd_rn(z0.y, s0.y), __fmul_rn(a.mu, __fsub_rn(z0.y, zp0.y)));
            zn.z = __fadd_rn(__fadd_rn(z0.z, s0.z), __fmul_rn(a.mu, __fsub_rn(z0.z, zp0.z)));
            zn.w = __fadd_rn(__fadd_rn(z0.w, s0.w), __fmul_rn(a.mu, __fsub_rn(z0.w, zp0.w)));
            *reinterpret_cast<float4*>(zo + p0) = zn;
            bad |= !finite4(zn);
            if (two) {
              zn.x = __fadd_rn(__fadd_rn(z1.x, s1.x), __fmul_rn(a.mu, __fsub_rn(z1.x, zp1.x)));
              zn.y = __fadd_rn(__fadd_rn(z1.y, s1.y), __fmul_rn(a.mu, __fsub_rn(z1.y, zp1.y)));
              zn.z = __fadd_rn(__fadd_rn(z1.z, s1.z), __fmul_rn(a.mu, __fsub_rn(z1.z, zp1.z)));
              zn.w = __fadd_rn(__fadd_rn(z1.w, s1.w), __fmul_rn(a.mu, __fsub_rn(z1.w, zp1.w)));
              *reinterpret_cast<float4*>(zo + p1) = zn;
              bad |= !finite4(zn);
            }
          }
          pmark(13);
        group_sync(2, nzt);
        if (zt == 0) st_release_gpu(fZD + 32 * blockIdx.x, ep);  // done reading W^i, z^{i+1} written
        // every CTA has read W^i (before any replica store) and z^{i+1} is complete
        for (int c = zt; c < (int)gridDim.x; c += nzt) flag_poll(fZD + 32 * c, ep);
        group_sync(2, nzt);
        pmark(14);
        if (i + 1 < m.count && zw == 0) {  // prefetch round i + 1's z block
          fence_proxy_async();  // z^{i+1} was written by other CTAs (generic proxy)
          issue_z_warp(zo, (i + 1) & 1);
        }
      }
      if (pre) {  // the next round's norms
        bulk::wait(&mbar[(i + 1) & 1], ((i + 1) >> 1) & 1);
        x_norms(xs + ((i + 1) & 1) * kRows * xld, xnb + ((i + 1) & 1) * kRows, zw, nzt / 32);
      }
      pmark(15);
    }
    if (warp < nw1) {  // group 1: phase 2 up to da1

      // ---- phase 2 (group 1): learner j's logits (one TMA bulk copy of its partials)
      if (tid < nblk) flag_poll(fPL + 32 * (j * nblk + tid), ep);
      group_sync(1, nt1);
      // b2^i: block 0 of learner j stored it in m.B2[i & 1][j] in round i - 1,
      // before its partial-logit flag of round i
      // (cluster mode: block 0 keeps its own b2 in b2s, which its peers read through DSMEM)
      if (i > 0 && tid < classes && !(m.cl && blk == 0))
        b2s[tid] = ld_cg(m.B2 + ((i & 1) * m.a.r + j) * 32 + tid);
      pmark(4);
      if (tid == 0) {
        fence_proxy_async();
        const uint32_t bytes = 4u * (uint32_t)(nblk * npl);
        bulk::expect_tx(&mbar[5], bytes);
        bulk::copy(plg, m.PL + ((int64_t)(i & 1) * gridDim.x + (int64_t)j * nblk) * npl, bytes, &mbar[5]);
      }
      bulk::wait(&mbar[5], i & 1);
      if (i > 0) group_sync(1, nt1);  // b2s
      for (int q = tid; q < b * classes; q += nt1) {
        const int t = q / classes, c = q - t * classes;
        // four interleaved partial sums (blocks k = 0, 1, 2, 3 mod 4, each in
        // ascending order), combined as ((s0 + s1) + (s2 + s3)): a fixed order
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        int k = 0;
        for (; k + 4 <= nblk; k += 4) {
          s0 = __fadd_rn(s0, plg[k * npl + q]);
          s1 = __fadd_rn(s1, plg[(k + 1) * npl + q]);
          s2 = __fadd_rn(s2, plg[(k + 2) * npl + q]);
          s3 = __fadd_rn(s3, plg[(k + 3) * npl + q]);
        }
        for (; k < nblk; ++k) s0 = __fadd_rn(s0, plg[k * npl + q]);
        const float s = __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
        lg[t * 32 + c] = __fadd_rn(s, b2s[c]);
      }
      group_sync(1, nt1);
      pmark(5);
      if (classes <= 16) {  // two rows per warp (half-warps), bitwise the same
        for (int t = 2 * warp; t < b; t += 2 * nw1) {
          const bool v1 = t + 1 < b;
          halfwarp_softmax_grad(lg + t * 32, lg + (t + 1) * 32, classes, yr[t], v1 ? yr[t + 1] : 0, v1,
                                es + t * 32, es + (t + 1) * 32);
        }
      } else {
        for (int t = warp; t < b; t += nw1) warp_softmax_grad(lg + t * 32, classes, yr[t], es + t * 32);
      }
      group_sync(1, nt1);
      pmark(6);
      for (int q = tid; q < kRows * U; q += nt1) {  // da1 = (W2^T e) [a1 > 0]  (W2^i)
        const int t = q / U, ul = q - t * U;
        float s = 0.f;
        if (t < b)
          for (int c = 0; c < classes; ++c) s = __fmaf_rn(w2s[c * U + ul], es[t * 32 + c], s);
        das[q] = msk[q] ? s : 0.f;
      }
      if (UPDATE && m.cl) {  // the cluster barriers every thread takes part in
        if (i > 0) cluster_wait();  // (P_{i-1})
        cluster_arrive();           // (Z_i)
      }
      pmark(7);
    }
    __syncthreads();  // join: das; (UPDATE) every CTA's z slice done; next rows staged
    if (UPDATE && m.cl) cluster_wait();  // (Z_i) the cluster's z^{i+1} parts stored, W^i read
    // this round's z^i block (cluster mode: through DSMEM after round 0)
    if (UPDATE && !(m.cl && i > 0)) bulk::wait(&mbar[3 + (i & 1)], (i >> 1) & 1);
    pmark(8);

    // ---- phase 2 (all warps): gradients of the block and the replica update.
    // The small items (dW2, db1, db2) go to the highest thread indices, which
    // have no dW1 item when U / UT * n4 < 256 (k = 4: 196 items).
    const int zb = i & 1;
    {
      const int nw2 = classes * U, nsmall = nw2 + U + (blk == 0 ? classes : 0);
      for (int q = kThr - 1 - tid; q < nsmall; q += kThr) {
        if (q < nw2) {  // dW2 = e^T h / b (its columns)
          const int c = q / U, ul = q - c * U;
          float s = 0.f;
          for (int t = 0; t < b; ++t) s = __fmaf_rn(es[t * 32 + c], hs[t * U + ul], s);
          const float g = __fdiv_rn(s, fb);
          const int64_t o = oW2 + (int64_t)c * hidden + u0 + ul;
          if (wg) G[o] = g;
          if (UPDATE) {
            float cc;
            const float wv = elem_w(w2s[q], g, zw2s[zb * 32 * U + q], a.alpha, a.gamma, cc);
            W[o] = wv;
            w2s[q] = wv;  // (every da1 read of W2^i is done: the join)
            bad |= !isfinite(wv);
          }
        } else if (q < nw2 + U) {  // db1
          const int ul = q - nw2;
          float s = 0.f;
          for (int t = 0; t < b; ++t) s = __fadd_rn(s, das[t * U + ul]);
          const float g = __fdiv_rn(s, fb);
          if (wg) G[ob1 + u0 + ul] = g;
          if (UPDATE) {
            float cc;
            const float wv = elem_w(b1s[ul], g, zb1s[zb * U + ul], a.alpha, a.gamma, cc);
            W[ob1 + u0 + ul] = wv;
            b1s[ul] = wv;
            bad |= !isfinite(wv);
          }
        } else {  // db2 (block 0)
          const int c = q - nw2 - U;
          float s = 0.f;
          for (int t = 0; t < b; ++t) s = __fadd_rn(s, es[t * 32 + c]);
          const float g = __fdiv_rn(s, fb);
          if (wg) G[ob2 + c] = g;
          if (UPDATE) {
            float cc;
            const float wv = elem_w(b2s[c], g, zb2s[c], a.alpha, a.gamma, cc);
            W[ob2 + c] = wv;
            m.B2[(((i + 1) & 1) * m.a.r + j) * 32 + c] = wv;  // b2^{i+1} for the learner's CTAs
            if (m.cl) b2s[c] = wv;  // (after every read of b2^i in this CTA: logits, da1's join)
            bad |= !isfinite(wv);
          }
        }
      }
    }
    pmark(9);
    {  // dW1[u][f] = sum_t da1[t][u] x_t[f] / b: one item = 4 features x UT units
       // (UT float4 accumulators: one x load and UT/4 broadcast da1 loads per UT
       // x 4 FMAs), then the block's update of those UT W1 rows in place
      constexpr int UT = TU == 1 ? 4 : 8;
      const int n4 = in_dim >> 2, nq = (U / UT) * n4;
      const bool w_res = nch == 1;  // the whole block's W1 rows are in w1s
      const float* zsb = zs + (m.nzb == 2 ? zb : 0) * U * xld;
      for (int q = tid; q < nq; q += kThr) {
        const int ug = q / n4, f4 = q - ug * n4;
        const int ub = ug * UT;  // first unit of the item within the block
        // z^i (and W^i) rows from L2 when they are not staged: issued before the
        // FMAs so their latency overlaps them
        float4 zg[UT];
        if (UPDATE && !m.nzb) {
#pragma unroll
          for (int u = 0; u < UT; ++u) zg[u] = ld_z4(zc + (int64_t)(u0 + ub + u) * in_dim + 4 * f4);
        }
        float4 s[UT];
#pragma unroll
        for (int u = 0; u < UT; ++u) s[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int t = 0; t < b; ++t) {
          const float4 x = reinterpret_cast<const float4*>(xr + t * xld)[f4];
          float dv[UT];
#pragma unroll
          for (int u = 0; u < UT; u += 4) {
            const float4 d4 = *reinterpret_cast<const float4*>(das + t * U + ub + u);
            dv[u] = d4.x; dv[u + 1] = d4.y; dv[u + 2] = d4.z; dv[u + 3] = d4.w;
          }
#pragma unroll
          for (int u = 0; u < UT; ++u) {
            s[u].x = __fmaf_rn(dv[u], x.x, s[u].x);
            s[u].y = __fmaf_rn(dv[u], x.y, s[u].y);
            s[u].z = __fmaf_rn(dv[u], x.z, s[u].z);
            s[u].w = __fmaf_rn(dv[u], x.w, s[u].w);
          }
        }
#pragma unroll
        for (int u = 0; u < UT; ++u) {
          const int ul = ub + u;
          float4 g = s[u];
          if (pow2) {
            g.x = __fmul_rn(g.x, inv_b); g.y = __fmul_rn(g.y, inv_b);
            g.z = __fmul_rn(g.z, inv_b); g.w = __fmul_rn(g.w, inv_b);
          } else {
            g.x = __fdiv_rn(g.x, fb); g.y = __fdiv_rn(g.y, fb);
            g.z = __fdiv_rn(g.z, fb); g.w = __fdiv_rn(g.w, fb);
          }
          const int64_t o = (int64_t)(u0 + ul) * in_dim + 4 * f4;
          if (wg) *reinterpret_cast<float4*>(G + o) = g;
          if (UPDATE) {
            float4* ws = reinterpret_cast<float4*>(w1s + ul * xld) + f4;
            const float4 wv = w_res ? *ws : ld_z4(W + o);
            const float4 zv = m.nzb ? reinterpret_cast<const float4*>(zsb + ul * xld)[f4] : zg[u];
            const float4 wn4 = elem_w4(wv, g, zv, a.alpha, a.gamma);
            *reinterpret_cast<float4*>(W + o) = wn4;
            if (w_res) *ws = wn4;
            bad |= !finite4(wn4);
          }
        }
      }
    }
    pmark(10);
    // W^{i+1} of this block is stored (the next round's z slices read it)
    if (UPDATE && i + 1 < m.count && m.cl) {
      __syncthreads();   // shared buffers are reused by the next round
      cluster_arrive();  // (P_i) my W^{i+1} (shared memory) is complete for the peers
    } else if (UPDATE && i + 1 < m.count) {
      // released by the last warp of group 2, whose next duty is to wait for
      // every CTA's P2 anyway: the release waits ~1.4 us for this CTA's replica
      // stores, and issued by thread 0 it held up the next round's phase 1
      // (SMA_MLP_P2REL=0: thread 0, as before)
      flag_arrive(fP2 + 32 * blockIdx.x, ep, (nzw > 0 && m.p2rel) ? kThr - 32 : 0);
    } else {
      __syncthreads();  // shared buffers are reused by the next round
    }
    pmark(11);
  }
  if (UPDATE && a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
  if (PROF && (tid == 0 || tid == nt1))
    for (int q = 0; q < 16; ++q)
      if ((tid == 0) == (q < 12)) m.prof[blockIdx.x * 16 + q] = pacc[q];
}

size_t round_smem(int in_dim, int U, int CU, int nblk, int classes, int nx, int nzb) {
  const size_t xld = (size_t)in_dim + 4;
  const size_t fl = (size_t)nx * kRows * xld + (size_t)CU * xld + (size_t)nzb * U * xld +
                    (size_t)kSlices * kRows * CU + 2 * (size_t)kRows * U + 2 * (size_t)kRows * 32 +
                    2 * kRows + CU + 32 * (size_t)U + U + 2 * (32 * (size_t)U + U) +
                    (size_t)nblk * kRows * classes;
  return sizeof(float) * fl + (size_t)kRows * U + 16;
}

// Every CTA of the grid must be resident: CTAs wait on each other's flags.
// The launcher guarantees it by construction: grid <= #SMs and one CTA fits per SM
// (checked with the occupancy API), so once the previous kernel drains every
// CTA gets an SM.  SMA_MLP_COOP=1 adds the cooperative-launch attribute (the
// driver's own co-residency check), which also stops programmatic dependent
// launch from starting the next round's CTAs early (measured slower).
bool mlp_coop() {
  static const bool on = [] {
    const char* e = getenv("SMA_MLP_COOP");
    return e && e[0] == '1';
  }();
  return on;
}

// Warps of group 2 (see the kernel): measured best 2 for one round per launch
// and 4 for several (MLP rounds/s, b = 16, profiles/r02_mlp_fused.txt);
// SMA_MLP_ZWARPS = 0 / 2 / 4 forces it.
int mlp_zwarps(int count, bool cl = false) {
  static const int forced = [] {
    const char* e = getenv("SMA_MLP_ZWARPS");
    const int v = e ? atoi(e) : -1;
    return (v == 0 || v == 2 || v == 4) ? v : -1;
  }();
  return forced >= 0 ? forced : (count > 1 && !cl ? 4 : 2);
}

template <int TU, bool UPDATE>
cudaError_t launch_tu(const MlpRoundArgs& m, int grid, size_t smem, cudaStream_t s) {
  // b = 16 and classes = 10 unrolled where it fits the register budget (TU = 1
  // spills with it); other shapes use the generic instantiation
  constexpr int kFB = TU >= 2 ? kRows : 0;
  constexpr int kFC = TU >= 2 ? 10 : 0;
  constexpr int kFI = TU >= 2 ? 784 : 0;
  const bool fixed = m.b == kRows && m.classes == 10 && m.in_dim == 784;
  auto k = fixed ? (m.prof ? mlp_round_kernel<TU, UPDATE, true, kFB, kFC, kFI>
                           : mlp_round_kernel<TU, UPDATE, false, kFB, kFC, kFI>)
                 : (m.prof ? mlp_round_kernel<TU, UPDATE, true, 0, 0> : mlp_round_kernel<TU, UPDATE, false, 0, 0>);
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(k), (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThr, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[3];
  int n = 0;
  if (m.cl) {  // the r CTAs of a unit block as one cluster (blockIdx.x = blk * r + j)
    if (m.a.r > 8) {
      e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = (unsigned)m.a.r;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
    // every cluster must be resident at once (the CTAs wait on each other)
    cfg.attrs = at;
    cfg.numAttrs = n;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k, &cfg) != cudaSuccess || nc * m.a.r < grid) {
      cudaGetLastError();
      return cudaErrorNotSupported;
    }
  }
  if (mlp_coop()) {
    at[n].id = cudaLaunchAttributeCooperative;
    at[n].val.cooperative = 1;
    ++n;
  }
  if (pdl::enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k, m);
}
}  // namespace

// SMA_MLP_PROF=N (debugging only): launch N runs the PROF instantiation (cycle
// sums per phase boundary over its rounds) and the launcher prints the mean
// and max over CTAs, in us per round, to stderr, synchronising the stream.
static int prof_launch() {
  static const int n = [] {
    const char* e = getenv("SMA_MLP_PROF");
    return e ? atoi(e) : 0;
  }();
  return n;
}
unsigned long long* mlp_prof_buffer() {
  static unsigned long long* buf = nullptr;
  if (prof_launch() > 0 && !buf && cudaMalloc(&buf, 1024 * 16 * sizeof(unsigned long long)) != cudaSuccess)
    buf = nullptr;
  return buf;
}

bool mlp_fused_enabled() {
  static const bool on = [] {
    const char* e = getenv("SMA_MLP_FUSED");
    return !(e && e[0] == '0') && mlp_tc_policy() < 0;  // a forced GEMM policy keeps 5 kernels
  }();
  return on;
}

cudaError_t launch_mlp_round(const float* X, const int32_t* y, const int32_t* perm, int64_t pos0,
                             int64_t kb, int count, int b, int in_dim, int hidden, int classes,
                             int j0, float* PL, unsigned* bar, unsigned epoch, float* G,
                             const ReplicaArgs& a, bool update, int num_sms, cudaStream_t s) {
  if (!mlp_fused_enabled() || b > kRows || classes > 32 || (in_dim & 3) || a.r < 1 || count < 1 ||
      (count > 1 && !update) || (reinterpret_cast<uintptr_t>(X) & 15) || (a.ld & 3))
    return cudaErrorNotSupported;
  // the fewest units per CTA (4, 8, ..., 64) whose grid r * hidden / U fits one
  // CTA per SM, with U dividing hidden
  // (SMA_MLP_U = 4 ... 64, experiments: a larger U on fewer CTAs)
  static const int u_knob = [] {
    const char* e = getenv("SMA_MLP_U");
    return e ? atoi(e) : 0;
  }();
  int U = 0;
  for (int u = 4; u <= 64; u *= 2)
    if (hidden % u == 0 && (int64_t)a.r * (hidden / u) <= num_sms && u >= u_knob) {
      U = u;
      break;
    }
  if (!U) return cudaErrorNotSupported;
  // phase 1 runs over chunks of CU <= 32 units staged in shared memory; with one
  // chunk the block's weights stay resident.  Several rounds per launch need
  // that, and take (in order of preference) two batch-row buffers (the next
  // round's rows prefetched) and two z-row buffers (the next round's z block
  // prefetched) where they fit.
  const int CU = U < 32 ? U : 32;
  const int nblk = hidden / U;
  if (count > 1 && CU != U) return cudaErrorNotSupported;
  constexpr size_t kSmemMax = 225 * 1024;
  // Cluster mode (SMA_MLP_CLUSTER=1, read per launch; off by default): the r CTAs
  // of a unit block form a cluster and exchange z through DSMEM (no z slice,
  // no ZD / P2 flags, no z TMA after round 0); needs r a power of two <= 16 and
  // z^i and z^{i-1} of the block on chip (k <= 4 at the MLP shape).  Measured
  // slower than the flag protocol (profiles/r02_mlp_fused.txt: k = 4 70.2k vs
  // 77.2k rounds/s -- each cluster-scope release after the replica stores costs
  // ~1.3 us, and the DSMEM z parts on 2 warps lengthen group 2), kept as a
  // tested alternative (bitwise equal to the default).
  const char* cl_env = getenv("SMA_MLP_CLUSTER");
  const bool cl_knob = cl_env && cl_env[0] == '1';
  const bool cl_ok = cl_knob && update && CU == U && a.r >= 2 && a.r <= 16 && (a.r & (a.r - 1)) == 0 &&
                     mlp_zwarps(count) > 0;
  int nx = 1, nzb = 0;
  auto configure = [&](bool cl) -> bool {
    nx = 1;
    nzb = 0;
    if (count > 1) {
      const int cand_fl[3][2] = {{2, 2}, {2, 0}, {1, 0}};
      const int cand_cl[2][2] = {{2, 2}, {1, 2}};  // z^i and z^{i-1} of the block on chip
      const int nc = cl ? 2 : 3;
      for (int q = 0; q < nc; ++q) {
        const int* c = cl ? cand_cl[q] : cand_fl[q];
        if (round_smem(in_dim, U, CU, nblk, classes, c[0], c[1]) <= kSmemMax) {
          nx = c[0];
          nzb = c[1];
          return true;
        }
      }
      return false;
    }
    if (cl) {
      nzb = 2;
      return round_smem(in_dim, U, CU, nblk, classes, 1, 2) <= kSmemMax;
    }
    if (round_smem(in_dim, U, CU, nblk, classes, 1, 0) > kSmemMax) return false;
    if (update && CU == U && round_smem(in_dim, U, CU, nblk, classes, 1, 1) <= kSmemMax) nzb = 1;
    return true;
  };
  bool cl = cl_ok && configure(true);
  if (!cl && !configure(false)) return cudaErrorNotSupported;
  size_t smem = round_smem(in_dim, U, CU, nblk, classes, nx, nzb);
  MlpRoundArgs m{};
  m.X = X; m.y = y; m.perm = perm; m.pos0 = pos0;
  m.b = b; m.in_dim = in_dim; m.hidden = hidden; m.classes = classes; m.j0 = j0;
  m.kb = kb; m.count = count;
  {  // R18 threshold: 2^bexp >= 6 gamma_n, n = the longest summation path of a1
    const int n = 4 * ((in_dim / 4 + kSlices - 1) / kSlices) + kSlices + 1;
    m.bexp = (int)std::ceil(std::log2(6.0 * n * std::ldexp(1.0, -24) * (1.0 + 1e-6)));
    if (m.bexp < -15) m.bexp = -15;
    m.bscale = std::ldexp(1.0f, m.bexp);
  }
  m.nzw = mlp_zwarps(count, cl);
  m.U = U; m.nblk = nblk; m.nch = U / CU; m.nx = nx; m.nzb = nzb; m.cl = cl ? 1 : 0;
  m.PL = PL; m.B2 = PL + 2 * (size_t)num_sms * kRows * 32; m.G = G; m.bar = bar; m.a = a;
  m.fstride = num_sms; m.epoch = epoch;
  m.prof = mlp_prof_buffer();
  static const int p2rel = [] {
    const char* e = getenv("SMA_MLP_P2REL");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  m.p2rel = p2rel;
  const int grid = a.r * m.nblk;
  cudaError_t e;
#define SMA_MLP_ROUND(TU)                                                                      \
  e = update ? launch_tu<TU, true>(m, grid, smem, s) : launch_tu<TU, false>(m, grid, smem, s); \
  break;
  for (int attempt = 0; attempt < 2; ++attempt) {
    switch (CU / kUG) {
      case 1: SMA_MLP_ROUND(1)
      case 2: SMA_MLP_ROUND(2)
      case 4: SMA_MLP_ROUND(4)
      default: SMA_MLP_ROUND(8)
    }
    // the clusters cannot all be resident: the flag-only configuration
    if (e != cudaErrorNotSupported || !m.cl || !configure(false)) break;
    m.cl = 0;
    m.nx = nx;
    m.nzb = nzb;
    m.nzw = mlp_zwarps(count, false);
    smem = round_smem(in_dim, U, CU, nblk, classes, nx, nzb);
  }
#undef SMA_MLP_ROUND
  static int launches = 0;
  if (m.prof && e == cudaSuccess && ++launches == prof_launch()) {
    std::vector<unsigned long long> t((size_t)grid * 16);
    cudaStreamSynchronize(s);
    cudaMemcpy(t.data(), m.prof, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const char* names[] = {"loop", "rows(nx=1)", "phase1", "PL_flag", "PL_wait", "logits",
                           "softmax", "da1", "join+z_wait", "dW2/db", "dW1+update", "P2_flag",
                           "g2:rows+P2_wait", "g2:z_slice", "g2:ZD_flag+wait", "g2:prefetch+norms"};
    fprintf(stderr, "SMA_MLP_PROF launch %d (cluster=%d r=%d U=%d CU=%d nx=%d nzb=%d count=%d grid=%d "
            "smem=%zu) us per round at %.0f MHz, mean / max over CTAs:", launches, m.cl, a.r, U, CU,
            m.nx, m.nzb, count, grid, smem, clk_khz * 1e-3);
    for (int q = 0; q < 16; ++q) {
      double sum = 0, mx = 0;
      for (int c = 0; c < grid; ++c) {
        const double v = (double)t[(size_t)c * 16 + q];
        sum += v;
        mx = std::max(mx, v);
      }
      const double us = 1e3 / (clk_khz * (double)count);
      fprintf(stderr, " %s=%.2f/%.2f", names[q], sum / grid * us, mx * us);
    }
    fprintf(stderr, "\n");
  }
  return e;
}

}  // namespace sma
