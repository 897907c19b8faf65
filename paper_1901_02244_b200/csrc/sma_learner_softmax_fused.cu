// sma_learner_softmax_fused.cu -- config C1: the softmax-regression learner's
// gradient (a2', Eq. 2, back-propagation) AND the n = 1
// SMA round (a3-a7, Alg. 1 lines 9-13) of all r local learners, for `count`
// consecutive rounds of one epoch, in ONE launch of one thread-block cluster
// (sma_learner_step / sma_learner_steps on a single-GPU handle).
//
// Why: the C1 model is tiny (d = 7,850: 31 KB per replica), so a round is a
// chain of latencies, not bandwidth: the per-round kernels (logits,
// feature-sliced dW, the small-round replica kernel) pay three dependent
// launches plus the host's per-call cost, ~10 us per round.
//
// Layout: the m CTAs of the cluster split the in_dim features into m
// contiguous slices (float4 granularity).  CTA q owns, for EVERY learner j and
// class c, the weights W_j[c][slice q] -- and the same slice of z^i and
// z^{i-1} -- for the whole launch, in shared memory; the biases (classes
// values per learner) are replicated in every CTA and updated redundantly
// (same inputs, same operations: the same bits everywhere).  So the replica
// update and the central-model update of a parameter happen in the CTA that
// holds every replica of it: no data of W or z ever crosses CTAs.  Per round i
// (8 compute warps; a ninth, producer warp stages the batch-row slices of round
// i + 1 by TMA and reads the permutation of round i + 2 meanwhile):
//   P  partial logits of every (learner, row, class) over the CTA's features,
//      sent into slot q of the row's owner (row rr = j b + t, owner rr mod m) with
//      st.async (16-byte stores into distributed shared memory that count their
//      bytes on the receiver's mbarrier);
//   Z  while they fly (no gradient needed): z^{i+1} = (z^i + sum_j c_j) +
//      mu (z^i - z^{i-1}) with c_j = alpha (w_j^i - z^i) in ascending j (R7),
//      into the z^{i-1} half, each c_j kept;
//   S  the owner, once its mbarrier has all m slices' bytes: logits = partials
//      summed in ascending slice order + bias; e = softmax - onehot (two rows
//      per warp, the max-subtracted form of sma_softmax.cuh), broadcast to every
//      CTA the same way;
//   G  dW_j[c][slice] = e_j^T X_j / b (ascending t, then / b), db_j (replicated),
//      and right there w_j^{i+1} = fma(-gamma, g_j, w_j^i) - c_j  (the
//      arithmetic of replica_step_ldg<kFused>).
// No cluster-wide barrier per round: the partial buffers and their mbarriers
// alternate by round parity, and a CTA can be at most one round ahead of any
// other (it needs every CTA's partials of a round to finish it), so round
// i + 2's partials can only arrive after every CTA is done with round i's.
// Global memory is written once, after the last round (the slices of every
// w_j, of z^{count} and z^{count-1}, and the last round's gradient G, as
// sma_learner_grads leaves it).
//
// Deterministic (fixed summation orders), so several rounds per launch are
// bitwise equal to one round per launch; against the per-round kernels the
// logits differ in fp32 rounding (a sliced K order), both within the oracle
// bar.  Shapes outside it (b > 16, classes > 16, in_dim % 4, more learners than
// fit the shared memory, a cluster that cannot be resident) return
// cudaErrorNotSupported and the caller keeps the per-round kernels.
// SMA_SOFTMAX_CLUSTER=0 disables it; SMA_SOFTMAX_M=<m> forces the slice count.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cooperative_groups.h>

#include <array>
#include <map>
#include <mutex>

#include "sma_bulk.cuh"
#include "sma_pdl.cuh"
#include "sma_internal.h"

namespace sma {
namespace {
namespace cg = cooperative_groups;

constexpr int kProd = 8;                 // compute warps; warp kProd is the row producer
constexpr int kThr = (kProd + 1) * 32;
constexpr int kRows = 16;   // batch rows per learner (b <= 16)
constexpr int kCls = 16;    // classes <= 16 (two softmax rows per warp)
constexpr int kHalf = 8;    // classes per lane in the partial logits (two halves)
constexpr int kMaxR = 8;    // local learners

struct SoftmaxRoundArgs {
  const float* X;
  const int32_t* y;
  const int32_t* perm;    // this launch's epoch permutation
  int64_t pos0;           // perm position of learner 0, row 0 of the first round
  int64_t kb;             // perm positions per round (k * b)
  int count;              // rounds in this launch
  int b, in_dim, classes, j0;
  int m;                  // CTAs = feature slices
  int fs;                 // floats per slice buffer row (4 * max float4s per slice)
  float* G;               // gradients [r][ld] (the last round's)
  ReplicaArgs a;          // W, ld, r, z (z^0), zprev_next (z^{-1}), alpha, gamma, mu, nonfinite
  unsigned long long* prof;  // SMA_SOFTMAX_PROF: per-phase cycle sums [grid][2][8] (or nullptr)
};

// DSMEM producer / consumer primitives: st.async writes 16 bytes into a peer's
// shared memory and counts them on the peer's mbarrier (complete_tx with
// release semantics at cluster scope); the consumer's wait acquires at cluster
// scope.  No cluster-wide barrier per round.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, int rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}
__device__ __forceinline__ void st_async4(uint32_t addr, float4 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
               ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar) : "memory");
}
__device__ __forceinline__ void wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}

// SMA_SOFTMAX_PROF (debugging only): threads 0 and kProd * 32 (the producer)
// accumulate clock64() cycles per phase over the launch's rounds.
// FB, FC: the batch size and the class count as compile-time constants (16 and
// 10: config C1 -- the per-row and per-class loops unroll fully, the class
// guards fold) or 0 (read from the arguments).
template <bool PROF, int FB, int FC>
__global__ void __launch_bounds__(kThr, 1) softmax_cluster_kernel(const SoftmaxRoundArgs m) {
  extern __shared__ __align__(16) float sm[];
  const cg::cluster_group clu = cg::this_cluster();
  const int q = (int)clu.block_rank();  // feature slice
  const ReplicaArgs& a = m.a;
  const int r = a.r, M = m.m, in_dim = m.in_dim, classes = FC ? FC : m.classes, b = FB ? FB : m.b, FS = m.fs;
  const int n4k = in_dim >> 2;
  const int f4lo = q * n4k / M, f4hi = (q + 1) * n4k / M, nf4 = f4hi - f4lo;  // this slice
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool producer = warp == kProd;
  // batch rows of all learners, row rr = jj * b + t owned (summed, softmaxed)
  // by CTA rr % M in its slot rr / M
  const int R = r * b, maxown = (R + M - 1) / M, nown = (R - q + M - 1) / M;
  // shared memory (floats)
  float* ws = sm;                                  // [r][classes][FS] w_j slices
  float* gs = ws + r * classes * FS;               // [r][classes][FS] gradients (the last round's)
  float* cs = gs + r * classes * FS;               // [r][classes][FS] corrections alpha (w_j^i - z^i)
  float* zs = cs + r * classes * FS;               // [2][classes][FS] z^i / z^{i-1} slices
  float* xs = zs + 2 * classes * FS;               // [2][r][kRows][FS] batch-row slices
  float* pl = xs + 2 * r * kRows * FS;             // [2][M][maxown][kCls] partials of my rows (parity)
  float* es = pl + 2 * M * maxown * kCls;          // [r][kRows][32] softmax - onehot (every row)
  __shared__ float wb[kMaxR][kCls], cb[kMaxR][kCls], gb[kMaxR][kCls], zb[2][kCls];  // biases (replicated)
  __shared__ int rows[3][kMaxR][kRows], ys[2][kMaxR][kRows];
  // [0], [1] batch-row buffers full (TMA bytes + the producer's labels); [2] W
  // and z slices; [3], [4] partial logits of my rows; [5], [6] e rows; [7], [8]
  // batch-row buffers empty (the compute warps are done with them) -- all by
  // round parity
  __shared__ __align__(8) uint64_t mbar[9];
  const uint32_t slb = 16u * (uint32_t)nf4;        // bytes of one row / class slice
  const uint32_t plbytes = (uint32_t)(M * nown) * 64u;  // partial-logit bytes received per round
  const uint32_t ebytes = (uint32_t)R * 64u;             // e bytes received per round
  const float fb = (float)b;
  const bool pow2 = (b & (b - 1)) == 0;  // / b as an exact multiplication by 2^-k
  const float inv_b = 1.f / fb;
  const int64_t obias = (int64_t)classes * in_dim;

  // producer warp: perm -> rows[i % 3] (two rounds ahead), labels and the TMA of
  // round i's row slices (one round ahead)
  auto load_rows = [&](int i) {
    for (int u = lane; u < r * b; u += 32) {
      const int jj = u / b, t = u - jj * b;
      rows[i % 3][jj][t] = m.perm[m.pos0 + (int64_t)i * m.kb + (int64_t)(m.j0 + jj) * b + t];
    }
    __syncwarp();
  };
  auto issue_rows = [&](int i) {
    for (int u = lane; u < r * b; u += 32) {
      const int jj = u / b, t = u - jj * b;
      bulk::copy(xs + (((i & 1) * r + jj) * kRows + t) * FS, m.X + (int64_t)rows[i % 3][jj][t] * in_dim + 4 * f4lo,
                 slb, &mbar[i & 1]);
    }
    for (int u = lane; u < r * b; u += 32) {
      const int jj = u / b, t = u - jj * b;
      ys[i & 1][jj][t] = m.y[rows[i % 3][jj][t]];
    }
    __syncwarp();
    // the one arrival of the phase, after the labels: its release publishes them
    // (the TMA bytes may land before or after it; the phase needs both)
    if (lane == 0) bulk::expect_tx(&mbar[i & 1], slb * (uint32_t)(r * b));
  };
  // the compute warps' own barrier (the producer runs ahead on mbarriers)
  auto csync = [] { asm volatile("bar.sync 1, %0;" ::"n"(kProd * 32) : "memory"); };

  // ---- prologue: X, perm, y are never written by a kernel (before the PDL wait)
  if (tid == 0)
    for (int u = 0; u < 9; ++u) bulk::bar_init(&mbar[u]);
  for (int u = tid; u < 2 * r * kRows * FS; u += kThr) xs[u] = 0.f;  // rows t >= b stay 0
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");        // before the TMA writes
  __syncthreads();
  // split cluster barrier: arrive now (the mbarrier inits are fenced at cluster
  // scope), wait only right before this CTA's first st.async into a peer -- the
  // launch's staging overlaps the other CTAs' start
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  if (producer) {
    load_rows(0);
    if (m.count > 1) load_rows(1);
    issue_rows(0);
  }
  pdl::wait_and_release();  // the replicas and z were written by the previous launch
  if (warp == 1) {          // w_j, z^0 and z^{-1} slices of every class
    if (lane == 0) bulk::expect_tx(&mbar[2], slb * (uint32_t)(classes * (r + 2)));
    __syncwarp();
    for (int u = lane; u < classes * (r + 2); u += 32) {
      const int c = u % classes, v = u / classes;  // v < r: learner v; r: z; r + 1: z_prev
      const float* src = v < r ? a.W + (int64_t)v * a.ld : (v == r ? a.z : a.zprev_next);
      float* dst = v < r ? ws + (v * classes + c) * FS : zs + ((v - r) * classes + c) * FS;
      bulk::copy(dst, src + (int64_t)c * in_dim + 4 * f4lo, slb, &mbar[2]);
    }
  }
  if (tid < r * classes) {  // biases of every learner, z^0 / z^{-1} of the biases
    const int jj = tid / classes, c = tid - jj * classes;
    wb[jj][c] = a.W[(int64_t)jj * a.ld + obias + c];
    if (jj == 0) {
      zb[0][c] = a.z[obias + c];
      zb[1][c] = a.zprev_next[obias + c];
    }
  }
  bulk::wait(&mbar[2], 0);
  __syncthreads();
  // every CTA of the cluster is running and its mbarriers exist (the compute
  // warps send partial logits into them from round 0 on)
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");

  bool bad = false;
  unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = PROF ? clock64() : 0;
  auto pmark = [&](int ph) {
    if (PROF && (tid == 0 || tid == kProd * 32)) {
      const long long t = clock64();
      pacc[ph] += (unsigned long long)(t - tprev);
      tprev = t;
    }
  };
  for (int i = 0; i < m.count; ++i) {
    const int cur = i & 1;
    const float* xr = xs + cur * r * kRows * FS;
    float* plc = pl + cur * M * maxown * kCls;
    if (producer) {  // off the critical path: rows of round i + 1, perm of round i + 2
      if (i + 1 < m.count) {
        // buffer (i + 1) & 1 was last read in round i - 1
        if (i >= 1) bulk::wait(&mbar[7 + ((i + 1) & 1)], ((i - 1) >> 1) & 1);
        issue_rows(i + 1);
      }
      if (i + 2 < m.count) load_rows(i + 2);
      pmark(0);
      continue;
    } else {
      if (tid == 0) {  // this round's incoming partials (of my rows) and e rows
        if (nown > 0) bulk::expect_tx(&mbar[3 + cur], plbytes);
        bulk::expect_tx(&mbar[5 + cur], ebytes);
      }
      bulk::wait(&mbar[cur], (i >> 1) & 1);
      pmark(1);

      // ---- P: partial logits over this slice.  Warp item (learner jj, class
      // half h): lane = row t + 16 * (float4 parity), kHalf classes per lane;
      // the two parities combined with one xor-16 shuffle; lanes 0-15 then send
      // row t's kHalf values (two 16-byte st.async) into slot q of the row's owner.
      for (int it = warp; it < 2 * r; it += kProd) {
        const int jj = it >> 1, c0 = (it & 1) * kHalf;
        const int t = lane & 15, par = lane >> 4;
        float s[kHalf];
#pragma unroll
        for (int u = 0; u < kHalf; ++u) s[u] = 0.f;
        const float4* x4 = reinterpret_cast<const float4*>(xr + (jj * kRows + t) * FS);
        const float4* w4 = reinterpret_cast<const float4*>(ws + jj * classes * FS);
        for (int f = par; f < nf4; f += 2) {
          const float4 x = x4[f];
#pragma unroll
          for (int u = 0; u < kHalf; ++u) {
            if (c0 + u < classes) {
              const float4 w = w4[(c0 + u) * (FS / 4) + f];
              s[u] = __fmaf_rn(w.x, x.x, s[u]); s[u] = __fmaf_rn(w.y, x.y, s[u]);
              s[u] = __fmaf_rn(w.z, x.z, s[u]); s[u] = __fmaf_rn(w.w, x.w, s[u]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < kHalf; ++u) s[u] = __fadd_rn(s[u], __shfl_xor_sync(0xffffffffu, s[u], 16));
        if (par == 0 && t < b) {
          const int rr = jj * b + t, owner = rr % M;
          const uint32_t dst = mapa(smem_u32(plc + ((q * maxown + rr / M) * kCls + c0)), owner);
          const uint32_t pb = mapa(smem_u32(&mbar[3 + cur]), owner);
          st_async4(dst, make_float4(s[0], s[1], s[2], s[3]), pb);
          st_async4(dst + 16u, make_float4(s[4], s[5], s[6], s[7]), pb);
        }
      }
      // ---- Z (needs no gradient, so it runs while the partials fly):
      // z^{i+1} = (z^i + sum_j alpha (w_j^i - z^i)) + mu (z^i - z^{i-1}) from the
      // pre-update replicas, corrections in ascending j (R7), into the z^{i-1}
      // half; each c_j = alpha (w_j^i - z^i) kept for the replica update
      {
        const float* zc = zs + cur * classes * FS;   // z^i
        float* zn = zs + (cur ^ 1) * classes * FS;   // z^{i-1} -> z^{i+1}
        for (int u = tid; u < classes * nf4; u += kProd * 32) {
          const int c = u / nf4, f = u - c * nf4;
          const int o = c * FS + 4 * f;
          const float4 z = *reinterpret_cast<const float4*>(zc + o);
          const float4 zp = *reinterpret_cast<const float4*>(zn + o);
          float4 sacc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int jj = 0; jj < r; ++jj) {
            const float4 w = *reinterpret_cast<const float4*>(ws + jj * classes * FS + o);
            float4 cc;
            cc.x = __fmul_rn(a.alpha, __fsub_rn(w.x, z.x));
            cc.y = __fmul_rn(a.alpha, __fsub_rn(w.y, z.y));
            cc.z = __fmul_rn(a.alpha, __fsub_rn(w.z, z.z));
            cc.w = __fmul_rn(a.alpha, __fsub_rn(w.w, z.w));
            *reinterpret_cast<float4*>(cs + jj * classes * FS + o) = cc;
            sacc.x = __fadd_rn(sacc.x, cc.x); sacc.y = __fadd_rn(sacc.y, cc.y);
            sacc.z = __fadd_rn(sacc.z, cc.z); sacc.w = __fadd_rn(sacc.w, cc.w);
          }
          float4 znew;
          znew.x = __fadd_rn(__fadd_rn(z.x, sacc.x), __fmul_rn(a.mu, __fsub_rn(z.x, zp.x)));
          znew.y = __fadd_rn(__fadd_rn(z.y, sacc.y), __fmul_rn(a.mu, __fsub_rn(z.y, zp.y)));
          znew.z = __fadd_rn(__fadd_rn(z.z, sacc.z), __fmul_rn(a.mu, __fsub_rn(z.z, zp.z)));
          znew.w = __fadd_rn(__fadd_rn(z.w, sacc.w), __fmul_rn(a.mu, __fsub_rn(z.w, zp.w)));
          *reinterpret_cast<float4*>(zn + o) = znew;
          bad |= !(isfinite(znew.x) && isfinite(znew.y) && isfinite(znew.z) && isfinite(znew.w));
        }
        if (tid < classes) {  // the biases (replicated; every CTA the same bits)
          const int c = tid;
          const float z = zb[cur][c];
          float sacc = 0.f;
          for (int jj = 0; jj < r; ++jj) {
            cb[jj][c] = __fmul_rn(a.alpha, __fsub_rn(wb[jj][c], z));
            sacc = __fadd_rn(sacc, cb[jj][c]);
          }
          const float znew = __fadd_rn(__fadd_rn(z, sacc), __fmul_rn(a.mu, __fsub_rn(z, zb[cur ^ 1][c])));
          zb[cur ^ 1][c] = znew;
          bad |= !isfinite(znew);
        }
      }
      pmark(2);
      // ---- S (my rows): logits = partials in ascending slice order + bias,
      // e = softmax - onehot (two rows per warp, lane = class + 16 * row), sent
      // to every CTA as four 16-byte st.async per row (classes padded to 16)
      if (warp < (nown + 1) / 2) {
        wait_cluster(&mbar[3 + cur], (i >> 1) & 1);  // every slice's partials of my rows
        for (int ps = warp; ps < (nown + 1) / 2; ps += kProd) {
          const int so = 2 * ps + (lane >> 4), c = lane & 15;
          const bool vr = so < nown;
          const int rr = so * M + q, jj = vr ? rr / b : 0, t = vr ? rr - jj * b : 0;
          float v = -INFINITY;
          if (vr && c < classes) {
            const float* src = plc + so * kCls + c;
            float sum = 0.f;
            for (int p = 0; p < M; ++p) sum = __fadd_rn(sum, src[p * maxown * kCls]);
            v = __fadd_rn(sum, wb[jj][c]);
          }
          float mx = v;
#pragma unroll
          for (int off = 8; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
          const float ex = (vr && c < classes) ? expf(__fsub_rn(v, mx)) : 0.f;
          float den = ex;
#pragma unroll
          for (int off = 8; off >= 1; off >>= 1) den = __fadd_rn(den, __shfl_xor_sync(0xffffffffu, den, off));
          const float e = (vr && c < classes) ? __fsub_rn(__fdiv_rn(ex, den), c == ys[cur][jj][t] ? 1.f : 0.f) : 0.f;
          const float e1 = __shfl_down_sync(0xffffffffu, e, 1), e2 = __shfl_down_sync(0xffffffffu, e, 2),
                      e3 = __shfl_down_sync(0xffffffffu, e, 3);
          if (vr && (c & 3) == 0) {
            const uint32_t slot = smem_u32(es + (jj * kRows + t) * 32 + c), bar = smem_u32(&mbar[5 + cur]);
            const float4 v4 = make_float4(e, e1, e2, e3);
            for (int p = 0; p < M; ++p) st_async4(mapa(slot, p), v4, mapa(bar, p));
          }
        }
      }
      pmark(3);
      wait_cluster(&mbar[5 + cur], (i >> 1) & 1);  // every row's e of round i is here
      pmark(4);
    }
    csync();  // e of every row
    if (!producer) pmark(6);

    // ---- G: dW_j[c][f] over this slice, item (jj, float4 f, 4 classes), and
    // right there the replica update w' = fma(-gamma, g, w) - c  (Alg. 1 line 10
    // with replica_step_ldg<kFused>'s operation order)
    const bool last = i + 1 == m.count;
    if (!producer) {
      const int nqc = (classes + 3) >> 2;
      for (int it = tid; it < r * nf4 * nqc; it += kProd * 32) {
        const int h = it % nqc, rest = it / nqc, jj = rest / nf4, f = rest - jj * nf4;
        const int c0 = 4 * h;
        float4 s[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int t = 0; t < b; ++t) {
          const float4 x = reinterpret_cast<const float4*>(xr + (jj * kRows + t) * FS)[f];
          const float4 e4 = *reinterpret_cast<const float4*>(es + (jj * kRows + t) * 32 + c0);
          const float ev[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            s[u].x = __fmaf_rn(ev[u], x.x, s[u].x); s[u].y = __fmaf_rn(ev[u], x.y, s[u].y);
            s[u].z = __fmaf_rn(ev[u], x.z, s[u].z); s[u].w = __fmaf_rn(ev[u], x.w, s[u].w);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (c0 + u < classes) {
            float4 g = s[u];
            if (pow2) {
              g.x = __fmul_rn(g.x, inv_b); g.y = __fmul_rn(g.y, inv_b);
              g.z = __fmul_rn(g.z, inv_b); g.w = __fmul_rn(g.w, inv_b);
            } else {
              g.x = __fdiv_rn(g.x, fb); g.y = __fdiv_rn(g.y, fb);
              g.z = __fdiv_rn(g.z, fb); g.w = __fdiv_rn(g.w, fb);
            }
            const int o = (jj * classes + c0 + u) * FS + 4 * f;
            if (last) *reinterpret_cast<float4*>(gs + o) = g;
            float4* wp = reinterpret_cast<float4*>(ws + o);
            const float4 cc = *reinterpret_cast<const float4*>(cs + o);
            float4 w = *wp;
            w.x = __fsub_rn(__fmaf_rn(-a.gamma, g.x, w.x), cc.x);
            w.y = __fsub_rn(__fmaf_rn(-a.gamma, g.y, w.y), cc.y);
            w.z = __fsub_rn(__fmaf_rn(-a.gamma, g.z, w.z), cc.z);
            w.w = __fsub_rn(__fmaf_rn(-a.gamma, g.w, w.w), cc.w);
            *wp = w;
            bad |= !(isfinite(w.x) && isfinite(w.y) && isfinite(w.z) && isfinite(w.w));
          }
      }
      if (tid < r * classes) {  // db and the bias update (every CTA: replicated)
        const int jj = tid / classes, c = tid - jj * classes;
        float s = 0.f;
        for (int t = 0; t < b; ++t) s = __fadd_rn(s, es[(jj * kRows + t) * 32 + c]);
        const float g = pow2 ? __fmul_rn(s, inv_b) : __fdiv_rn(s, fb);
        if (last) gb[jj][c] = g;
        wb[jj][c] = __fsub_rn(__fmaf_rn(-a.gamma, g, wb[jj][c]), cb[jj][c]);
        bad |= !isfinite(wb[jj][c]);
      }
      pmark(5);
    }
    csync();  // w^{i+1}, z^{i+1} complete (the next round's partial logits)
    if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&mbar[7 + cur])) : "memory");
  }
  __syncthreads();  // the producer is done too
  if (PROF && (tid == 0 || tid == kProd * 32))
    for (int ph = 0; ph < 8; ++ph) m.prof[(blockIdx.x * 2 + (tid != 0)) * 8 + ph] = pacc[ph];

  // ---- write-back: this slice of every w_j, of z^{count} and z^{count-1}, and
  // of the last round's gradient; the biases from CTA 0
  {
    const int qn = m.count & 1;  // z^{count} in zs[qn] <-> global buffer qn
    float* zg[2] = {const_cast<float*>(a.z), a.zprev_next};
    for (int u = tid; u < (r + 2) * classes * nf4; u += kThr) {
      const int f = u % nf4, rest = u / nf4, c = rest % classes, v = rest / classes;
      const int64_t go = (int64_t)c * in_dim + 4 * (f4lo + f);
      if (v < r) {
        const int o = (v * classes + c) * FS + 4 * f;
        *reinterpret_cast<float4*>(a.W + (int64_t)v * a.ld + go) = *reinterpret_cast<const float4*>(ws + o);
        *reinterpret_cast<float4*>(m.G + (int64_t)v * a.ld + go) = *reinterpret_cast<const float4*>(gs + o);
      } else {
        const int zq = v == r ? qn : qn ^ 1;
        if (zq == qn || m.count > 1)  // (count == 1: z^0 is already there)
          *reinterpret_cast<float4*>(zg[zq] + go) = *reinterpret_cast<const float4*>(zs + (zq * classes + c) * FS + 4 * f);
      }
    }
    if (q == 0 && tid < r * classes) {
      const int jj = tid / classes, c = tid - jj * classes;
      a.W[(int64_t)jj * a.ld + obias + c] = wb[jj][c];
      m.G[(int64_t)jj * a.ld + obias + c] = gb[jj][c];
      if (jj == 0) {
        zg[qn][obias + c] = zb[qn][c];
        if (m.count > 1) zg[qn ^ 1][obias + c] = zb[qn ^ 1][c];
      }
    }
  }
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
  // No closing cluster barrier: every st.async aimed at this CTA carries data of
  // a round it waited for, so no peer addresses its shared memory after that.
}

size_t softmax_smem(int r, int b, int classes, int fs, int M) {
  const size_t npl = (size_t)((r * b + M - 1) / M) * kCls;
  return sizeof(float) * (3 * (size_t)r * classes * fs + 2 * (size_t)classes * fs + 2 * (size_t)r * kRows * fs +
                          2 * (size_t)M * npl + (size_t)r * kRows * 32);
}
}  // namespace

bool softmax_cluster_enabled() {
  static const bool on = [] {
    const char* e = getenv("SMA_SOFTMAX_CLUSTER");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t launch_softmax_cluster_rounds(const float* X, const int32_t* y, const int32_t* perm,
                                          int64_t pos0, int64_t kb, int count, int b, int in_dim,
                                          int classes, int j0, float* G, const ReplicaArgs& a,
                                          cudaStream_t s) {
  const int64_t d = (int64_t)classes * (in_dim + 1);
  if (!softmax_cluster_enabled() || count < 1 || a.r < 1 || a.r > kMaxR || b < 1 || b > kRows ||
      classes < 1 || classes > kCls || (in_dim & 3) || in_dim < 4 || a.d != d ||
      (reinterpret_cast<uintptr_t>(X) & 15) || (a.ld & 3))
    return cudaErrorNotSupported;
  static const int m_knob = [] {
    const char* e = getenv("SMA_SOFTMAX_M");
    return e ? atoi(e) : 0;
  }();
  const int n4k = in_dim / 4;
  static const int prof_n = [] {
    const char* e = getenv("SMA_SOFTMAX_PROF");
    return e ? atoi(e) : 0;
  }();
  static int nlaunch = 0;
  static unsigned long long* prof = nullptr;
  const bool do_prof = prof_n > 0 && ++nlaunch == prof_n;
  if (do_prof && !prof && cudaMalloc(&prof, 16 * 2 * 8 * sizeof(unsigned long long)) != cudaSuccess) return cudaErrorMemoryAllocation;
  const bool c1 = b == kRows && classes == 10;
  auto kfn = c1 ? (do_prof ? softmax_cluster_kernel<true, kRows, 10> : softmax_cluster_kernel<false, kRows, 10>)
                : (do_prof ? softmax_cluster_kernel<true, 0, 0> : softmax_cluster_kernel<false, 0, 0>);
  const void* fn = reinterpret_cast<const void*>(kfn);
  // The slice count: the most parallel (each slice >= 4 float4s) whose buffers
  // fit and whose cluster can be resident (> 8 needs a non-portable cluster,
  // which not every GPC may host); chosen once per (device, shape) -- the
  // attribute and occupancy queries cost host microseconds per call.
  struct Choice { int M, fs; size_t smem; };
  static std::mutex cache_mu;
  static std::map<std::array<int, 6>, Choice> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const std::array<int, 6> key = {dev, a.r, b, classes, in_dim, do_prof ? 1 : 0};  // (b picks the instantiation)
  Choice ch{0, 0, 0};
  {
    std::lock_guard<std::mutex> lock(cache_mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      ch = it->second;
    } else {
      const int cand[] = {16, 14, 12, 8, 7, 6, 4, 2, 1};
      for (int M : cand) {
        if (m_knob > 0 && M != m_knob) continue;
        if (M > 1 && n4k / M < 4) continue;
        // row stride in float4s made odd: the 8 rows of one 128-byte wavefront
        // land on distinct bank groups
        const int fs = 4 * (((n4k + M - 1) / M) | 1);
        const size_t smem = softmax_smem(a.r, b, classes, fs, M);
        if (smem > 225 * 1024) continue;
        e = ensure_dyn_smem(fn, (int)smem);
        if (e != cudaSuccess) return e;
        if (M > 8 && cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
          cudaGetLastError();
          continue;
        }
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3(M);
        q.blockDim = dim3(kThr);
        q.dynamicSmemBytes = smem;
        cudaLaunchAttribute qa;
        qa.id = cudaLaunchAttributeClusterDimension;
        qa.val.clusterDim.x = (unsigned)M;
        qa.val.clusterDim.y = 1;
        qa.val.clusterDim.z = 1;
        q.attrs = &qa;
        q.numAttrs = 1;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, kfn, &q) != cudaSuccess || nc < 1) {
          cudaGetLastError();
          continue;
        }
        ch = Choice{M, fs, smem};
        break;
      }
      cache[key] = ch;
    }
  }
  if (ch.M == 0) return cudaErrorNotSupported;
  const int M = ch.M, fs = ch.fs;
  const size_t smem = ch.smem;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(M);
    cfg.blockDim = dim3(kThr);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)M;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (pdl::enabled()) {
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.numAttrs = 2;
    }
    SoftmaxRoundArgs mm{};
    mm.X = X; mm.y = y; mm.perm = perm; mm.pos0 = pos0; mm.kb = kb; mm.count = count;
    mm.b = b; mm.in_dim = in_dim; mm.classes = classes; mm.j0 = j0; mm.m = M; mm.fs = fs;
    mm.G = G; mm.a = a; mm.prof = do_prof ? prof : nullptr;
    e = cudaLaunchKernelEx(&cfg, kfn, mm);
    if (do_prof && e == cudaSuccess) {  // mean over CTAs, us per round, per phase
      unsigned long long h[16 * 2 * 8];
      cudaStreamSynchronize(s);
      cudaMemcpy(h, prof, sizeof(unsigned long long) * M * 16, cudaMemcpyDeviceToHost);
      int khz = 0;
      cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
      const char* nm[7] = {"producer", "rows_wait", "partials+send+z", "my_rows_softmax", "e_wait", "dW+update", "csync_e(before dW)"};
      for (int w = 0; w < 2; ++w) {
        fprintf(stderr, "SMA_SOFTMAX_PROF M=%d r=%d count=%d thread %d:", M, a.r, count, w * kProd * 32);
        for (int ph = 0; ph < 7; ++ph) {
          double sum = 0;
          for (int c = 0; c < M; ++c) sum += (double)h[(c * 2 + w) * 8 + ph];
          fprintf(stderr, " %s=%.2f", nm[ph], sum / M / count / (khz * 1e-3));
        }
        fprintf(stderr, " (us/round)\n");
      }
    }
    return e;
  }
}

}  // namespace sma
