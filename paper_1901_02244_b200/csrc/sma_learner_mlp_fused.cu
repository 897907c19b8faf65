// sma_learner_mlp_fused.cu -- the MLP learner's gradient (a2', Eq. 2 P:228-232,
// back-propagation) for all r local learners AND, for the n = 1 round,
// the SMA update of every replica and of z (a3-a7, Alg. 1 lines 9-13), in ONE
// persistent kernel with two grid-wide barriers.
//
// Why: at the paper's small batches (b = 16) the learner is a chain of short
// dependent phases (layer 1 -> logits -> softmax -> head -> dW1 -> update).  As
// five kernels each boundary costs a drain + launch (PDL hides only part of it)
// and every phase re-stages its operands; measured 24 us per k = 4 round
// (DESIGN §13).  Here one CTA owns (learner j, a block of U hidden units) for
// the whole round, keeps the batch rows X_b, the block's W1 rows, W2 columns,
// b1 (and z's rows of the block) in shared memory -- staged once by TMA bulk
// copies -- together with h = relu(a1), the mask and da1, and exchanges only
// the (b x classes) partial logits through L2, across ONE grid barrier:
//
//   before   z^{i+1} on the CTA's 1/grid slice of the vector, from the PRE-update
//            replicas (Alg. 1 lines 9 + 13: z' = (z + sum_j alpha (w_j - z)) +
//            mu (z - z_prev), corrections in ascending j) -- it needs no
//            gradient, so it overlaps the TMA of the block, and nothing writes a
//            replica before the barrier;
//   phase 1  a1[t][u] = W1[u] . x_t + b1[u] for its units (fp32 FMA from shared
//            memory, K split over the 8 warps, a fixed-order cross-warp sum);
//            R18's mask decision is certain unless |a1| <= 2^-12 (||W1[u]||
//            ||x_t|| + |b1[u]|) -- the Cauchy-Schwarz bound of sum |w x|, > 40x
//            the fp32 error bound -- and only those few entries are recomputed
//            as a double-float Dot2 (~2^-48, like the oracle's fp64).
//            h = relu(a1); partial logits PL[j][blk][t][c] = sum_{u in blk}
//            W2[c][u] h[t][u] -> L2.
//   -- grid barrier --
//   phase 2  logits = b2 + sum_blk PL (ascending blk: every CTA of learner j
//            gets the same bits), e = softmax - onehot (one warp per row);
//            dW2 / db2 / db1 / da1 = (W2^T e) [a1 > 0] for its units, and
//            dW1[u][f] = sum_t da1[t][u] x_t[f] / b for its U rows -> G, and
//            (UPDATE) w' = fma(-gamma, g, w) - alpha (w - z) on the same block
//            right where its gradient is computed (every parameter of learner j
//            belongs to exactly one unit block; b2 to block 0).
//
// The arithmetic per element is replica_step_ldg<kFused>'s, so the round is
// bitwise the same as gradients-then-update with these gradients.
// The grid (r x hidden/U CTAs, U chosen so it fits one CTA per SM) is launched
// cooperatively, so every CTA is resident and the hand-rolled barrier (one
// arrival counter + a generation word in device memory, release / acquire at
// gpu scope) cannot deadlock.  Summation orders are fixed, so results are
// deterministic; they differ from the five-kernel path only in fp32 rounding
// (different K order of the layer-1 dot and of the logits).  Shapes outside
// this kernel (b > 16, in_dim % 4, hidden not a multiple of U, too many CTAs)
// return cudaErrorNotSupported and the caller uses the five-kernel path.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
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
// Weak coherent loads of the replicas: phase 3 of this same kernel rewrites
// them, so the read-only (.nc) path is not legal for W (PTX: .nc data must be
// read-only for the kernel's lifetime); no L1 allocation.
__device__ __forceinline__ float4 ld_w4(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_w(const float* p) {
  float v;
  asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
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
// the last arrival to the release).  Each CTA publishes this launch's epoch
// (a host-side launch counter, so flags only ever grow) in its own 128-byte
// line with a release store -- cumulative over the CTA's writes through the
// bar.sync before it -- and a consumer acquires exactly the lines it depends
// on, one thread per line, then bar.syncs.  Two such split-phase points:
//   PL flags: the partial logits of CTA c are written (consumers: the CTAs of
//             the same learner, right after their own partials);
//   ZD flags: CTA c's slice of z^{i+1} is computed, i.e. it has finished
//             reading the PRE-update replicas (consumers: every CTA, just
//             before its first replica store -- long satisfied by then).
__device__ __forceinline__ void flag_arrive(unsigned* line, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) st_release_gpu(line, epoch);
}
// Wait until lines[32 c] >= epoch for c in [0, n) (n <= blockDim.x).
__device__ __forceinline__ void flags_wait(const unsigned* lines, int n, unsigned epoch) {
  if ((int)threadIdx.x < n) {
    const long long t0 = clock64();
    while ((int)(ld_acquire_gpu(lines + 32 * threadIdx.x) - epoch) < 0)
      if (clock64() - t0 > 60000000000ll) __trap();  // ~30 s: a CTA never arrived
  }
  __syncthreads();
}
struct MlpRoundArgs {
  const float* X;
  const int32_t* y;
  const int32_t* perm;
  int64_t pos0;
  int b, in_dim, hidden, classes, j0;
  int U, nblk;            // hidden units per CTA, CTAs per learner
  int nch;                // phase-1 chunks of CU = TU * kUG units (U / CU)
  int stage_z;            // UPDATE: z's rows of the CTA's W1 block staged too
  float* PL;              // [r][nblk][kRows][classes] partial logits
  float* G;               // gradients [r][ld]
  unsigned* bar;          // flag lines: PL [grid][32], then ZD at bar + 32 * fstride
  int fstride;            // flag lines per kind (>= grid)
  unsigned epoch;         // this launch's number (host counter, >= 1, increasing)
  unsigned long long* prof;  // SMA_MLP_PROF: globaltimer stamps of CTA 0 (or nullptr)
  ReplicaArgs a;          // W, ld, r, z, zprev_next, alpha, gamma, mu, d, n4, nonfinite
};

// SMA_MLP_PROF: every CTA stamps %globaltimer at the phase boundaries
__device__ __forceinline__ void stamp(const MlpRoundArgs& m, int i) {
  if (m.prof && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    m.prof[blockIdx.x * 8 + i] = t;
  }
}

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
__device__ __forceinline__ float4 ld_nc4(const float* p) {  // z[cur]: never written by this kernel
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

// One CTA = (learner j, a block of U hidden units).  Phases:
//   prologue (before the PDL wait: X, perm, y are never written by a kernel)
//            batch rows -> shared memory (TMA), ||x_t||;
//   stage    W1 rows, W2 columns, b1 of the block (and, UPDATE, z's rows of the
//            block) -> shared memory with TMA bulk copies on one mbarrier;
//   z'       (UPDATE) z^{i+1} on this CTA's 1/grid slice of the vector from the
//            PRE-update replicas: z' = (z + sum_j alpha (w_j - z)) + mu (z - z_prev)
//            -- it needs no gradient, so it runs before the barrier while the
//            TMA lands, and no replica is written before the barrier;
//   phase 1  a1 for the block (K split over the warps, fixed-order cross-warp
//            sum), R18's certainty test + Dot2 for the uncertain, h = relu(a1),
//            partial logits -> L2;
//   -- the one grid barrier --
//   phase 2  logits (sum of the blocks' partials, ascending), softmax - onehot,
//            dW2 / db2 / db1 / dW1 of the block -> G and, UPDATE, the replica's
//            block updated right there: w' = fma(-gamma, g, w) - alpha (w - z)
//            with w from shared memory (it was staged for phase 1) and z staged
//            or loaded.
// Every parameter of learner j belongs to exactly one unit block (W1 rows,
// b1, W2 columns; b2 to block 0), so phase 2 touches disjoint data per CTA.
template <int TU, bool UPDATE>
__global__ void __launch_bounds__(kThr, 1) mlp_round_kernel(const MlpRoundArgs m) {
  constexpr int CU = TU * kUG;  // units per phase-1 chunk (<= 32)
  extern __shared__ __align__(16) float sm[];
  const int in_dim = m.in_dim, hidden = m.hidden, classes = m.classes, b = m.b, U = m.U;
  const int nch = m.nch;
  // rows padded to xld = in_dim + 4 floats: consecutive rows then start 20
  // banks apart (784 + 4 = 788 = 20 mod 32), so the 8 batch-row groups and the
  // 4 unit groups of a warp's 128-bit loads hit distinct banks (784 = 16 mod
  // 32 put rows t and t + 2 on the same banks)
  const int xld = in_dim + 4;
  float* xs = sm;                                        // [kRows][xld]
  float* w1s = xs + kRows * xld;                         // [CU][xld] W1 rows of a chunk
  float* zs = w1s + CU * xld;                            // [U][xld] z rows (stage_z)
  float* part = zs + (m.stage_z ? U * xld : 0);          // [kWarps][kRows][CU]
  float* hs = part + kWarps * kRows * CU;                // [kRows][U] relu(a1)
  float* das = hs + kRows * U;                           // [kRows][U] da1
  float* lg = das + kRows * U;                           // [kRows][32] logits
  float* es = lg + kRows * 32;                           // [kRows][32] softmax - onehot
  float* xn = es + kRows * 32;                           // [kRows] ||x_t||
  float* wn = xn + kRows;                                // [CU] ||W1[u]||
  float* w2s = wn + CU;                                  // [32][U] W2 columns of the block
  float* b1s = w2s + 32 * U;                             // [U] b1 of the block
  float* zw2s = b1s + U;                                 // [32][U] z of the W2 columns (UPDATE)
  float* zb1s = zw2s + 32 * U;                           // [U] z of b1 (UPDATE)
  unsigned char* msk = reinterpret_cast<unsigned char*>(zb1s + U);  // [kRows][U]
  __shared__ int rows[kRows], ys[kRows];
  __shared__ int n_unc;
  __shared__ short unc[kRows * 32];
  __shared__ __align__(8) uint64_t mbar[2];  // [0] batch rows, [1] weight / z blocks

  const int j = blockIdx.x / m.nblk, blk = blockIdx.x - j * m.nblk;
  const int u0 = blk * U;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const ReplicaArgs& a = m.a;
  const int64_t ob1 = (int64_t)hidden * in_dim, oW2 = ob1 + hidden, ob2 = oW2 + (int64_t)classes * hidden;
  float* W = a.W + (int64_t)j * a.ld;
  float* G = m.G + (int64_t)j * a.ld;

  // ---- prologue (X, perm, y are never written by a kernel: before the PDL wait)
  stamp(m, 0);
  if (tid < kRows) {
    const int r = tid < b ? m.perm[m.pos0 + (int64_t)(m.j0 + j) * b + tid] : 0;
    rows[tid] = r;
    ys[tid] = tid < b ? m.y[r] : 0;
  }
  if (tid == 0) {
    n_unc = 0;
    bulk::bar_init(&mbar[0]);
    bulk::bar_init(&mbar[1]);
  }
  __syncthreads();
  const uint32_t rowb = 4u * (uint32_t)in_dim;
  if (warp == 0) {  // the batch rows: one TMA bulk copy per row
    if (lane == 0) bulk::expect_tx(&mbar[0], rowb * (uint32_t)b);
    __syncwarp();
    if (lane < b) bulk::copy(xs + lane * xld, m.X + (int64_t)rows[lane] * in_dim, rowb, &mbar[0]);
  }
  for (int q = b * xld + tid; q < kRows * xld; q += kThr) xs[q] = 0.f;  // zero-padded batch rows
  bulk::wait(&mbar[0], 0);
  __syncthreads();
  for (int t = warp; t < kRows; t += kWarps) {  // ||x_t||
    const float4* x4 = reinterpret_cast<const float4*>(xs + t * xld);
    float s = 0.f;
    for (int f = lane; f < (in_dim >> 2); f += 32) {
      const float4 v = x4[f];
      s = __fmaf_rn(v.x, v.x, s); s = __fmaf_rn(v.y, v.y, s);
      s = __fmaf_rn(v.z, v.z, s); s = __fmaf_rn(v.w, v.w, s);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
    if (lane == 0) xn[t] = sqrtf(s);
  }
  stamp(m, 1);
  pdl::wait_and_release();  // the replicas and z were written by the previous round
  stamp(m, 2);

  // ---- stage the block: W1 chunk 0, W2 columns, b1 (and z's W1 rows) by TMA
  if (warp == 0) {
    if (lane == 0)
      bulk::expect_tx(&mbar[1], rowb * CU + 4u * (uint32_t)(classes * U + U) * (UPDATE ? 2u : 1u) +
                                    (m.stage_z ? rowb * (uint32_t)U : 0u));
    __syncwarp();
    for (int t = lane; t < CU; t += 32) bulk::copy(w1s + t * xld, W + (int64_t)(u0 + t) * in_dim, rowb, &mbar[1]);
    for (int c = lane; c < classes; c += 32)
      bulk::copy(w2s + c * U, W + oW2 + (int64_t)c * hidden + u0, 4u * U, &mbar[1]);
    if (lane == 0) bulk::copy(b1s, W + ob1 + u0, 4u * U, &mbar[1]);
    if (UPDATE) {
      for (int c = lane; c < classes; c += 32)
        bulk::copy(zw2s + c * U, a.z + oW2 + (int64_t)c * hidden + u0, 4u * U, &mbar[1]);
      if (lane == 0) bulk::copy(zb1s, a.z + ob1 + u0, 4u * U, &mbar[1]);
    }
    if (m.stage_z)
      for (int t = lane; t < U; t += 32)
        bulk::copy(zs + t * xld, a.z + (int64_t)(u0 + t) * in_dim, rowb, &mbar[1]);
  }

  bool bad = false;
  stamp(m, 3);

  // ---- phase 1: a1 = W1 x + b1 for (16 rows x U units), chunk by chunk
  for (int ch = 0; ch < nch; ++ch) {
    bulk::wait(&mbar[1], ch & 1);
    {
      const int rg = lane >> 2, ug = lane & 3;  // 8 row groups x 4 unit groups
      const int t0 = rg * kTR;
      const int n4k = in_dim >> 2;
      const int k4a = warp * n4k / kWarps, k4b = (warp + 1) * n4k / kWarps;
      float acc[kTR][TU];
#pragma unroll
      for (int u = 0; u < TU; ++u) {
#pragma unroll
        for (int i = 0; i < kTR; ++i) acc[i][u] = 0.f;
      }
      const float4* xr0 = reinterpret_cast<const float4*>(xs + t0 * xld);
      const float4* xr1 = reinterpret_cast<const float4*>(xs + (t0 + 1) * xld);
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
        for (int i = 0; i < kTR; ++i) part[(warp * kRows + t0 + i) * CU + ul] = acc[i][u];
      }
    }
    for (int ul = warp; ul < CU; ul += kWarps) {  // ||W1[u]|| (one warp per unit, fixed order)
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
    __syncthreads();
    const int uc = ch * CU;  // first unit of the chunk within the block
    for (int q = tid; q < kRows * CU; q += kThr) {  // cross-warp sum, bias, certainty test
      const int t = q / CU, ul = q - t * CU;
      float s = 0.f;
      for (int w = 0; w < kWarps; ++w) s = __fadd_rn(s, part[(w * kRows + t) * CU + ul]);
      const float bias = b1s[uc + ul];
      const float av = __fadd_rn(s, bias);
      // |fl(a) - a| <= ~110 u (sum |w x| + |b|) << 2^-12 (||w|| ||x|| + |b|)
      const float bound = ldexpf(__fmaf_rn(wn[ul], xn[t], fabsf(bias)), -12);
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
    __syncthreads();
    for (int i = warp; i < n_unc; i += kWarps) {  // R18: decide near a kink at ~2^-48
      const int q = unc[i], t = q / CU, ul = q - t * CU;
      const float4* w4 = reinterpret_cast<const float4*>(w1s + ul * xld);
      const float4* x4 = reinterpret_cast<const float4*>(xs + t * xld);
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
    __syncthreads();  // every thread is done with this chunk's W1 rows
    if (ch + 1 < nch && warp == 0) {
      if (lane == 0) {
        n_unc = 0;
        bulk::expect_tx(&mbar[1], rowb * CU);
      }
      __syncwarp();
      for (int t = lane; t < CU; t += 32)
        bulk::copy(w1s + t * xld, W + (int64_t)(u0 + uc + CU + t) * in_dim, rowb, &mbar[1]);
    }
  }
  // partial logits of this unit block
  float* PL = m.PL + (int64_t)blockIdx.x * kRows * classes;
  for (int q = tid; q < kRows * classes; q += kThr) {
    const int t = q / classes, c = q - t * classes;
    float s = 0.f;
#pragma unroll 8
    for (int ul = 0; ul < U; ++ul) s = __fmaf_rn(w2s[c * U + ul], hs[t * U + ul], s);
    PL[q] = s;
  }
  flag_arrive(m.bar + 32 * blockIdx.x, m.epoch);  // my partial logits are written
  stamp(m, 3);
  // ---- z^{i+1} on this CTA's slice, from the pre-update replicas (a3 + a7 sum),
  // while the other CTAs of this learner finish their partial logits
  if (UPDATE) {
    const int64_t per = (a.n4 + gridDim.x - 1) / gridDim.x;
    const int64_t c_lo = (int64_t)blockIdx.x * per;
    const int64_t c_hi = c_lo + per < a.n4 ? c_lo + per : a.n4;
    // two columns per thread and iteration, every load of a replica group issued
    // before its arithmetic (the compiler cannot hoist loads across the stores)
    const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t c4 = c_lo + tid; c4 < c_hi; c4 += 2 * kThr) {
      const bool two = c4 + kThr < c_hi;
      const int64_t p0 = c4 << 2, p1 = (c4 + kThr) << 2;
      const float4 z0 = ld_nc4(a.z + p0), zp0 = *reinterpret_cast<const float4*>(a.zprev_next + p0);
      const float4 z1 = two ? ld_nc4(a.z + p1) : zero;
      const float4 zp1 = two ? *reinterpret_cast<const float4*>(a.zprev_next + p1) : zero;
      float4 s0 = zero, s1 = zero;
      for (int jj = 0; jj < a.r; jj += 4) {
        float4 w0[4], w1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          w0[u] = jj + u < a.r ? ld_w4(a.W + (int64_t)(jj + u) * a.ld + p0) : zero;
          w1[u] = two && jj + u < a.r ? ld_w4(a.W + (int64_t)(jj + u) * a.ld + p1) : zero;
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
      *reinterpret_cast<float4*>(a.zprev_next + p0) = zn;
      bad |= !finite4(zn);
      if (two) {
        zn.x = __fadd_rn(__fadd_rn(z1.x, s1.x), __fmul_rn(a.mu, __fsub_rn(z1.x, zp1.x)));
        zn.y = __fadd_rn(__fadd_rn(z1.y, s1.y), __fmul_rn(a.mu, __fsub_rn(z1.y, zp1.y)));
        zn.z = __fadd_rn(__fadd_rn(z1.z, s1.z), __fmul_rn(a.mu, __fsub_rn(z1.z, zp1.z)));
        zn.w = __fadd_rn(__fadd_rn(z1.w, s1.w), __fmul_rn(a.mu, __fsub_rn(z1.w, zp1.w)));
        *reinterpret_cast<float4*>(a.zprev_next + p1) = zn;
        bad |= !finite4(zn);
      }
    }
  }
  if (UPDATE) flag_arrive(m.bar + 32 * (m.fstride + blockIdx.x), m.epoch);  // done reading W
  stamp(m, 4);
  flags_wait(m.bar + 32 * (j * m.nblk), m.nblk, m.epoch);  // learner j's partial logits
  stamp(m, 5);

  // ---- phase 2: logits, softmax, gradients of the block (+ the replica's update)
  const float* PLj = m.PL + (int64_t)j * m.nblk * kRows * classes;
  for (int q = tid; q < b * classes; q += kThr) {
    const int t = q / classes, c = q - t * classes;
    float s = 0.f;
    for (int k = 0; k < m.nblk; k += 16) {  // 16 loads in flight, added in ascending blk
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i)
        v[i] = k + i < m.nblk ? ld_cg(PLj + (int64_t)(k + i) * kRows * classes + q) : 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (k + i < m.nblk) s = __fadd_rn(s, v[i]);
    }
    lg[t * 32 + c] = __fadd_rn(s, ld_w(W + ob2 + c));
  }
  __syncthreads();
  for (int t = warp; t < b; t += kWarps) warp_softmax_grad(lg + t * 32, classes, ys[t], es + t * 32);
  __syncthreads();
  const float fb = (float)b;
  const bool pow2 = (b & (b - 1)) == 0;
  const float inv_b = 1.f / fb;
  // no replica may be written before every CTA has read the pre-update ones
  if (UPDATE) flags_wait(m.bar + 32 * m.fstride, gridDim.x, m.epoch);
  for (int q = tid; q < classes * U; q += kThr) {  // dW2 = e^T h / b (its columns)
    const int c = q / U, ul = q - c * U;
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fmaf_rn(es[t * 32 + c], hs[t * U + ul], s);
    const float g = __fdiv_rn(s, fb);
    const int64_t o = oW2 + (int64_t)c * hidden + u0 + ul;
    G[o] = g;
    if (UPDATE) {
      float cc;
      const float wv = elem_w(w2s[q], g, zw2s[q], a.alpha, a.gamma, cc);
      W[o] = wv;
      bad |= !isfinite(wv);
    }
  }
  if (blk == 0 && tid < classes) {  // db2
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, es[t * 32 + tid]);
    const float g = __fdiv_rn(s, fb);
    G[ob2 + tid] = g;
    if (UPDATE) {
      float cc;
      const float wv = elem_w(W[ob2 + tid], g, a.z[ob2 + tid], a.alpha, a.gamma, cc);
      W[ob2 + tid] = wv;
      bad |= !isfinite(wv);
    }
  }
  for (int q = tid; q < kRows * U; q += kThr) {  // da1 = (W2^T e) [a1 > 0]
    const int t = q / U, ul = q - t * U;
    float s = 0.f;
    if (t < b)
      for (int c = 0; c < classes; ++c) s = __fmaf_rn(w2s[c * U + ul], es[t * 32 + c], s);
    das[q] = msk[q] ? s : 0.f;
  }
  __syncthreads();
  for (int ul = tid; ul < U; ul += kThr) {  // db1
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, das[t * U + ul]);
    const float g = __fdiv_rn(s, fb);
    G[ob1 + u0 + ul] = g;
    if (UPDATE) {
      float cc;
      const float wv = elem_w(b1s[ul], g, zb1s[ul], a.alpha, a.gamma, cc);
      W[ob1 + u0 + ul] = wv;
      bad |= !isfinite(wv);
    }
  }
  {  // dW1[u][f] = sum_t da1[t][u] x_t[f] / b: one item = 4 features x UT units
     // (UT float4 accumulators: one x load and UT/4 broadcast da1 loads per UT
     // x 4 FMAs), then the block's update of those UT W1 rows in place
    constexpr int UT = TU == 1 ? 4 : 8;
    const int n4 = in_dim >> 2, nq = (U / UT) * n4;
    const bool w_res = nch == 1;  // the whole block's W1 rows are still in w1s
    for (int q = tid; q < nq; q += kThr) {
      const int ug = q / n4, f4 = q - ug * n4;
      const int ub = ug * UT;  // first unit of the item within the block
      float4 s[UT];
#pragma unroll
      for (int i = 0; i < UT; ++i) s[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int t = 0; t < b; ++t) {
        const float4 x = reinterpret_cast<const float4*>(xs + t * xld)[f4];
        float dv[UT];
#pragma unroll
        for (int i = 0; i < UT; i += 4) {
          const float4 d4 = *reinterpret_cast<const float4*>(das + t * U + ub + i);
          dv[i] = d4.x; dv[i + 1] = d4.y; dv[i + 2] = d4.z; dv[i + 3] = d4.w;
        }
#pragma unroll
        for (int i = 0; i < UT; ++i) {
          s[i].x = __fmaf_rn(dv[i], x.x, s[i].x);
          s[i].y = __fmaf_rn(dv[i], x.y, s[i].y);
          s[i].z = __fmaf_rn(dv[i], x.z, s[i].z);
          s[i].w = __fmaf_rn(dv[i], x.w, s[i].w);
        }
      }
#pragma unroll
      for (int i = 0; i < UT; ++i) {
        const int ul = ub + i;
        float4 g = s[i];
        if (pow2) {
          g.x = __fmul_rn(g.x, inv_b); g.y = __fmul_rn(g.y, inv_b);
          g.z = __fmul_rn(g.z, inv_b); g.w = __fmul_rn(g.w, inv_b);
        } else {
          g.x = __fdiv_rn(g.x, fb); g.y = __fdiv_rn(g.y, fb);
          g.z = __fdiv_rn(g.z, fb); g.w = __fdiv_rn(g.w, fb);
        }
        const int64_t o = (int64_t)(u0 + ul) * in_dim + 4 * f4;
        *reinterpret_cast<float4*>(G + o) = g;
        if (UPDATE) {
          const float4 wv = w_res ? reinterpret_cast<const float4*>(w1s + ul * xld)[f4] : ld_w4(W + o);
          const float4 zv = m.stage_z ? reinterpret_cast<const float4*>(zs + ul * xld)[f4] : ld_nc4(a.z + o);
          const float4 wn4 = elem_w4(wv, g, zv, a.alpha, a.gamma);
          *reinterpret_cast<float4*>(W + o) = wn4;
          bad |= !finite4(wn4);
        }
      }
    }
  }
  if (UPDATE && a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
  stamp(m, 6);
}

size_t round_smem(int in_dim, int U, int CU, bool stage_z) {
  const size_t xld = (size_t)in_dim + 4;
  const size_t fl = (size_t)kRows * xld + (size_t)CU * xld + (stage_z ? (size_t)U * xld : 0) +
                    (size_t)kWarps * kRows * CU + 2 * (size_t)kRows * U + 2 * (size_t)kRows * 32 +
                    kRows + CU + 2 * (32 * (size_t)U + U);
  return sizeof(float) * fl + (size_t)kRows * U + 16;
}

// Every CTA of the grid must be resident for the grid barrier.  The launcher
// guarantees it by construction: grid <= #SMs and one CTA fits per SM
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

template <int TU, bool UPDATE>
cudaError_t launch_tu(const MlpRoundArgs& m, int grid, size_t smem, cudaStream_t s) {
  auto k = mlp_round_kernel<TU, UPDATE>;
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
  cudaLaunchAttribute at[2];
  int n = 0;
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

// SMA_MLP_PROF=N (debugging only): CTA 0 stamps %globaltimer at the phase
// boundaries of every launch and the launcher prints launch N's phase times
// (us) to stderr, synchronising the stream after that launch.
static int prof_launch() {
  static const int n = [] {
    const char* e = getenv("SMA_MLP_PROF");
    return e ? atoi(e) : 0;
  }();
  return n;
}
unsigned long long* mlp_prof_buffer() {
  static unsigned long long* buf = nullptr;
  if (prof_launch() > 0 && !buf && cudaMalloc(&buf, 1024 * 8 * sizeof(unsigned long long)) != cudaSuccess)
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
                             int b, int in_dim, int hidden, int classes, int j0, float* PL,
                             unsigned* bar, unsigned epoch, float* G, const ReplicaArgs& a,
                             bool update, int num_sms, cudaStream_t s) {
  if (!mlp_fused_enabled() || b > kRows || classes > 32 || (in_dim & 3) || a.r < 1 ||
      (reinterpret_cast<uintptr_t>(X) & 15) || (a.ld & 3))
    return cudaErrorNotSupported;
  // the fewest units per CTA (4, 8, ..., 64) whose grid r * hidden / U fits one
  // CTA per SM (cooperative launch), with U dividing hidden
  int U = 0;
  for (int u = 4; u <= 64; u *= 2)
    if (hidden % u == 0 && (int64_t)a.r * (hidden / u) <= num_sms) {
      U = u;
      break;
    }
  if (!U) return cudaErrorNotSupported;
  // phase 1 runs over chunks of CU <= 32 units staged in shared memory; with
  // one chunk the block's W1 rows stay resident for the update, and z's rows
  // of the block are staged too when they fit
  const int CU = U < 32 ? U : 32;
  constexpr size_t kSmemMax = 225 * 1024;
  size_t smem = round_smem(in_dim, U, CU, false);
  if (smem > kSmemMax) return cudaErrorNotSupported;
  const bool stage_z = update && CU == U && round_smem(in_dim, U, CU, true) <= kSmemMax;
  if (stage_z) smem = round_smem(in_dim, U, CU, true);
  MlpRoundArgs m{};
  m.X = X; m.y = y; m.perm = perm; m.pos0 = pos0;
  m.b = b; m.in_dim = in_dim; m.hidden = hidden; m.classes = classes; m.j0 = j0;
  m.U = U; m.nblk = hidden / U; m.nch = U / CU; m.stage_z = stage_z ? 1 : 0;
  m.PL = PL; m.G = G; m.bar = bar; m.a = a;
  m.fstride = num_sms; m.epoch = epoch;
  m.prof = mlp_prof_buffer();
  const int grid = a.r * m.nblk;
  cudaError_t e;
#define SMA_MLP_ROUND(TU)                                                                      \
  e = update ? launch_tu<TU, true>(m, grid, smem, s) : launch_tu<TU, false>(m, grid, smem, s); \
  break;
  switch (CU / kUG) {
    case 1: SMA_MLP_ROUND(1)
    case 2: SMA_MLP_ROUND(2)
    case 4: SMA_MLP_ROUND(4)
    default: SMA_MLP_ROUND(8)
  }
#undef SMA_MLP_ROUND
  static int launches = 0;
  if (m.prof && e == cudaSuccess && ++launches == prof_launch()) {
    // per phase boundary: CTA 0's stamp and the latest over all CTAs, relative
    // to the earliest CTA start
    std::vector<unsigned long long> t((size_t)grid * 8);
    cudaStreamSynchronize(s);
    cudaMemcpy(t.data(), m.prof, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, mx[7] = {};
    for (int c = 0; c < grid; ++c) {
      t0 = std::min(t0, t[(size_t)c * 8]);
      for (int i = 0; i < 7; ++i) mx[i] = std::max(mx[i], t[(size_t)c * 8 + i]);
    }
    const char* names[] = {"start", "prologue", "pdl_wait", "phase1+PL", "zslice", "PL_wait",
                           "phase2+update"};
    fprintf(stderr, "SMA_MLP_PROF launch %d (r=%d U=%d CU=%d stage_z=%d grid=%d smem=%zu coop=%d) "
            "boundary: CTA0 / max over CTAs (us from the first CTA start):", launches, a.r, U, CU,
            (int)stage_z, grid, smem, (int)mlp_coop());
    for (int i = 0; i < 7; ++i)
      fprintf(stderr, " %s=%.2f/%.2f", names[i], (t[i] - t0) * 1e-3, (mx[i] - t0) * 1e-3);
    fprintf(stderr, "\n");
  }
  return e;
}

}  // namespace sma
