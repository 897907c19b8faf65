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
// the whole gradient, keeps the batch rows X_b, its h = relu(a1), the mask and
// da1 in shared memory, and exchanges only the (b x classes) partial logits
// through L2:
//
//   phase 1  a1[t][u] = W1[u] . x_t + b1[u] for its units (fp32 FMA, K split over
//            the 8 warps, a fixed-order cross-warp sum); R18's mask decision is
//            certain unless |a1| <= 2^-12 (||W1[u]|| ||x_t|| + |b1[u]|) -- the
//            Cauchy-Schwarz bound of sum |w x|, > 40x the fp32 error bound --
//            and only those few entries are recomputed as a double-float Dot2
//            (~2^-48, like the oracle's fp64).  h = relu(a1); partial logits
//            PL[j][blk][t][c] = sum_{u in blk} W2[c][u] h[t][u] -> L2.
//   -- grid barrier --
//   phase 2  logits = b2 + sum_blk PL (ascending blk: every CTA of learner j
//            gets the same bits), e = softmax - onehot (one warp per row);
//            dW2 / db2 / db1 / da1 = (W2^T e) [a1 > 0] for its units, and
//            dW1[u][f] = sum_t da1[t][u] x_t[f] / b for its U rows -> G.
//   -- grid barrier (UPDATE only) --
//   phase 3  the fused n = 1 round over every parameter (replica_step_ldg<kFused>'s
//            arithmetic: c = alpha (w - z), w' = fma(-gamma, g, w) - c, the
//            corrections summed in ascending j, z' = (z + sum c) + mu (z - z_prev)).
//
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

__device__ __forceinline__ float4 ld_cg4(const float* p) {  // L2 only: data written this kernel
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
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

// Grid-wide barrier over a co-resident grid: bar[0] arrivals, bar[1] generation.
// The generation is read BEFORE arriving, so it cannot already be the new one;
// the last arrival resets the counter and then publishes the next generation.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire_gpu(bar + 1);
    __threadfence();
    const unsigned prev = atomicAdd(bar, 1u);
    if (prev == gridDim.x - 1) {
      bar[0] = 0;
      st_release_gpu(bar + 1, gen + 1u);
    } else {
      while (ld_acquire_gpu(bar + 1) == gen) __nanosleep(20);
    }
    __threadfence();
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
  float* PL;              // [r][nblk][kRows][classes] partial logits
  float* G;               // gradients [r][ld]
  unsigned* bar;          // grid barrier state [2]
  unsigned long long* prof;  // SMA_MLP_PROF: globaltimer stamps of CTA 0 (or nullptr)
  ReplicaArgs a;          // W, ld, r, z, zprev_next, alpha, gamma, mu, d, n4, nonfinite
};

__device__ __forceinline__ void stamp(const MlpRoundArgs& m, int i) {
  if (m.prof && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    m.prof[i] = t;
  }
}

// sma_elem / central_elem of sma_kernels.cu.
__device__ __forceinline__ float elem_w(float w, float g, float z, float alpha, float gamma,
                                       float& c) {
  c = __fmul_rn(alpha, __fsub_rn(w, z));
  return __fsub_rn(__fmaf_rn(-gamma, g, w), c);
}

template <int TU, bool UPDATE>
__global__ void __launch_bounds__(kThr, 1) mlp_round_kernel(const MlpRoundArgs m) {
  constexpr int U = TU * kUG;
  extern __shared__ __align__(16) float sm[];
  const int in_dim = m.in_dim, hidden = m.hidden, classes = m.classes, b = m.b;
  float* xs = sm;                                   // [kRows][in_dim]
  float* part = xs + kRows * in_dim;                // [kWarps][kRows][U] K-split partials
  float* wn2 = part + kWarps * kRows * U;           // [kWarps][U] partial sum w^2
  float* hs = wn2 + kWarps * U;                     // [kRows][U] relu(a1)
  float* das = hs + kRows * U;                      // [kRows][U] da1 (mask applied)
  float* lg = das + kRows * U;                      // [kRows][32] logits
  float* es = lg + kRows * 32;                      // [kRows][32] softmax - onehot
  float* xn = es + kRows * 32;                      // [kRows] ||x_t||
  float* wn = xn + kRows;                           // [U] ||W1[u]||
  float* w2s = wn + U;                              // [32][U] W2 columns of my units
  unsigned char* msk = reinterpret_cast<unsigned char*>(w2s + 32 * U);  // [kRows][U]
  __shared__ int rows[kRows], ys[kRows];
  __shared__ int n_unc;
  __shared__ short unc[kRows * 64];
  __shared__ __align__(8) uint64_t mbar;

  const int j = blockIdx.x / m.nblk, blk = blockIdx.x - j * m.nblk;
  const int u0 = blk * U;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* W = m.a.W + (int64_t)j * m.a.ld;
  const float* W1 = W;
  const float* b1 = W + (int64_t)hidden * in_dim;
  const float* W2 = b1 + hidden;
  const float* b2 = W2 + (int64_t)classes * hidden;
  float* G = m.G + (int64_t)j * m.a.ld;

  // ---- prologue (X, perm, y are never written by a kernel: before the PDL wait)
  stamp(m, 0);
  if (tid < kRows) {
    const int r = tid < b ? m.perm[m.pos0 + (int64_t)(m.j0 + j) * b + tid] : 0;
    rows[tid] = r;
    ys[tid] = tid < b ? m.y[r] : 0;
  }
  if (tid == 0) n_unc = 0;
  __syncthreads();
  bulk::stage_rows_span(xs, m.X, rows, b, in_dim, in_dim, 0, nullptr, nullptr, 0, &mbar, 0, true);
  for (int q = b * in_dim + tid; q < kRows * in_dim; q += kThr) xs[q] = 0.f;  // padded rows
  __syncthreads();
  for (int t = warp; t < kRows; t += kWarps) {  // ||x_t||
    const float4* x4 = reinterpret_cast<const float4*>(xs + t * in_dim);
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
  pdl::wait_and_release();  // the replicas (W) were written by the previous round
  stamp(m, 2);

  // ---- phase 1: a1 = W1 x + b1 for (16 rows x U units), K split over the warps
  {
    const int rg = lane >> 2, ug = lane & 3;         // 8 row groups x 4 unit groups
    const int t0 = rg * kTR;
    const int n4k = in_dim >> 2;
    const int k4a = warp * n4k / kWarps, k4b = (warp + 1) * n4k / kWarps;
    float acc[kTR][TU], w2a[TU];
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      w2a[u] = 0.f;
#pragma unroll
      for (int i = 0; i < kTR; ++i) acc[i][u] = 0.f;
    }
    const float4* xr0 = reinterpret_cast<const float4*>(xs + t0 * in_dim);
    const float4* xr1 = reinterpret_cast<const float4*>(xs + (t0 + 1) * in_dim);
#pragma unroll 2
    for (int k4 = k4a; k4 < k4b; ++k4) {
      float4 wv[TU];
#pragma unroll
      for (int u = 0; u < TU; ++u)
        wv[u] = ld_w4(W1 + (int64_t)(u0 + ug + kUG * u) * in_dim + 4 * k4);
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
        if (rg == 0) {
          w2a[u] = __fmaf_rn(wv[u].x, wv[u].x, w2a[u]);
          w2a[u] = __fmaf_rn(wv[u].y, wv[u].y, w2a[u]);
          w2a[u] = __fmaf_rn(wv[u].z, wv[u].z, w2a[u]);
          w2a[u] = __fmaf_rn(wv[u].w, wv[u].w, w2a[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      const int ul = ug + kUG * u;
#pragma unroll
      for (int i = 0; i < kTR; ++i) part[(warp * kRows + t0 + i) * U + ul] = acc[i][u];
      if (rg == 0) wn2[warp * U + ul] = w2a[u];
    }
  }
  __syncthreads();
  for (int ul = tid; ul < U; ul += kThr) {  // ||W1[u]||, fixed warp order
    float s = 0.f;
    for (int w = 0; w < kWarps; ++w) s = __fadd_rn(s, wn2[w * U + ul]);
    wn[ul] = sqrtf(s);
  }
  __syncthreads();
  for (int q = tid; q < kRows * U; q += kThr) {  // cross-warp sum, bias, certainty test
    const int t = q / U, ul = q - t * U;
    float s = 0.f;
    for (int w = 0; w < kWarps; ++w) s = __fadd_rn(s, part[(w * kRows + t) * U + ul]);
    const float bias = ld_w(b1 + u0 + ul);
    const float a = __fadd_rn(s, bias);
    // |fl(a) - a| <= ~110 u (sum |w x| + |b|) << 2^-12 (||w|| ||x|| + |b|)
    const float bound = ldexpf(__fmaf_rn(wn[ul], xn[t], fabsf(bias)), -12);
    if (t < b && fabsf(a) <= bound) {
      const int slot = atomicAdd(&n_unc, 1);
      unc[slot] = (short)q;
      hs[q] = 0.f;
      msk[q] = 0;
    } else {
      const bool on = a > 0.f;
      hs[q] = (on && t < b) ? a : 0.f;
      msk[q] = (on && t < b) ? 1 : 0;
    }
  }
  __syncthreads();
  for (int i = warp; i < n_unc; i += kWarps) {  // R18: decide near a kink at ~2^-48
    const int q = unc[i], t = q / U, ul = q - t * U;
    const float* w = W1 + (int64_t)(u0 + ul) * in_dim;
    const float* x = xs + t * in_dim;
    f2 acc = {0.f, 0.f};
    for (int f = lane; f < (in_dim >> 2); f += 32) {
      const float4 av = ld_w4(w + 4 * f);
      const float4 cv = reinterpret_cast<const float4*>(x)[f];
      dot2::dot2_step(acc, av.x, cv.x);
      dot2::dot2_step(acc, av.y, cv.y);
      dot2::dot2_step(acc, av.z, cv.z);
      dot2::dot2_step(acc, av.w, cv.w);
    }
    acc = dot2::f2_add(dot2::warp_sum(acc), f2{ld_w(b1 + u0 + ul), 0.f});
    if (lane == 0) {
      const bool on = dot2::positive(acc.hi, acc.lo);
      hs[q] = on ? __fadd_rn(acc.hi, acc.lo) : 0.f;
      msk[q] = on ? 1 : 0;
    }
  }
  __syncthreads();
  stamp(m, 3);
  // partial logits of this unit block (W2's columns of the block staged once)
  for (int q = tid; q < classes * U; q += kThr) {
    const int c = q / U, ul = q - c * U;
    w2s[q] = ld_w(W2 + (int64_t)c * hidden + u0 + ul);
  }
  __syncthreads();
  float* PL = m.PL + (int64_t)blockIdx.x * kRows * classes;
  for (int q = tid; q < kRows * classes; q += kThr) {
    const int t = q / classes, c = q - t * classes;
    float s = 0.f;
#pragma unroll 8
    for (int ul = 0; ul < U; ++ul) s = __fmaf_rn(w2s[c * U + ul], hs[t * U + ul], s);
    PL[q] = s;
  }
  stamp(m, 4);
  grid_barrier(m.bar);
  stamp(m, 5);

  // ---- phase 2: logits, softmax, head, dW1 for this unit block
  const float* PLj = m.PL + (int64_t)j * m.nblk * kRows * classes;
  for (int q = tid; q < b * classes; q += kThr) {
    const int t = q / classes, c = q - t * classes;
    float s = 0.f;
    int k = 0;
    for (; k + 8 <= m.nblk; k += 8) {  // 8 loads in flight, added in ascending blk
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = ld_cg(PLj + (int64_t)(k + i) * kRows * classes + q);
#pragma unroll
      for (int i = 0; i < 8; ++i) s = __fadd_rn(s, v[i]);
    }
    for (; k < m.nblk; ++k) s = __fadd_rn(s, ld_cg(PLj + (int64_t)k * kRows * classes + q));
    lg[t * 32 + c] = __fadd_rn(s, ld_w(b2 + c));
  }
  __syncthreads();
  for (int t = warp; t < b; t += kWarps) warp_softmax_grad(lg + t * 32, classes, ys[t], es + t * 32);
  __syncthreads();
  const float fb = (float)b;
  const bool pow2 = (b & (b - 1)) == 0;
  const float inv_b = 1.f / fb;
  float* gW2 = G + (int64_t)hidden * in_dim + hidden;
  for (int q = tid; q < classes * U; q += kThr) {  // dW2 = e^T h / b (its columns)
    const int c = q / U, ul = q - c * U;
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fmaf_rn(es[t * 32 + c], hs[t * U + ul], s);
    gW2[(int64_t)c * hidden + u0 + ul] = __fdiv_rn(s, fb);
  }
  if (blk == 0 && tid < classes) {  // db2
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, es[t * 32 + tid]);
    gW2[(int64_t)classes * hidden + tid] = __fdiv_rn(s, fb);
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
    G[(int64_t)hidden * in_dim + u0 + ul] = __fdiv_rn(s, fb);
  }
  {  // dW1[u][f] = sum_t da1[t][u] x_t[f] / b, 4 features per thread
    const int n4 = in_dim >> 2;
    for (int q = tid; q < U * n4; q += kThr) {
      const int ul = q / n4, f4 = q - ul * n4;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int t = 0; t < b; ++t) {
        const float a = das[t * U + ul];
        const float4 x = reinterpret_cast<const float4*>(xs + t * in_dim)[f4];
        s.x = __fmaf_rn(a, x.x, s.x);
        s.y = __fmaf_rn(a, x.y, s.y);
        s.z = __fmaf_rn(a, x.z, s.z);
        s.w = __fmaf_rn(a, x.w, s.w);
      }
      if (pow2) {
        s.x = __fmul_rn(s.x, inv_b); s.y = __fmul_rn(s.y, inv_b);
        s.z = __fmul_rn(s.z, inv_b); s.w = __fmul_rn(s.w, inv_b);
      } else {
        s.x = __fdiv_rn(s.x, fb); s.y = __fdiv_rn(s.y, fb);
        s.z = __fdiv_rn(s.z, fb); s.w = __fdiv_rn(s.w, fb);
      }
      reinterpret_cast<float4*>(G + (int64_t)(u0 + ul) * in_dim)[f4] = s;
    }
  }
  stamp(m, 6);
  if (!UPDATE) return;
  grid_barrier(m.bar);
  stamp(m, 7);

  // ---- phase 3: the fused n = 1 round over all parameters (a3-a7)
  const ReplicaArgs& a = m.a;
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * kThr;
  for (int64_t c4 = (int64_t)blockIdx.x * kThr + tid; c4 < a.n4; c4 += stride) {
    const int64_t p0 = c4 << 2;
    const float4 z = *reinterpret_cast<const float4*>(a.z + p0);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int jj = 0;
    for (; jj + 4 <= a.r; jj += 4) {
      float4 w[4], g[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = ld_cg4(a.W + (int64_t)(jj + u) * a.ld + p0);
#pragma unroll
      for (int u = 0; u < 4; ++u) g[u] = ld_cg4(m.G + (int64_t)(jj + u) * a.ld + p0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float c;
        w[u].x = elem_w(w[u].x, g[u].x, z.x, a.alpha, a.gamma, c); acc.x = __fadd_rn(acc.x, c);
        w[u].y = elem_w(w[u].y, g[u].y, z.y, a.alpha, a.gamma, c); acc.y = __fadd_rn(acc.y, c);
        w[u].z = elem_w(w[u].z, g[u].z, z.z, a.alpha, a.gamma, c); acc.z = __fadd_rn(acc.z, c);
        w[u].w = elem_w(w[u].w, g[u].w, z.w, a.alpha, a.gamma, c); acc.w = __fadd_rn(acc.w, c);
        *reinterpret_cast<float4*>(a.W + (int64_t)(jj + u) * a.ld + p0) = w[u];
        bad |= !(isfinite(w[u].x) && isfinite(w[u].y) && isfinite(w[u].z) && isfinite(w[u].w));
      }
    }
    for (; jj < a.r; ++jj) {
      float4 w = ld_cg4(a.W + (int64_t)jj * a.ld + p0);
      const float4 g = ld_cg4(m.G + (int64_t)jj * a.ld + p0);
      float c;
      w.x = elem_w(w.x, g.x, z.x, a.alpha, a.gamma, c); acc.x = __fadd_rn(acc.x, c);
      w.y = elem_w(w.y, g.y, z.y, a.alpha, a.gamma, c); acc.y = __fadd_rn(acc.y, c);
      w.z = elem_w(w.z, g.z, z.z, a.alpha, a.gamma, c); acc.z = __fadd_rn(acc.z, c);
      w.w = elem_w(w.w, g.w, z.w, a.alpha, a.gamma, c); acc.w = __fadd_rn(acc.w, c);
      *reinterpret_cast<float4*>(a.W + (int64_t)jj * a.ld + p0) = w;
      bad |= !(isfinite(w.x) && isfinite(w.y) && isfinite(w.z) && isfinite(w.w));
    }
    const float4 zp = *reinterpret_cast<const float4*>(a.zprev_next + p0);
    float4 zn;
    zn.x = __fadd_rn(__fadd_rn(z.x, acc.x), __fmul_rn(a.mu, __fsub_rn(z.x, zp.x)));
    zn.y = __fadd_rn(__fadd_rn(z.y, acc.y), __fmul_rn(a.mu, __fsub_rn(z.y, zp.y)));
    zn.z = __fadd_rn(__fadd_rn(z.z, acc.z), __fmul_rn(a.mu, __fsub_rn(z.z, zp.z)));
    zn.w = __fadd_rn(__fadd_rn(z.w, acc.w), __fmul_rn(a.mu, __fsub_rn(z.w, zp.w)));
    *reinterpret_cast<float4*>(a.zprev_next + p0) = zn;
    bad |= !(isfinite(zn.x) && isfinite(zn.y) && isfinite(zn.z) && isfinite(zn.w));
  }
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
  stamp(m, 8);
}

size_t round_smem(int in_dim, int U) {
  return sizeof(float) * ((size_t)kRows * in_dim + (size_t)kWarps * kRows * U + (size_t)kWarps * U +
                          2 * (size_t)kRows * U + 2 * (size_t)kRows * 32 + kRows + U + 32 * (size_t)U) +
         (size_t)kRows * U + 16;
}

template <int TU, bool UPDATE>
cudaError_t launch_tu(const MlpRoundArgs& m, int grid, size_t smem, cudaStream_t s) {
  auto k = mlp_round_kernel<TU, UPDATE>;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(k), (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThr);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  at[n].id = cudaLaunchAttributeCooperative;  // every CTA resident: the grid barrier is safe
  at[n].val.cooperative = 1;
  ++n;
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
  if (prof_launch() > 0 && !buf && cudaMalloc(&buf, 16 * sizeof(unsigned long long)) != cudaSuccess)
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
                             unsigned* bar, float* G, const ReplicaArgs& a, bool update,
                             int num_sms, cudaStream_t s) {
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
  const size_t smem = round_smem(in_dim, U);
  if (smem > 200 * 1024) return cudaErrorNotSupported;
  MlpRoundArgs m{};
  m.X = X; m.y = y; m.perm = perm; m.pos0 = pos0;
  m.b = b; m.in_dim = in_dim; m.hidden = hidden; m.classes = classes; m.j0 = j0;
  m.U = U; m.nblk = hidden / U;
  m.PL = PL; m.G = G; m.bar = bar; m.a = a;
  m.prof = mlp_prof_buffer();
  const int grid = a.r * m.nblk;
  cudaError_t e;
#define SMA_MLP_ROUND(TU)                                                                      \
  e = update ? launch_tu<TU, true>(m, grid, smem, s) : launch_tu<TU, false>(m, grid, smem, s); \
  break;
  switch (U / kUG) {
    case 1: SMA_MLP_ROUND(1)
    case 2: SMA_MLP_ROUND(2)
    case 4: SMA_MLP_ROUND(4)
    case 8: SMA_MLP_ROUND(8)
    default: SMA_MLP_ROUND(16)
  }
#undef SMA_MLP_ROUND
  static int launches = 0;
  if (m.prof && e == cudaSuccess && ++launches == prof_launch()) {
    unsigned long long t[16] = {};
    cudaStreamSynchronize(s);
    cudaMemcpy(t, m.prof, sizeof t, cudaMemcpyDeviceToHost);
    const char* names[] = {"prologue", "pdl_wait", "phase1", "partial_logits", "barrier1",
                           "phase2", "barrier2", "phase3"};
    fprintf(stderr, "SMA_MLP_PROF launch %d (r=%d U=%d grid=%d):", launches, a.r, U, grid);
    for (int i = 0; i < 8; ++i) fprintf(stderr, " %s=%.2f", names[i], (t[i + 1] - t[i]) * 1e-3);
    fprintf(stderr, " total=%.2f us\n", (t[8] - t[0]) * 1e-3);
  }
  return e;
}

}  // namespace sma
