// sma_learner_mlp.cu -- NEXT-2: the built-in MLP learner (in_dim-hidden-classes,
// ReLU; "MLP (784-256-10)"), batch-mean gradient (Eq. 2, PAPER.md:
// 228-232) by back-propagation, for all r local replicas.
//
// Three small kernels per round (the learner is latency-bound at b = 16):
//   1. mlp_hidden_kernel  grid (r, hidden/8): gather the batch rows into shared
//      memory; pre-activations a1 = W1 x + b1 in fp32 with an a-priori error
//      bound, recomputed in double-float (Dot2, ~2^-48) when the fp32 sign is
//      not certain (R18: the ReLU mask is an integer decision, taken at
//      fp64-level accuracy on both sides, so the GPU and the fp64 oracle agree
//      on it except within ~1e-13 of a kink).
//   2. mlp_logits_kernel  grid (r, b): h = relu(a1) (fp32), logits, max-subtracted
//      softmax, e = p - onehot   ->  E
//   2b. mlp_head_kernel   grid (r, 16): dW2 = e^T h / b, db2, da1 = (W2^T e) * [a1 > 0].
//   3. mlp_w1_kernel      grid (r, hidden/16, in_dim/64): dW1 = da1^T X / b, db1.
// fp32 FFMA elsewhere; no TF32.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "sma_bulk.cuh"
#include "sma_dot2.cuh"
#include "sma_pdl.cuh"
#include "sma_softmax.cuh"
#include "sma_internal.h"

namespace sma {
namespace {
constexpr int kUnits = 16;       // hidden units per CTA of the dW1 kernel
constexpr int kHidUnits = 4;     // hidden units per CTA of the forward kernel (fallback)
constexpr int kMaxHidUnits = 16;
constexpr int kRowBatch = 8;     // batch rows per warp of the forward kernel (independent chains)
constexpr int kMlpThreads = 256;
constexpr int kHeadSplit = 16;   // CTAs per learner of the head-gradient kernel

__device__ __forceinline__ int batch_row(const int32_t* perm, int64_t pos0, int j, int b, int t) {
  return perm[pos0 + (int64_t)j * b + t];
}

using dot2::f2;
using dot2::dot2_step;
using dot2::f2_add;

__global__ void __launch_bounds__(kMlpThreads, 1) mlp_hidden_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ perm, int64_t pos0, int b, int in_dim,
    int hidden, const float* __restrict__ Wall, int64_t ld, int j0, float2* __restrict__ A1,
    int hid_units) {
  // R18: the pre-activation that decides the ReLU mask is accumulated in
  // double-float (hi + lo), accurate to ~2^-48 like the oracle's fp64.
  extern __shared__ __align__(16) float sm[];
  float* xs = sm;                                // [b][in_dim]
  float* ws = xs + (int64_t)b * in_dim;          // [hid_units][in_dim]
  const int slot = blockIdx.x, k0 = blockIdx.y * hid_units;
  const int nu = min(hid_units, hidden - k0);
  const float* W1 = Wall + (int64_t)slot * ld;
  const float* b1 = W1 + (int64_t)hidden * in_dim;
  __shared__ int rows[64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x < b) rows[threadIdx.x] = batch_row(perm, pos0, j0 + slot, b, threadIdx.x);
  __syncthreads();
  // the batch rows (X, perm: never written by a kernel) while the previous
  // kernel drains (PDL), then -- after the wait -- this CTA's W1 rows (the replica)
  const bool used = bulk::stage_rows_span(xs, X, rows, b, in_dim, in_dim, 0, nullptr, nullptr, 0,
                                          &bar, 0, true);
  pdl::wait_and_release();
  bulk::stage_rows_span(nullptr, X, rows, 0, in_dim, in_dim, 0, ws, W1 + (int64_t)k0 * in_dim,
                        nu * in_dim, &bar, used ? 1u : 0u, !used);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // Each warp takes one hidden unit u and a group of kRowBatch batch rows: the W1
  // row chunk is loaded once per lane iteration and reused for every row, and
  // the rows' accumulators are independent FMA chains (the per-row arithmetic,
  // lane-strided over f with 4 components per float4, is unchanged).
  const int ngrp = (b + kRowBatch - 1) / kRowBatch;
  for (int pr = warp; pr < nu * ngrp; pr += nw) {
    const int u = pr % nu, t0 = (pr / nu) * kRowBatch;
    const int nt = min(kRowBatch, b - t0);
    const float* w = ws + (int64_t)u * in_dim;
    // fast path: plain fp32 dot and sum_f |w x|; the fp32 result's sign is
    // certain unless |a| <= 2^-12 sum|w x| (> 3x the n u sum|w x| error bound
    // for n <= 1024), and only then (rare; warp-uniform) is the dot redone
    // with the Dot2 accumulation.
    float sv[kRowBatch], sa[kRowBatch];
#pragma unroll
    for (int i = 0; i < kRowBatch; ++i) sv[i] = sa[i] = 0.f;
    if ((in_dim & 3) == 0) {  // 128-bit shared-memory loads: half the instructions
      const float4* w4 = reinterpret_cast<const float4*>(w);
      for (int f = lane; f < (in_dim >> 2); f += 32) {
        const float4 p = w4[f];
#pragma unroll
        for (int i = 0; i < kRowBatch; ++i) {
          if (i < nt) {
            const float4 q = reinterpret_cast<const float4*>(xs + (int64_t)(t0 + i) * in_dim)[f];
            sv[i] = __fmaf_rn(p.x, q.x, sv[i]);
            sv[i] = __fmaf_rn(p.y, q.y, sv[i]);
            sv[i] = __fmaf_rn(p.z, q.z, sv[i]);
            sv[i] = __fmaf_rn(p.w, q.w, sv[i]);
            sa[i] = __fmaf_rn(fabsf(p.x), fabsf(q.x), sa[i]);
            sa[i] = __fmaf_rn(fabsf(p.y), fabsf(q.y), sa[i]);
            sa[i] = __fmaf_rn(fabsf(p.z), fabsf(q.z), sa[i]);
            sa[i] = __fmaf_rn(fabsf(p.w), fabsf(q.w), sa[i]);
          }
        }
      }
    } else {
      for (int f = lane; f < in_dim; f += 32) {
#pragma unroll
        for (int i = 0; i < kRowBatch; ++i) {
          if (i < nt) {
            const float q = xs[(int64_t)(t0 + i) * in_dim + f];
            sv[i] = __fmaf_rn(w[f], q, sv[i]);
            sa[i] = __fmaf_rn(fabsf(w[f]), fabsf(q), sa[i]);
          }
        }
      }
    }
    const float bias = b1[k0 + u];
#pragma unroll
    for (int i = 0; i < kRowBatch; ++i) {
      if (i >= nt) break;
      float v = sv[i], va = sa[i];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
        va = __fadd_rn(va, __shfl_xor_sync(0xffffffffu, va, off));
      }
      const int t = t0 + i;
      const float* x = xs + (int64_t)t * in_dim;
      f2 acc = {__fadd_rn(v, bias), 0.f};
      const float bound = ldexpf(__fadd_rn(va, fabsf(bias)), -12);
      if (fabsf(acc.hi) <= bound) {  // near a ReLU kink: decide at ~2^-48 (warp-uniform)
        acc = f2{0.f, 0.f};
        if ((in_dim & 3) == 0) {
          const float4* w4 = reinterpret_cast<const float4*>(w);
          const float4* x4 = reinterpret_cast<const float4*>(x);
          for (int f = lane; f < (in_dim >> 2); f += 32) {
            const float4 a = w4[f], c = x4[f];
            dot2_step(acc, a.x, c.x);
            dot2_step(acc, a.y, c.y);
            dot2_step(acc, a.z, c.z);
            dot2_step(acc, a.w, c.w);
          }
        } else {
          for (int f = lane; f < in_dim; f += 32) dot2_step(acc, w[f], x[f]);
        }
        acc = f2_add(dot2::warp_sum(acc), f2{bias, 0.f});
      }
      if (lane == 0) A1[((int64_t)slot * b + t) * hidden + k0 + u] = make_float2(acc.hi, acc.lo);
    }
  }
}

// grid (r, b): the logits of one (learner, row) -- one warp per class over the
// relu'd hidden row staged in shared memory -- and e = softmax - onehot(y)
// (max-subtracted), written to E [r][b][classes].
__global__ void __launch_bounds__(kMlpThreads) mlp_logits_kernel(
    const int32_t* __restrict__ y, const int32_t* __restrict__ perm, int64_t pos0, int b,
    int in_dim, int hidden, int classes, const float* __restrict__ Wall, int64_t ld, int j0,
    const float2* __restrict__ A1, float* __restrict__ E) {
  extern __shared__ __align__(16) float sm[];
  float* hrow = sm;                 // [hidden]
  float* w2s = sm + hidden;         // [classes][hidden] + b2 [classes]
  __shared__ float lg[32];
  const int slot = blockIdx.x, t = blockIdx.y;
  const float* W2 = Wall + (int64_t)slot * ld + (int64_t)hidden * in_dim + hidden;
  const float2* a1 = A1 + ((int64_t)slot * b + t) * hidden;
  __shared__ int yt_sm;
  if (threadIdx.x == 0) yt_sm = y[batch_row(perm, pos0, j0 + slot, b, t)];  // early: off the tail
  // W2 and b2 before the wait: the replicas were last written by the previous
  // round's replica kernel, which the layer-1 kernel's own wait (before it
  // released this grid) already saw complete; only A1 is the predecessor's output
  for (int q = threadIdx.x; q < classes * hidden + classes; q += blockDim.x) w2s[q] = __ldg(W2 + q);
  pdl::wait_and_release();
  for (int k = threadIdx.x; k < hidden; k += blockDim.x) {  // relu of the double-float a1
    const float2 v = a1[k];
    hrow[k] = dot2::positive(v.x, v.y) ? __fadd_rn(v.x, v.y) : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = warp; c < classes; c += nw) {
    float s = 0.f;
    for (int k = lane; k < hidden; k += 32) s = __fmaf_rn(w2s[c * hidden + k], hrow[k], s);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
    if (lane == 0) lg[c] = __fadd_rn(s, w2s[classes * hidden + c]);
  }
  __syncthreads();
  if (threadIdx.x < 32)  // max-subtracted softmax, e = p - onehot(y_t)
    warp_softmax_grad(lg, classes, yt_sm, E + ((int64_t)slot * b + t) * classes);
}

// grid (r, kHeadSplit): slices of dW2 = e^T h / b, db2, and
// da1 = (W2^T e) [a1 > 0] (written to DA for the dW1 kernel).
__global__ void __launch_bounds__(kMlpThreads) mlp_head_kernel(
    int b, int in_dim, int hidden, int classes, const float* __restrict__ Wall, int64_t ld,
    const float2* __restrict__ A1, const float* __restrict__ E, float* __restrict__ DA,
    float* __restrict__ Gall) {
  pdl::wait_and_release();
  extern __shared__ __align__(16) float sm[];
  float* hs = sm;                              // [b][hidden]
  float* w2s = hs + b * hidden;                // [classes][hidden]
  float* e = w2s + classes * hidden;           // [b][classes]
  const int slot = blockIdx.x;
  const float* W2 = Wall + (int64_t)slot * ld + (int64_t)hidden * in_dim + hidden;
  float* G = Gall + (int64_t)slot * ld;
  float* gW2 = G + (int64_t)hidden * in_dim + hidden;
  float* gb2 = gW2 + (int64_t)classes * hidden;
  float2* a1 = reinterpret_cast<float2*>(e + ((b * classes + 3) & ~3));  // staged copy of A1
  __shared__ int zero_row;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) zero_row = 0;
  for (int q = threadIdx.x; q < b * classes; q += blockDim.x) e[q] = E[(int64_t)slot * b * classes + q];
  __syncthreads();
  bulk::stage_rows_span(reinterpret_cast<float*>(a1),
                        reinterpret_cast<const float*>(A1 + (int64_t)slot * b * hidden), &zero_row,
                        1, 2 * b * hidden, 0, 0, w2s, W2, classes * hidden, &bar, 0, true);
  for (int q = threadIdx.x; q < b * hidden; q += blockDim.x) {
    const float2 v = a1[q];
    hs[q] = dot2::positive(v.x, v.y) ? __fadd_rn(v.x, v.y) : 0.f;
  }
  __syncthreads();
  const float fb = (float)b;
  const int nsl = gridDim.y, sl = blockIdx.y;
  for (int q = sl * blockDim.x + threadIdx.x; q < classes * hidden; q += nsl * blockDim.x) {
    const int c = q / hidden, k = q - c * hidden;   // dW2 = e^T h / b
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fmaf_rn(e[t * classes + c], hs[t * hidden + k], s);
    gW2[q] = __fdiv_rn(s, fb);
  }
  if (sl == 0 && threadIdx.x < classes) {
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, e[t * classes + threadIdx.x]);
    gb2[threadIdx.x] = __fdiv_rn(s, fb);
  }
  for (int q = sl * blockDim.x + threadIdx.x; q < b * hidden; q += nsl * blockDim.x) {  // da1
    const int t = q / hidden, k = q - t * hidden;
    float s = 0.f;
    for (int c = 0; c < classes; ++c) s = __fmaf_rn(w2s[c * hidden + k], e[t * classes + c], s);
    const float2 v = a1[q];
    DA[(int64_t)slot * b * hidden + q] = dot2::positive(v.x, v.y) ? s : 0.f;
  }
}

// grid (r, hidden/kUnits, in_dim/kFeat): one (unit block x feature block) tile
// of dW1 = da1^T X / b per CTA, staging only its slices of da1 and X.
constexpr int kFeat = 64;
__global__ void __launch_bounds__(kMlpThreads) mlp_w1_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ perm, int64_t pos0, int b, int in_dim,
    int hidden, int j0, int64_t ld, const float* __restrict__ DA, float* __restrict__ Gall) {
  extern __shared__ __align__(16) float sm[];
  float* xs = sm;                       // [b][kFeat]
  float* da = xs + b * kFeat;           // [b][kUnits]
  __shared__ int rows[64];
  const int slot = blockIdx.x, k0 = blockIdx.y * kUnits, f0 = blockIdx.z * kFeat;
  const int nf = min(kFeat, in_dim - f0);
  float* G = Gall + (int64_t)slot * ld;
  const int nu = min(kUnits, hidden - k0);
  if (threadIdx.x < b) rows[threadIdx.x] = batch_row(perm, pos0, j0 + slot, b, threadIdx.x);
  __syncthreads();
  // X[rows][f0, f0 + nf) -> xs [b][nf] (one 16-byte load per thread: 16 short
  // rows as TMA bulk copies from one thread were slower) while the head kernel
  // drains (PDL); then da1[t][k0, k0 + nu) -> da [b][nu], its output
  bulk::load_tile(xs, X, rows, b, nf, in_dim, f0);
  pdl::wait_and_release();
  for (int q = threadIdx.x; q < b * nu; q += blockDim.x) {
    const int t = q / nu, u = q - t * nu;
    da[q] = DA[((int64_t)slot * b + t) * hidden + k0 + u];
  }
  __syncthreads();
  const float fb = (float)b;
  // / b as * 2^-log2(b) when b is a power of two: both are the correctly
  // rounded s / b, so the result is bitwise the same and the IEEE division's
  // instruction sequence (the kernel is issue-bound) is gone
  const bool pow2 = (b & (b - 1)) == 0;
  const float inv_b = 1.f / fb;
  if ((in_dim & 3) == 0 && (ld & 3) == 0) {
    // 4 adjacent features per thread: one da load and one 128-bit x load per
    // 4 FMAs, one 128-bit store; per output the same ascending-t FMA chain
    const int nf4 = nf >> 2;
    for (int q = threadIdx.x; q < nu * nf4; q += blockDim.x) {  // dW1 = da^T x / b
      const int u = q / nf4, f = (q - u * nf4) << 2;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int t = 0; t < b; ++t) {
        const float a = da[t * nu + u];
        const float4 x = *reinterpret_cast<const float4*>(xs + t * nf + f);
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
      *reinterpret_cast<float4*>(G + (int64_t)(k0 + u) * in_dim + f0 + f) = s;
    }
  } else {
    for (int q = threadIdx.x; q < nu * nf; q += blockDim.x) {  // dW1 = da^T x / b
      const int u = q / nf, f = q - u * nf;
      float s = 0.f;
      for (int t = 0; t < b; ++t) s = __fmaf_rn(da[t * nu + u], xs[t * nf + f], s);
      G[(int64_t)(k0 + u) * in_dim + f0 + f] = pow2 ? __fmul_rn(s, inv_b) : __fdiv_rn(s, fb);
    }
  }
  if (blockIdx.z == 0 && threadIdx.x < nu) {
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, da[t * nu + threadIdx.x]);
    G[(int64_t)hidden * in_dim + k0 + threadIdx.x] = __fdiv_rn(s, fb);
  }
}
}  // namespace

cudaError_t launch_mlp_grad(const float* X, const int32_t* y, const int32_t* perm, int64_t pos0,
                            int b, int in_dim, int hidden, int classes, const float* W, int64_t ld,
                            int r, int j0, float2* A1, float* E, float* DA, float* G,
                            cudaStream_t s) {
  if (classes > 32) return cudaErrorInvalidValue;
  // Hidden units per CTA of the SIMT layer-1 kernel: the fewest (1, 2, 4, 8, 16)
  // whose grid r x ceil(hidden / u) still fits one wave at the kernel's occupancy.
  // Measured (profiles/r01_mlp_hid_units.txt, MLP rounds/s, SIMT): k = 4 best at
  // u = 4 (256 CTAs; 39.0k vs 31.6k at 2, 32.8k at 8), k = 8 at u = 8 (256 CTAs;
  // 28.8k vs 27.2k at 4): more CTAs than one wave re-stage the batch rows in a
  // second wave, fewer leave the per-CTA chain longer. SMA_MLP_HID_UNITS forces u.
  static const int env_units = [] {
    const char* v = getenv("SMA_MLP_HID_UNITS");
    const int u = v ? atoi(v) : 0;
    return u >= 1 && u <= kMaxHidUnits ? u : 0;
  }();
  int hid_units = env_units;
  bool simt_fills = false;
  if (!hid_units) {
    struct UnitsCache {
      int dev = -1, r = 0, b = 0, in_dim = 0, hidden = 0, units = kHidUnits;
      bool fills = false;  // the grid fills >= 85 % of one wave
    };
    thread_local UnitsCache uc;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (uc.dev != dev || uc.r != r || uc.b != b || uc.in_dim != in_dim || uc.hidden != hidden) {
      int sms = 0;
      if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return e;
      int units = kMaxHidUnits;
      bool fills = false;
      for (int u = 1; u <= kMaxHidUnits; u *= 2) {
        const size_t smu = sizeof(float) * ((size_t)b * in_dim + (size_t)u * in_dim);
        if (ensure_dyn_smem(reinterpret_cast<const void*>(mlp_hidden_kernel), (int)smu) != cudaSuccess)
          break;
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mlp_hidden_kernel, kMlpThreads, smu) !=
            cudaSuccess)
          break;
        const int64_t ctas = (int64_t)r * ((hidden + u - 1) / u), slots = (int64_t)occ * sms;
        if (ctas <= slots) {
          units = u;
          fills = ctas * 100 >= slots * 85;
          break;
        }
      }
      uc = UnitsCache{dev, r, b, in_dim, hidden, units, fills};
    }
    hid_units = uc.units;
    simt_fills = uc.fills;
  }
  const size_t sm1 = sizeof(float) * ((size_t)b * in_dim + (size_t)hid_units * in_dim);
  const size_t smL = sizeof(float) * ((size_t)hidden + (size_t)classes * hidden + classes);
  const size_t sm2 = sizeof(float) * ((size_t)b * hidden + (size_t)classes * hidden +
                                      (size_t)b * classes) +
                     16 + sizeof(float2) * (size_t)b * hidden;
  const size_t sm3 = sizeof(float) * ((size_t)b * kFeat + (size_t)b * kUnits);
  cudaError_t e;
  if ((e = ensure_dyn_smem(reinterpret_cast<const void*>(mlp_hidden_kernel), (int)sm1)) != cudaSuccess)
    return e;
  if ((e = ensure_dyn_smem(reinterpret_cast<const void*>(mlp_logits_kernel), (int)smL)) != cudaSuccess)
    return e;
  if ((e = ensure_dyn_smem(reinterpret_cast<const void*>(mlp_head_kernel), (int)sm2)) != cudaSuccess)
    return e;
  const dim3 g1(r, (hidden + hid_units - 1) / hid_units), gL(r, b), g2(r, kHeadSplit),
      g3(r, (hidden + kUnits - 1) / kUnits, (in_dim + kFeat - 1) / kFeat);
  // layer 1 on the tensor cores (sma_learner_mlp_tc.cu) where the shape allows,
  // else the SIMT kernel; both write the same A1 contract
  // (default policy: a SIMT grid that fills one wave beats the tensor cores even
  // at r >= 12 -- k = 16: 18.4k vs 16.8k rounds/s, profiles/r01_mlp_hid_units2.txt)
  e = (mlp_tc_policy() < 0 && simt_fills)
          ? cudaErrorNotSupported
          : launch_mlp_hidden_tc(X, perm, pos0, b, in_dim, hidden, W, ld, r, j0, A1, s);
  if (e == cudaErrorNotSupported)
    e = pdl::launch(mlp_hidden_kernel, g1, dim3(kMlpThreads), sm1, s, 1, X, perm, pos0, b, in_dim,
                    hidden, W, ld, j0, A1, hid_units);
  if (e != cudaSuccess) return e;
  if ((e = pdl::launch(mlp_logits_kernel, gL, dim3(kMlpThreads), smL, s, 1, y, perm, pos0, b, in_dim,
                       hidden, classes, W, ld, j0, (const float2*)A1, E)) != cudaSuccess)
    return e;
  if ((e = pdl::launch(mlp_head_kernel, g2, dim3(kMlpThreads), sm2, s, 1, b, in_dim, hidden, classes,
                       W, ld, (const float2*)A1, (const float*)E, DA, G)) != cudaSuccess)
    return e;
  e = launch_mlp_w1_tc(X, perm, pos0, b, in_dim, hidden, j0, ld, r, DA, G, s);
  if (e == cudaErrorNotSupported)
    e = pdl::launch(mlp_w1_kernel, g3, dim3(kMlpThreads), sm3, s, 1, X, perm, pos0, b, in_dim, hidden,
                    j0, ld, (const float*)DA, G);
  return e;
}

}  // namespace sma
