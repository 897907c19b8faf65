// sma_learner_mlp.cu -- NEXT-2: the built-in MLP learner (in_dim-hidden-classes,
// ReLU; "MLP (784-256-10)"), batch-mean gradient (Eq. 2, PAPER.md:
// 228-232) by back-propagation, for all r local replicas.
//
// Three small kernels per round (the learner is latency-bound at b = 16):
//   1. mlp_hidden_kernel  grid (r, hidden/8): gather the batch rows into shared
//      memory; pre-activations a1 = W1 x + b1 accumulated in double-float
//      (Dot2, ~2^-48; R18: the ReLU mask is an integer decision, taken at
//      fp64-level accuracy on both sides, so the GPU and the fp64 oracle agree
//      on it except within ~1e-13 of a kink).
//   2. mlp_head_kernel    grid (r): h = relu(a1) (fp32), logits, max-subtracted
//      softmax, e = p - onehot, dW2 = e^T h / b, db2, da1 = (W2^T e) * [a1 > 0].
//   3. mlp_w1_kernel      grid (r, hidden/16, in_dim/64): dW1 = da1^T X / b, db1.
// fp32 FFMA elsewhere; no TF32.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sma_internal.h"

namespace sma {
namespace {
constexpr int kUnits = 16;       // hidden units per CTA of the dW1 kernel
constexpr int kHidUnits = 8;     // hidden units per CTA of the forward kernel
constexpr int kMlpThreads = 256;
constexpr int kHeadSplit = 8;    // CTAs per learner of the head kernel

__device__ __forceinline__ int batch_row(const int32_t* perm, int64_t pos0, int j, int b, int t) {
  return perm[pos0 + (int64_t)j * b + t];
}

// Stage the b batch rows of X into xs[t][in_dim] (128-bit loads when aligned).
__device__ __forceinline__ void stage_batch(float* xs, const float* __restrict__ X,
                                            const int32_t* __restrict__ perm, int64_t pos0, int j,
                                            int b, int in_dim) {
  if ((in_dim & 3) == 0 && ((reinterpret_cast<uintptr_t>(X) & 15) == 0)) {
    const int v = in_dim >> 2;
    for (int q = threadIdx.x; q < b * v; q += blockDim.x) {
      const int t = q / v, f4 = q - t * v;
      reinterpret_cast<float4*>(xs)[q] = __ldg(
          reinterpret_cast<const float4*>(X + (int64_t)batch_row(perm, pos0, j, b, t) * in_dim) + f4);
    }
  } else {
    for (int q = threadIdx.x; q < b * in_dim; q += blockDim.x) {
      const int t = q / in_dim, f = q - t * in_dim;
      xs[q] = X[(int64_t)batch_row(perm, pos0, j, b, t) * in_dim + f];
    }
  }
}
__device__ __forceinline__ void stage_span(float* dst, const float* __restrict__ src, int n) {
  if ((n & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
    for (int q = threadIdx.x; q < (n >> 2); q += blockDim.x)
      reinterpret_cast<float4*>(dst)[q] = __ldg(reinterpret_cast<const float4*>(src) + q);
  } else {
    for (int q = threadIdx.x; q < n; q += blockDim.x) dst[q] = src[q];
  }
}

// Error-free transformations (Knuth TwoSum, FMA TwoProd): the Ogita-Rump-Oishi
// "Dot2" accumulation gives a dot product as accurate as one computed in twice
// the working precision (~2^-48), with fp32 instructions only (the F2F
// conversions of a plain fp64 accumulation were the bottleneck: profiles/).
struct f2 { float hi, lo; };
__device__ __forceinline__ void two_sum(float a, float b, float& s, float& e) {
  s = __fadd_rn(a, b);
  const float bb = __fsub_rn(s, a);
  e = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
}
__device__ __forceinline__ void dot2_step(f2& acc, float w, float x) {
  const float p = __fmul_rn(w, x);
  const float pe = __fmaf_rn(w, x, -p);        // exact: w*x = p + pe
  float s, e;
  two_sum(acc.hi, p, s, e);
  acc.hi = s;
  acc.lo = __fadd_rn(acc.lo, __fadd_rn(e, pe));
}
__device__ __forceinline__ f2 f2_add(f2 a, f2 b) {
  f2 r;
  float e;
  two_sum(a.hi, b.hi, r.hi, e);
  r.lo = __fadd_rn(__fadd_rn(a.lo, b.lo), e);
  return r;
}

__global__ void __launch_bounds__(kMlpThreads) mlp_hidden_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ perm, int64_t pos0, int b, int in_dim,
    int hidden, const float* __restrict__ Wall, int64_t ld, int j0, float2* __restrict__ A1) {
  // R18: the pre-activation that decides the ReLU mask is accumulated in
  // double-float (hi + lo), accurate to ~2^-48 like the oracle's fp64.
  extern __shared__ __align__(16) float sm[];
  float* xs = sm;                                // [b][in_dim]
  float* ws = xs + (int64_t)b * in_dim;          // [kHidUnits][in_dim]
  const int slot = blockIdx.x, k0 = blockIdx.y * kHidUnits;
  const int nu = min(kHidUnits, hidden - k0);
  const float* W1 = Wall + (int64_t)slot * ld;
  const float* b1 = W1 + (int64_t)hidden * in_dim;
  stage_batch(xs, X, perm, pos0, j0 + slot, b, in_dim);
  stage_span(ws, W1 + (int64_t)k0 * in_dim, nu * in_dim);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int pr = warp; pr < b * nu; pr += nw) {
    const int t = pr / nu, u = pr - t * nu;
    const float* w = ws + (int64_t)u * in_dim;
    const float* x = xs + (int64_t)t * in_dim;
    f2 acc = {0.f, 0.f};
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
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      f2 o;
      o.hi = __shfl_xor_sync(0xffffffffu, acc.hi, off);
      o.lo = __shfl_xor_sync(0xffffffffu, acc.lo, off);
      acc = f2_add(acc, o);
    }
    if (lane == 0) {
      acc = f2_add(acc, f2{b1[k0 + u], 0.f});
      A1[((int64_t)slot * b + t) * hidden + k0 + u] = make_float2(acc.hi, acc.lo);
    }
  }
}

__global__ void __launch_bounds__(kMlpThreads) mlp_head_kernel(
    const int32_t* __restrict__ y, const int32_t* __restrict__ perm, int64_t pos0, int b,
    int in_dim, int hidden, int classes, const float* __restrict__ Wall, int64_t ld, int j0,
    const float2* __restrict__ A1, float* __restrict__ DA, float* __restrict__ Gall) {
  extern __shared__ __align__(16) float sm[];
  float* hs = sm;                              // [b][hidden]
  float* w2s = hs + b * hidden;                // [classes][hidden]
  float* e = w2s + classes * hidden;           // [b][classes]
  const int slot = blockIdx.x;
  const float* W2 = Wall + (int64_t)slot * ld + (int64_t)hidden * in_dim + hidden;
  const float* b2 = W2 + (int64_t)classes * hidden;
  float* G = Gall + (int64_t)slot * ld;
  float* gW2 = G + (int64_t)hidden * in_dim + hidden;
  float* gb2 = gW2 + (int64_t)classes * hidden;
  const float2* a1 = A1 + (int64_t)slot * b * hidden;
  // relu on the double-float pre-activation: positive iff hi > 0, or hi == 0 and lo > 0
  for (int q = threadIdx.x; q < b * hidden; q += blockDim.x) {
    const float2 v = a1[q];
    hs[q] = (v.x > 0.f || (v.x == 0.f && v.y > 0.f)) ? __fadd_rn(v.x, v.y) : 0.f;
  }
  stage_span(w2s, W2, classes * hidden);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int pr = warp; pr < b * classes; pr += nw) {  // logits
    const int t = pr / classes, c = pr - t * classes;
    float s = 0.f;
#pragma unroll 4
    for (int k = lane; k < hidden; k += 32) s = __fmaf_rn(w2s[c * hidden + k], hs[t * hidden + k], s);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
    if (lane == 0) e[pr] = __fadd_rn(s, b2[c]);
  }
  __syncthreads();
  if (threadIdx.x < b) {  // max-subtracted softmax, e = p - onehot(y)
    const int t = threadIdx.x;
    float mx = e[t * classes];
    for (int c = 1; c < classes; ++c) mx = fmaxf(mx, e[t * classes + c]);
    float den = 0.f;
    for (int c = 0; c < classes; ++c) den = __fadd_rn(den, expf(__fsub_rn(e[t * classes + c], mx)));
    const int yt = y[batch_row(perm, pos0, j0 + slot, b, t)];
    for (int c = 0; c < classes; ++c)
      e[t * classes + c] =
          __fsub_rn(__fdiv_rn(expf(__fsub_rn(e[t * classes + c], mx)), den), c == yt ? 1.f : 0.f);
  }
  __syncthreads();
  const float fb = (float)b;
  // every CTA of the learner recomputed the (cheap) logits; each writes its
  // slice blockIdx.y of dW2 and of da1
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
    DA[(int64_t)slot * b * hidden + q] = (v.x > 0.f || (v.x == 0.f && v.y > 0.f)) ? s : 0.f;
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
  if (threadIdx.x < b) rows[threadIdx.x] = batch_row(perm, pos0, j0 + slot, b, threadIdx.x);
  for (int q = threadIdx.x; q < b * kUnits; q += blockDim.x) {
    const int t = q / kUnits, u = q - t * kUnits;
    da[q] = (k0 + u < hidden) ? DA[((int64_t)slot * b + t) * hidden + k0 + u] : 0.f;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < b * kFeat; q += blockDim.x) {
    const int t = q / kFeat, f = q - t * kFeat;
    xs[q] = f < nf ? __ldg(X + (int64_t)rows[t] * in_dim + f0 + f) : 0.f;
  }
  __syncthreads();
  const float fb = (float)b;
  for (int q = threadIdx.x; q < kUnits * kFeat; q += blockDim.x) {  // dW1 = da^T x / b
    const int u = q / kFeat, f = q - u * kFeat;
    if (k0 + u >= hidden || f >= nf) continue;
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fmaf_rn(da[t * kUnits + u], xs[t * kFeat + f], s);
    G[(int64_t)(k0 + u) * in_dim + f0 + f] = __fdiv_rn(s, fb);
  }
  if (blockIdx.z == 0 && threadIdx.x < kUnits && k0 + threadIdx.x < hidden) {
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, da[t * kUnits + threadIdx.x]);
    G[(int64_t)hidden * in_dim + k0 + threadIdx.x] = __fdiv_rn(s, fb);
  }
}
}  // namespace

cudaError_t launch_mlp_grad(const float* X, const int32_t* y, const int32_t* perm, int64_t pos0,
                            int b, int in_dim, int hidden, int classes, const float* W, int64_t ld,
                            int r, int j0, float2* A1, float* DA, float* G, cudaStream_t s) {
  const size_t sm1 = sizeof(float) * ((size_t)b * in_dim + (size_t)kHidUnits * in_dim);
  const size_t sm2 = sizeof(float) * ((size_t)b * hidden + (size_t)classes * hidden +
                                      (size_t)b * classes);
  const size_t sm3 = sizeof(float) * ((size_t)b * kFeat + (size_t)b * kUnits);
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(mlp_hidden_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sm1)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(mlp_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sm2)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(mlp_w1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sm3)) != cudaSuccess)
    return e;
  const dim3 g1(r, (hidden + kHidUnits - 1) / kHidUnits), g2(r, kHeadSplit),
      g3(r, (hidden + kUnits - 1) / kUnits, (in_dim + kFeat - 1) / kFeat);
  mlp_hidden_kernel<<<g1, kMlpThreads, sm1, s>>>(X, perm, pos0, b, in_dim, hidden, W, ld, j0, A1);
  mlp_head_kernel<<<g2, kMlpThreads, sm2, s>>>(y, perm, pos0, b, in_dim, hidden, classes, W, ld, j0,
                                               A1, DA, G);
  mlp_w1_kernel<<<g3, kMlpThreads, sm3, s>>>(X, perm, pos0, b, in_dim, hidden, j0, ld, DA, G);
  return cudaGetLastError();
}

}  // namespace sma
