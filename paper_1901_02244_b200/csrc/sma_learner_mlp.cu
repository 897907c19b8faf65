// sma_learner_mlp.cu -- NEXT-2: the built-in MLP learner (in_dim-hidden-classes,
// ReLU; "MLP (784-256-10)"), batch-mean gradient (Eq. 2, PAPER.md:
// 228-232) by back-propagation, for all r local replicas.
//
// Three small kernels per round (the learner is latency-bound at b = 16):
//   1. mlp_hidden_kernel  grid (r, hidden/16): gather the batch rows into shared
//      memory; pre-activations a1 = W1 x + b1 accumulated in fp64 (R18: the ReLU
//      mask is an integer decision, taken in fp64 on both sides, so the GPU and
//      the fp64 oracle agree on it except within ~1e-15 of a kink).
//   2. mlp_head_kernel    grid (r): h = relu(a1) (fp32), logits, max-subtracted
//      softmax, e = p - onehot, dW2 = e^T h / b, db2, da1 = (W2^T e) * [a1 > 0].
//   3. mlp_w1_kernel      grid (r, hidden/16): dW1 = da1^T X / b, db1.
// fp32 FFMA elsewhere; no TF32.
#include <cuda_runtime.h>
#include <stdint.h>

#include "sma_internal.h"

namespace sma {
namespace {
constexpr int kUnits = 16;       // hidden units per CTA (kernels 1 and 3)
constexpr int kMlpThreads = 256;

__device__ __forceinline__ int batch_row(const int32_t* perm, int64_t pos0, int j, int b, int t) {
  return perm[pos0 + (int64_t)j * b + t];
}

__global__ void __launch_bounds__(kMlpThreads) mlp_hidden_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ perm, int64_t pos0, int b, int in_dim,
    int hidden, const float* __restrict__ Wall, int64_t ld, int j0, double* __restrict__ A1) {
  extern __shared__ float xs[];  // [b][in_dim]
  const int slot = blockIdx.x, k0 = blockIdx.y * kUnits;
  const float* W1 = Wall + (int64_t)slot * ld;
  const float* b1 = W1 + (int64_t)hidden * in_dim;
  for (int q = threadIdx.x; q < b * in_dim; q += blockDim.x) {
    const int t = q / in_dim, f = q - t * in_dim;
    xs[q] = X[(int64_t)batch_row(perm, pos0, j0 + slot, b, t) * in_dim + f];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int pr = warp; pr < b * kUnits; pr += nw) {
    const int t = pr / kUnits, k = k0 + pr % kUnits;
    if (k >= hidden) continue;
    double s = 0.0;
    for (int f = lane; f < in_dim; f += 32)
      s = fma((double)W1[(int64_t)k * in_dim + f], (double)xs[t * in_dim + f], s);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) A1[((int64_t)slot * b + t) * hidden + k] = s + (double)b1[k];
  }
}

__global__ void __launch_bounds__(kMlpThreads) mlp_head_kernel(
    const int32_t* __restrict__ y, const int32_t* __restrict__ perm, int64_t pos0, int b,
    int in_dim, int hidden, int classes, const float* __restrict__ Wall, int64_t ld, int j0,
    const double* __restrict__ A1, float* __restrict__ DA, float* __restrict__ Gall) {
  extern __shared__ float sm[];
  float* hs = sm;                              // [b][hidden]
  float* e = hs + b * hidden;                  // [b][classes]
  const int slot = blockIdx.x;
  const float* W2 = Wall + (int64_t)slot * ld + (int64_t)hidden * in_dim + hidden;
  const float* b2 = W2 + (int64_t)classes * hidden;
  float* G = Gall + (int64_t)slot * ld;
  float* gW2 = G + (int64_t)hidden * in_dim + hidden;
  float* gb2 = gW2 + (int64_t)classes * hidden;
  const double* a1 = A1 + (int64_t)slot * b * hidden;
  for (int q = threadIdx.x; q < b * hidden; q += blockDim.x) hs[q] = a1[q] > 0.0 ? (float)a1[q] : 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int pr = warp; pr < b * classes; pr += nw) {  // logits
    const int t = pr / classes, c = pr - t * classes;
    float s = 0.f;
    for (int k = lane; k < hidden; k += 32) s = __fmaf_rn(W2[(int64_t)c * hidden + k], hs[t * hidden + k], s);
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
  for (int q = threadIdx.x; q < classes * hidden; q += blockDim.x) {  // dW2 = e^T h / b
    const int c = q / hidden, k = q - c * hidden;
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fmaf_rn(e[t * classes + c], hs[t * hidden + k], s);
    gW2[q] = __fdiv_rn(s, fb);
  }
  if (threadIdx.x < classes) {
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, e[t * classes + threadIdx.x]);
    gb2[threadIdx.x] = __fdiv_rn(s, fb);
  }
  for (int q = threadIdx.x; q < b * hidden; q += blockDim.x) {  // da1 = (W2^T e) [a1 > 0]
    const int t = q / hidden, k = q - t * hidden;
    float s = 0.f;
    for (int c = 0; c < classes; ++c) s = __fmaf_rn(W2[(int64_t)c * hidden + k], e[t * classes + c], s);
    DA[(int64_t)slot * b * hidden + q] = a1[q] > 0.0 ? s : 0.f;
  }
}

__global__ void __launch_bounds__(kMlpThreads) mlp_w1_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ perm, int64_t pos0, int b, int in_dim,
    int hidden, int j0, int64_t ld, const float* __restrict__ DA, float* __restrict__ Gall) {
  extern __shared__ float sm[];
  float* xs = sm;                       // [b][in_dim]
  float* da = xs + b * in_dim;          // [b][kUnits]
  const int slot = blockIdx.x, k0 = blockIdx.y * kUnits;
  float* G = Gall + (int64_t)slot * ld;
  for (int q = threadIdx.x; q < b * in_dim; q += blockDim.x) {
    const int t = q / in_dim, f = q - t * in_dim;
    xs[q] = X[(int64_t)batch_row(perm, pos0, j0 + slot, b, t) * in_dim + f];
  }
  for (int q = threadIdx.x; q < b * kUnits; q += blockDim.x) {
    const int t = q / kUnits, u = q - t * kUnits;
    da[q] = (k0 + u < hidden) ? DA[((int64_t)slot * b + t) * hidden + k0 + u] : 0.f;
  }
  __syncthreads();
  const float fb = (float)b;
  for (int q = threadIdx.x; q < kUnits * in_dim; q += blockDim.x) {  // dW1 = da^T x / b
    const int u = q / in_dim, f = q - u * in_dim;
    if (k0 + u >= hidden) continue;
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fmaf_rn(da[t * kUnits + u], xs[t * in_dim + f], s);
    G[(int64_t)(k0 + u) * in_dim + f] = __fdiv_rn(s, fb);
  }
  if (threadIdx.x < kUnits && k0 + threadIdx.x < hidden) {
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, da[t * kUnits + threadIdx.x]);
    G[(int64_t)hidden * in_dim + k0 + threadIdx.x] = __fdiv_rn(s, fb);
  }
}
}  // namespace

cudaError_t launch_mlp_grad(const float* X, const int32_t* y, const int32_t* perm, int64_t pos0,
                            int b, int in_dim, int hidden, int classes, const float* W, int64_t ld,
                            int r, int j0, double* A1, float* DA, float* G, cudaStream_t s) {
  const size_t sm1 = sizeof(float) * (size_t)b * in_dim;
  const size_t sm2 = sizeof(float) * ((size_t)b * hidden + (size_t)b * classes);
  const size_t sm3 = sizeof(float) * ((size_t)b * in_dim + (size_t)b * kUnits);
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
  const dim3 g13(r, (hidden + kUnits - 1) / kUnits);
  mlp_hidden_kernel<<<g13, kMlpThreads, sm1, s>>>(X, perm, pos0, b, in_dim, hidden, W, ld, j0, A1);
  mlp_head_kernel<<<r, kMlpThreads, sm2, s>>>(y, perm, pos0, b, in_dim, hidden, classes, W, ld, j0,
                                              A1, DA, G);
  mlp_w1_kernel<<<g13, kMlpThreads, sm3, s>>>(X, perm, pos0, b, in_dim, hidden, j0, ld, DA, G);
  return cudaGetLastError();
}

}  // namespace sma
