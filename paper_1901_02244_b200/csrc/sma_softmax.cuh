// sma_softmax.cuh -- the softmax cross-entropy gradient of one batch row by one
// warp, shared by the softmax-regression and MLP learners (a2').
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace sma {

// e_c = exp(l_c - max) / sum_c' exp(l_c' - max) - [c == y]   (R16: max-subtracted),
// lane c = class c (classes <= 32); the max and the sum are xor-butterfly
// reductions, so every lane holds the same bits.  All 32 lanes must call it.
__device__ __forceinline__ void warp_softmax_grad(const float* lg, int classes, int yt, float* e) {
  const int lane = threadIdx.x & 31;
  const float v = lane < classes ? lg[lane] : -INFINITY;
  float mx = v;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  const float ex = lane < classes ? expf(__fsub_rn(v, mx)) : 0.f;
  float den = ex;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) den = __fadd_rn(den, __shfl_xor_sync(0xffffffffu, den, off));
  if (lane < classes) e[lane] = __fsub_rn(__fdiv_rn(ex, den), lane == yt ? 1.f : 0.f);
}

// The same for TWO rows per warp when classes <= 16: lanes 0-15 take row
// lg0 / e0, lanes 16-31 row lg1 / e1 (valid1 = false: the second half computes
// but stores nothing).  Bitwise equal to warp_softmax_grad: there the first
// butterfly step (xor 16) only adds the -inf / 0 of lanes >= classes, after
// which both reduce over the same lanes in the same order.
__device__ __forceinline__ void halfwarp_softmax_grad(const float* lg0, const float* lg1, int classes,
                                                      int y0, int y1, bool valid1, float* e0,
                                                      float* e1) {
  const int lane = threadIdx.x & 31, c = lane & 15;
  const bool hi = lane >= 16;
  const float* lg = hi ? lg1 : lg0;
  const int yt = hi ? y1 : y0;
  const float v = c < classes ? lg[c] : -INFINITY;
  float mx = v;
#pragma unroll
  for (int off = 8; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  const float ex = c < classes ? expf(__fsub_rn(v, mx)) : 0.f;
  float den = ex;
#pragma unroll
  for (int off = 8; off >= 1; off >>= 1) den = __fadd_rn(den, __shfl_xor_sync(0xffffffffu, den, off));
  if (c < classes && (!hi || valid1)) (hi ? e1 : e0)[c] = __fsub_rn(__fdiv_rn(ex, den), c == yt ? 1.f : 0.f);
}

}  // namespace sma
