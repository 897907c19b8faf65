// sma_dot2.cuh -- double-float dot-product accumulation for the MLP learner's
// ReLU-mask decision (reading R18): error-free transformations (Knuth TwoSum,
// FMA TwoProd) give the Ogita-Rump-Oishi "Dot2" accumulation, as accurate as a
// dot product computed in twice the working precision (~2^-48), with fp32
// instructions only.  Shared by the SIMT and the tensor-core layer-1 kernels.
#pragma once
#include <cuda_runtime.h>

namespace sma {
namespace dot2 {

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
// The ReLU decision [a > 0] on a double-float a = hi + lo.  hi is NOT the
// rounded value of the pair: neither dot2_step nor f2_add renormalises, so after
// cancellation |lo| can exceed |hi| (lo collects every rounding error of the
// running sum) and sign(hi) can differ from sign(hi + lo).  fl(hi + lo) has the
// sign of hi + lo exactly (round-to-nearest keeps the sign and returns 0 only
// for an exact 0), so the decision is taken on it.  (Deciding on hi first
// flipped a mask at a1 = +1.3e-8 in the k = 32 MLP parity test.)
__device__ __forceinline__ bool positive(float hi, float lo) { return __fadd_rn(hi, lo) > 0.f; }

// Warp-wide sum of per-lane double-float partials (every lane gets the total).
__device__ __forceinline__ f2 warp_sum(f2 acc) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    f2 o;
    o.hi = __shfl_xor_sync(0xffffffffu, acc.hi, off);
    o.lo = __shfl_xor_sync(0xffffffffu, acc.lo, off);
    acc = f2_add(acc, o);
  }
  return acc;
}

}  // namespace dot2
}  // namespace sma
