// sma_kernels.cu -- sm_100a kernels of the SMA hot path (arXiv 1901.02244, Alg. 1).
//
// All kernels are HBM-bandwidth-bound streaming kernels (about 5 flop per 12
// bytes), so they are written for the memory system, not the tensor cores:
// 128-bit coalesced accesses, L1 bypass for single-use streams, a persistent
// grid of (#SMs x resident CTAs), and several independent 16-byte loads in
// flight per thread.  Each floating-point operation is written with an
// explicit-rounding intrinsic so the fp32 operation sequence is fixed (and
// documented in DESIGN.md "Arithmetic") rather than left to FMA contraction.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "sma_bulk.cuh"
#include "sma_pdl.cuh"
#include "sma_softmax.cuh"
#include "sma_internal.h"

namespace sma {
namespace {

// ---------------------------------------------------------------- memory ops
// Single-use streams: do not allocate in L1.  `.nc` only for data that is
// read-only for the whole kernel (gradients, z); replicas are read then
// written by the same thread, so they use the coherent path.
__device__ __forceinline__ float4 ld_ro(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_rw(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st4(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
// Cache-policy variants of the streaming ops (experiment knob SMA_LDG_POLICY,
// profiles/r01_ldg_policy.jsonl): 1 = evict-first streaming (.cs) loads and
// stores of the replica/gradient streams, 2 = 256-byte L2 prefetch on loads.
template <int POL>
__device__ __forceinline__ float4 ld_rw_p(const float* p) {
  float4 v;
  if (POL == 1)
    asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else if (POL == 2)
    asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
template <int POL>
__device__ __forceinline__ float4 ld_ro_p(const float* p) {
  float4 v;
  if (POL == 1)
    asm volatile("ld.global.cs.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else if (POL == 2)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}
template <int POL>
__device__ __forceinline__ void st4_p(float* p, float4 v) {
  if (POL == 1)
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
  else
    asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// Gradient chunk that straddles (or lies beyond) d: scalar loads, zeros past d.
__device__ __forceinline__ float4 ld_tail(const float* g, int64_t p0, int64_t d) {
  float4 v;
  v.x = (p0 + 0 < d) ? g[p0 + 0] : 0.f;
  v.y = (p0 + 1 < d) ? g[p0 + 1] : 0.f;
  v.z = (p0 + 2 < d) ? g[p0 + 2] : 0.f;
  v.w = (p0 + 3 < d) ? g[p0 + 3] : 0.f;
  return v;
}

__device__ __forceinline__ bool finite4(float4 v) {
  return isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
}

// ------------------------------------------------------------- arithmetic
// Alg. 1 line 9:  c = alpha (w - z)
// Alg. 1 line 10: w' = (w - gamma g) - c        (w - gamma g rounded once, FMA)
struct StepOut { float wn, c; };
__device__ __forceinline__ StepOut sma_elem(float w, float g, float z, float alpha, float gamma) {
  const float c = __fmul_rn(alpha, __fsub_rn(w, z));
  const float wn = __fsub_rn(__fmaf_rn(-gamma, g, w), c);
  return {wn, c};
}
// Alg. 1 line 13: z' = (z + sum c) + mu (z - z_prev)
__device__ __forceinline__ float central_elem(float z, float csum, float zp, float mu) {
  return __fadd_rn(__fadd_rn(z, csum), __fmul_rn(mu, __fsub_rn(z, zp)));
}

template <int MODE>
__device__ __forceinline__ void replica_update4(float4& w, const float4 g, const float4 z,
                                               float4& acc, float4& c4, float alpha, float gamma) {
  if (MODE == kLocal) {  // no correction, no central model (R17): w' = w - gamma g
    w.x = __fmaf_rn(-gamma, g.x, w.x);
    w.y = __fmaf_rn(-gamma, g.y, w.y);
    w.z = __fmaf_rn(-gamma, g.z, w.z);
    w.w = __fmaf_rn(-gamma, g.w, w.w);
    return;
  }
  StepOut o;
  o = sma_elem(w.x, g.x, z.x, alpha, gamma); w.x = o.wn; c4.x = o.c;
  o = sma_elem(w.y, g.y, z.y, alpha, gamma); w.y = o.wn; c4.y = o.c;
  o = sma_elem(w.z, g.z, z.z, alpha, gamma); w.z = o.wn; c4.z = o.c;
  o = sma_elem(w.w, g.w, z.w, alpha, gamma); w.w = o.wn; c4.w = o.c;
  if (MODE == kPartialB || MODE == kHierB0) {  // Q accumulates (w' - z), DESIGN.md "Mode B"
    acc.x = __fadd_rn(acc.x, __fsub_rn(w.x, z.x));
    acc.y = __fadd_rn(acc.y, __fsub_rn(w.y, z.y));
    acc.z = __fadd_rn(acc.z, __fsub_rn(w.z, z.z));
    acc.w = __fadd_rn(acc.w, __fsub_rn(w.w, z.w));
  } else {                  // sum_j c_j in ascending local j (R7)
    acc.x = __fadd_rn(acc.x, c4.x);
    acc.y = __fadd_rn(acc.y, c4.y);
    acc.z = __fadd_rn(acc.z, c4.z);
    acc.w = __fadd_rn(acc.w, c4.w);
  }
}

// ------------------------------------------------------- replica kernel (LDG)
// One thread owns one float4 column chunk of the padded vector per iteration
// and walks the r local replicas in groups of UJ, issuing the UJ replica and
// UJ gradient loads of a group before any arithmetic (2*UJ independent
// 16-byte loads in flight per thread).  The cross-replica sum is a register
// accumulation: every replica of a column is owned by the same thread, so no
// shuffle or shared memory is needed for it.
constexpr int kThreads = 256;

// Finish one float4 column chunk: the fused central update (n == 1) or the
// per-GPU partial (collective path).
// Reference model of the per-replica correction: z, or this GPU's u_g under
// the two-level rule (kHierA/B), which the same thread also rewrites.
template <int MODE>
__device__ __forceinline__ float4 ld_ref(const ReplicaArgs& a, int64_t p0) {
  if (MODE == kLocal) return make_float4(0.f, 0.f, 0.f, 0.f);
  if (MODE == kHierA || MODE == kHierB) return ld_rw(a.U + p0);
  return ld_ro(a.z + p0);
}

// The per-GPU partial of a float4 column chunk: to `out`, or (SMA_FLAG_P2P_PUSH)
// into slot push_rank of the owner of this chunk's shard -- a peer store over
// NVLink for every shard but this GPU's own.
__device__ __forceinline__ void store_partial(const ReplicaArgs& a, int64_t p0, float4 v) {
  if (a.push_n > 0) {
    const int g = (int)(p0 / a.push_shard);
    st4(a.push.p[g] + (int64_t)a.push_rank * a.push_shard + (p0 - (int64_t)g * a.push_shard), v);
  } else {
    st4(a.out + p0, v);
  }
}

// Section 3.3 / R20 on one component: c = alpha_g (u - z); u' = (u + D) - c.
__device__ __forceinline__ float hier_ref_elem(float u, float D, float zc, float ag, float& c) {
  c = __fmul_rn(ag, __fsub_rn(u, zc));
  return __fsub_rn(__fadd_rn(u, D), c);
}

template <int MODE>
__device__ __forceinline__ void replica_finish(const ReplicaArgs& a, int64_t p0, const float4 z,
                                               const float4 acc, bool& bad) {
  if (MODE == kLocal) return;
  if (MODE == kHierA || MODE == kHierB) {  // z holds u_g here (ld_ref)
    const float4 zc = ld_ro(a.z + p0);
    float4 un, c;
    un.x = hier_ref_elem(z.x, acc.x, zc.x, a.alpha_g, c.x);
    un.y = hier_ref_elem(z.y, acc.y, zc.y, a.alpha_g, c.y);
    un.z = hier_ref_elem(z.z, acc.z, zc.z, a.alpha_g, c.z);
    un.w = hier_ref_elem(z.w, acc.w, zc.w, a.alpha_g, c.w);
    st4(a.U + p0, un);
    if (MODE == kHierB) {  // lookahead partial alpha_g (u' - z^i)
      c.x = __fmul_rn(a.alpha_g, __fsub_rn(un.x, zc.x));
      c.y = __fmul_rn(a.alpha_g, __fsub_rn(un.y, zc.y));
      c.z = __fmul_rn(a.alpha_g, __fsub_rn(un.z, zc.z));
      c.w = __fmul_rn(a.alpha_g, __fsub_rn(un.w, zc.w));
    }
    store_partial(a, p0, c);
    bad |= !finite4(un);
    return;
  }
  if (MODE == kHierB0) {
    store_partial(a, p0, make_float4(__fmul_rn(a.alpha, acc.x), __fmul_rn(a.alpha, acc.y),
                                     __fmul_rn(a.alpha, acc.z), __fmul_rn(a.alpha, acc.w)));
    return;
  }
  if (MODE == kFused) {
    const float4 zp = ld_rw(a.zprev_next + p0);
    float4 zn;
    zn.x = central_elem(z.x, acc.x, zp.x, a.mu);
    zn.y = central_elem(z.y, acc.y, zp.y, a.mu);
    zn.z = central_elem(z.z, acc.z, zp.z, a.mu);
    zn.w = central_elem(z.w, acc.w, zp.w, a.mu);
    st4(a.zprev_next + p0, zn);
    bad |= !finite4(zn);
  } else {
    store_partial(a, p0, acc);
  }
}

template <int MODE, int kUJ, int kMinBlocks = (kUJ >= 8 ? 2 : 4), int POL = 0>
__global__ void __launch_bounds__(kThreads, kMinBlocks) replica_step_ldg(const ReplicaArgs a) {
  pdl::wait_and_release();
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  const int64_t dfull4 = a.d >> 2;  // chunks entirely below d: vector path
  const bool matc = a.C != nullptr;
  bool bad = false;
  for (int64_t c = a.c0 + (int64_t)blockIdx.x * kThreads + threadIdx.x; c < dfull4; c += stride) {
    const int64_t p0 = c << 2;
    const float4 z = ld_ref<MODE>(a, p0);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 c4;
    int j = 0;
    for (; j + kUJ <= a.r; j += kUJ) {
      float4 w[kUJ], g[kUJ];
#pragma unroll
      for (int u = 0; u < kUJ; ++u) w[u] = ld_rw_p<POL>(a.W + (int64_t)(j + u) * a.ld + p0);
#pragma unroll
      for (int u = 0; u < kUJ; ++u) g[u] = ld_ro_p<POL>(a.g.p[j + u] + p0);
#pragma unroll
      for (int u = 0; u < kUJ; ++u) {
        replica_update4<MODE>(w[u], g[u], z, acc, c4, a.alpha, a.gamma);
        st4_p<POL>(a.W + (int64_t)(j + u) * a.ld + p0, w[u]);
        if (matc) st4(a.C + (int64_t)(j + u) * a.ld + p0, c4);
        bad |= !finite4(w[u]);
      }
    }
    for (; j < a.r; ++j) {
      float4 w = ld_rw(a.W + (int64_t)j * a.ld + p0);
      const float4 g = ld_ro(a.g.p[j] + p0);
      replica_update4<MODE>(w, g, z, acc, c4, a.alpha, a.gamma);
      st4(a.W + (int64_t)j * a.ld + p0, w);
      if (matc) st4(a.C + (int64_t)j * a.ld + p0, c4);
      bad |= !finite4(w);
    }
    if (!matc) replica_finish<MODE>(a, p0, z, acc, bad);
  }
  // The chunk straddling d and the zero padding [d, d_pad): gradients are read
  // with scalar loads below d and taken as 0 above it (padding stays 0).
  const int64_t tail0 = dfull4 > a.c0 ? dfull4 : a.c0;
  for (int64_t c = tail0 + (int64_t)blockIdx.x * kThreads + threadIdx.x; c < a.n4; c += stride) {
    const int64_t p0 = c << 2;
    const float4 z = ld_ref<MODE>(a, p0);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 c4;
    for (int j = 0; j < a.r; ++j) {
      float4 w = ld_rw(a.W + (int64_t)j * a.ld + p0);
      const float4 g = ld_tail(a.g.p[j], p0, a.d);
      replica_update4<MODE>(w, g, z, acc, c4, a.alpha, a.gamma);
      st4(a.W + (int64_t)j * a.ld + p0, w);
      if (matc) st4(a.C + (int64_t)j * a.ld + p0, c4);
      bad |= !finite4(w);
    }
    if (!matc) replica_finish<MODE>(a, p0, z, acc, bad);
  }
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0)
    atomicOr(a.nonfinite, 1);
}

// ------------------------------------------- replica kernel, small rounds
// For rounds too small to fill the GPU with one thread per column (C1-C3
// sizes: the full-grid kernel runs only ~3 CTAs per SM there), G lanes share a
// float4 column: lane = group * (32/G) + column, group g takes replicas
// j = g, g + G, ... (two per load batch), and the G partial sums are combined
// with log2(G) xor-shuffles (bitwise identical in every lane: fp addition is
// commutative); group 0 finishes the column.  4x the threads for the same d.
#ifndef SMA_SPLIT_MINB
#define SMA_SPLIT_MINB 4
#endif
constexpr int kSplitMinBlocks = SMA_SPLIT_MINB;  // resident CTAs per SM the register budget allows
template <int MODE, int G, int UJ = 2>
__global__ void __launch_bounds__(kThreads, kSplitMinBlocks) replica_step_split(const ReplicaArgs a) {
  pdl::wait_and_release();
  constexpr int CPW = 32 / G;  // columns per warp
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / CPW, col = lane - grp * CPW;
  const int64_t c = ((int64_t)blockIdx.x * (kThreads / 32) + warp) * CPW + col;
  const bool valid = c < a.n4;
  const bool full = c < (a.d >> 2);
  const bool matc = a.C != nullptr;
  const int64_t p0 = c << 2;
  const float4 z = valid ? ld_ref<MODE>(a, p0) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 c4;
  bool bad = false;
  if (valid) {
    int j = grp;
    for (; j + (UJ - 1) * G < a.r; j += UJ * G) {  // UJ replicas of this lane in flight
      float4 w[UJ], g[UJ];
#pragma unroll
      for (int u = 0; u < UJ; ++u) w[u] = ld_rw(a.W + (int64_t)(j + u * G) * a.ld + p0);
#pragma unroll
      for (int u = 0; u < UJ; ++u)
        g[u] = full ? ld_ro(a.g.p[j + u * G] + p0) : ld_tail(a.g.p[j + u * G], p0, a.d);
#pragma unroll
      for (int u = 0; u < UJ; ++u) {
        replica_update4<MODE>(w[u], g[u], z, acc, c4, a.alpha, a.gamma);
        st4(a.W + (int64_t)(j + u * G) * a.ld + p0, w[u]);
        if (matc) st4(a.C + (int64_t)(j + u * G) * a.ld + p0, c4);
        bad |= !finite4(w[u]);
      }
    }
    for (; j < a.r; j += G) {
      float4 w0 = ld_rw(a.W + (int64_t)j * a.ld + p0);
      const float4 g0 = full ? ld_ro(a.g.p[j] + p0) : ld_tail(a.g.p[j], p0, a.d);
      replica_update4<MODE>(w0, g0, z, acc, c4, a.alpha, a.gamma);
      st4(a.W + (int64_t)j * a.ld + p0, w0);
      if (matc) st4(a.C + (int64_t)j * a.ld + p0, c4);
      bad |= !finite4(w0);
    }
  }
#pragma unroll
  for (int off = CPW; off < 32; off <<= 1) {  // combine the G replica groups
    acc.x = __fadd_rn(acc.x, __shfl_xor_sync(0xffffffffu, acc.x, off));
    acc.y = __fadd_rn(acc.y, __shfl_xor_sync(0xffffffffu, acc.y, off));
    acc.z = __fadd_rn(acc.z, __shfl_xor_sync(0xffffffffu, acc.z, off));
    acc.w = __fadd_rn(acc.w, __shfl_xor_sync(0xffffffffu, acc.w, off));
  }
  if (valid && grp == 0 && !matc) replica_finish<MODE>(a, p0, z, acc, bad);
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
}

// ---------------------------------------- MATERIALIZE_C: reduce c_j over j
// The north_star-literal intra-GPU reduction of the materialised corrections.
// A warp covers 8 float4 columns x 4 replica groups (lane = group*8 + column:
// four 128-byte row segments per load); the 8 warps of a block form
// `wc` column sets x `wr` replica slices (wr*wc = 8, wr = min(8, ceil(r/4))
// rounded up to a power of two).  Lane (group g, slice s) sums replicas
// j = g + 4 (s + wr t); the 4 groups are combined with two xor-shuffles and
// the wr slices with a shared-memory tree.
constexpr int kRedWarps = 8;
template <int MODE>
__global__ void __launch_bounds__(kRedWarps * 32) reduce_corrections(const ReplicaArgs a, int wr) {
  __shared__ float4 part[kRedWarps][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int col = lane & 7, grp = lane >> 3;
  const int wc = kRedWarps / wr;
  const int cs = warp % wc, sl = warp / wc;     // column set, replica slice
  const int64_t cols_per_block = 8 * wc;
  const int64_t nblk = (a.n4 + cols_per_block - 1) / cols_per_block;
  for (int64_t t = blockIdx.x; t < nblk; t += gridDim.x) {
    const int64_t c = t * cols_per_block + cs * 8 + col;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < a.n4) {
      int j = grp + 4 * sl;
      const int step = 4 * wr;
      for (; j + step < a.r; j += 2 * step) {  // two loads in flight per lane
        const float4 v0 = ld_ro(a.C + (int64_t)j * a.ld + (c << 2));
        const float4 v1 = ld_ro(a.C + (int64_t)(j + step) * a.ld + (c << 2));
        s.x = __fadd_rn(s.x, v0.x); s.y = __fadd_rn(s.y, v0.y);
        s.z = __fadd_rn(s.z, v0.z); s.w = __fadd_rn(s.w, v0.w);
        s.x = __fadd_rn(s.x, v1.x); s.y = __fadd_rn(s.y, v1.y);
        s.z = __fadd_rn(s.z, v1.z); s.w = __fadd_rn(s.w, v1.w);
      }
      for (; j < a.r; j += step) {
        const float4 v = ld_ro(a.C + (int64_t)j * a.ld + (c << 2));
        s.x = __fadd_rn(s.x, v.x); s.y = __fadd_rn(s.y, v.y);
        s.z = __fadd_rn(s.z, v.z); s.w = __fadd_rn(s.w, v.w);
      }
    }
#pragma unroll
    for (int off = 8; off <= 16; off <<= 1) {
      s.x = __fadd_rn(s.x, __shfl_xor_sync(0xffffffffu, s.x, off));
      s.y = __fadd_rn(s.y, __shfl_xor_sync(0xffffffffu, s.y, off));
      s.z = __fadd_rn(s.z, __shfl_xor_sync(0xffffffffu, s.z, off));
      s.w = __fadd_rn(s.w, __shfl_xor_sync(0xffffffffu, s.w, off));
    }
    if (grp == 0) part[warp][col] = s;
    __syncthreads();
    for (int h = wr / 2; h >= 1; h >>= 1) {  // block-level tree over replica slices
      if (sl < h && grp == 0) {
        const float4 o = part[warp + h * wc][col];
        float4 m = part[warp][col];
        m.x = __fadd_rn(m.x, o.x); m.y = __fadd_rn(m.y, o.y);
        m.z = __fadd_rn(m.z, o.z); m.w = __fadd_rn(m.w, o.w);
        part[warp][col] = m;
      }
      __syncthreads();
    }
    if (sl == 0 && grp == 0 && c < a.n4) {
      const int64_t p0 = c << 2;
      const float4 acc = part[warp][col];
      if (MODE == kFused) {
        const float4 z = ld_ro(a.z + p0);
        const float4 zp = ld_rw(a.zprev_next + p0);
        float4 zn;
        zn.x = central_elem(z.x, acc.x, zp.x, a.mu);
        zn.y = central_elem(z.y, acc.y, zp.y, a.mu);
        zn.z = central_elem(z.z, acc.z, zp.z, a.mu);
        zn.w = central_elem(z.w, acc.w, zp.w, a.mu);
        st4(a.zprev_next + p0, zn);
        if (a.nonfinite && !finite4(zn)) atomicOr(a.nonfinite, 1);
      } else {
        st4(a.out + p0, acc);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ shard update
// a7 on this GPU's shard, in place into the z_prev half of the ping-pong.
template <int MODE>
__global__ void __launch_bounds__(kThreads) zsync_kernel(const float* __restrict__ S,
                                                         const float* __restrict__ z,
                                                         float* zprev_next, int64_t n4,
                                                         float alpha, float mu, float coef_b,
                                                         int* nonfinite) {
  bool bad = false;
  for (int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x; c < n4;
       c += (int64_t)gridDim.x * kThreads) {
    const int64_t p0 = c << 2;
    const float4 s = ld_ro(S + p0), zc = ld_ro(z + p0), zp = ld_rw(zprev_next + p0);
    float4 zn;
    if (MODE == kPartialA) {  // z' = z + S + mu (z - z_prev), S = sum_j c_j
      zn.x = central_elem(zc.x, s.x, zp.x, mu);
      zn.y = central_elem(zc.y, s.y, zp.y, mu);
      zn.z = central_elem(zc.z, s.z, zp.z, mu);
      zn.w = central_elem(zc.w, s.w, zp.w, mu);
    } else {  // z' = (z + alpha S) + (mu - alpha k)(z - z_prev), S = sum_j (w_j - z_prev)
      zn.x = __fadd_rn(__fmaf_rn(alpha, s.x, zc.x), __fmul_rn(coef_b, __fsub_rn(zc.x, zp.x)));
      zn.y = __fadd_rn(__fmaf_rn(alpha, s.y, zc.y), __fmul_rn(coef_b, __fsub_rn(zc.y, zp.y)));
      zn.z = __fadd_rn(__fmaf_rn(alpha, s.z, zc.z), __fmul_rn(coef_b, __fsub_rn(zc.z, zp.z)));
      zn.w = __fadd_rn(__fmaf_rn(alpha, s.w, zc.w), __fmul_rn(coef_b, __fsub_rn(zc.w, zp.w)));
    }
    st4(zprev_next + p0, zn);
    bad |= !finite4(zn);
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

// Q = sum_j (w_j - z_prev) (Mode B prologue).
// Hierarchical (R20): Q = scale (sum_j (w_j - z_prev)) on GPU 0 (scale = alpha_l),
// Q = scale (u_g - z_prev) on GPU g >= 1 (U != nullptr, scale = alpha_g).
__global__ void __launch_bounds__(kThreads) q_prologue_kernel(const float* __restrict__ W,
                                                              int64_t ld, int r,
                                                              const float* __restrict__ zp,
                                                              float* __restrict__ Q, int64_t n4,
                                                              const float* __restrict__ U,
                                                              float scale) {
  for (int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x; c < n4;
       c += (int64_t)gridDim.x * kThreads) {
    const int64_t p0 = c << 2;
    const float4 z = ld_ro(zp + p0);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (U) {
      const float4 u = ld_ro(U + p0);
      acc = make_float4(__fsub_rn(u.x, z.x), __fsub_rn(u.y, z.y), __fsub_rn(u.z, z.z),
                        __fsub_rn(u.w, z.w));
    } else {
      for (int j = 0; j < r; ++j) {
        const float4 w = ld_ro(W + (int64_t)j * ld + p0);
        acc.x = __fadd_rn(acc.x, __fsub_rn(w.x, z.x));
        acc.y = __fadd_rn(acc.y, __fsub_rn(w.y, z.y));
        acc.z = __fadd_rn(acc.z, __fsub_rn(w.z, z.z));
        acc.w = __fadd_rn(acc.w, __fsub_rn(w.w, z.w));
      }
    }
    st4(Q + p0, make_float4(__fmul_rn(scale, acc.x), __fmul_rn(scale, acc.y),
                            __fmul_rn(scale, acc.z), __fmul_rn(scale, acc.w)));
  }
}

// ------------------------------------------------------ synthetic gradients
// DESIGN.md "Input recipe" (R9), implemented here independently of the oracle.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void __launch_bounds__(kThreads) synth_grads_kernel(float* __restrict__ G, int64_t ld,
                                                               int r, int j0, int k, int64_t d,
                                                               int64_t round, uint64_t key) {
  const int64_t n4 = ld >> 2;
  const int64_t total = n4 * r;
  for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * kThreads) {
    const int slot = (int)(t / n4);
    const int64_t p0 = (t - (int64_t)slot * n4) << 2;
    const uint64_t base = ((uint64_t)round * (uint64_t)k + (uint64_t)(j0 + slot)) * (uint64_t)d;
    float v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t p = p0 + q;
      const uint64_t h = splitmix64(key + base + (uint64_t)p);
      // (U - 1/2) 2^-4 with U = (h >> 40) 2^-24: exact in fp32
      v[q] = (p < d) ? ((float)(h >> 40) * 0x1p-24f - 0.5f) * 0.0625f : 0.f;
    }
    st4(G + (int64_t)slot * ld + p0, make_float4(v[0], v[1], v[2], v[3]));
  }
}

// ------------------------------------------------ softmax learner (a2')
// Two kernels, both spread over many SMs (one CTA per learner was bound by
// instruction issue on r SMs: 21 us; profiles/r01_ncu_learners.txt):
//  softmax_logits_kernel  grid (r, b), one warp per class: logits of row t,
//      max-subtracted softmax, E[slot][t][c] = p - onehot(y_t)   (fp32)
//  softmax_wgrad_kernel   grid (r, ceil(in_dim / kFeat)): for a slice of
//      kFeat features, dW[c][f] = (1/b) sum_t E[t][c] x[t][f]; db on slice 0.
// fp32 FFMA throughout (no TF32: SURVEY Appendix A5).
constexpr int kFeat = 64;
constexpr int kMaxClasses = 32;



__global__ void __launch_bounds__(kMaxClasses * 32) softmax_logits_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ y, const int32_t* __restrict__ perm,
    int64_t pos0, int b, int in_dim, int classes, const float* __restrict__ Wall, int64_t ld,
    int j0, float* __restrict__ E) {
  extern __shared__ __align__(16) float xs[];  // [in_dim]
  __shared__ float lg[kMaxClasses];
  const int slot = blockIdx.x, t = blockIdx.y;
  __shared__ int row_sm;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) row_sm = perm[pos0 + (int64_t)(j0 + slot) * b + t];
  __syncthreads();
  const int row = row_sm;
  // the label, in flight while the row is staged (off the softmax's tail)
  const int yt0 = threadIdx.x == 0 ? __ldg(y + row) : 0;
  const float* W = Wall + (int64_t)slot * ld;
  const bool vec = (in_dim & 3) == 0 && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  bulk::stage_rows_span(xs, X, &row_sm, 1, in_dim, in_dim, 0, nullptr, nullptr, 0, &bar, 0, true);
  // PDL: the batch row (X, perm, y: never written by a kernel) is staged while
  // the previous kernel drains; the replica W is read only after the wait
  pdl::wait_and_release();
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  if (c < classes) {  // warp c: logit of class c, W row c read straight from L2
    const float* w = W + (int64_t)c * in_dim;
    float s = 0.f;
    if (vec) {
      const float4* w4 = reinterpret_cast<const float4*>(w);
      const float4* x4 = reinterpret_cast<const float4*>(xs);
#pragma unroll 4
      for (int f = lane; f < (in_dim >> 2); f += 32) {
        const float4 a = __ldg(w4 + f), v = x4[f];
        s = __fmaf_rn(a.x, v.x, s);
        s = __fmaf_rn(a.y, v.y, s);
        s = __fmaf_rn(a.z, v.z, s);
        s = __fmaf_rn(a.w, v.w, s);
      }
    } else {
      for (int f = lane; f < in_dim; f += 32) s = __fmaf_rn(w[f], xs[f], s);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
    if (lane == 0) lg[c] = __fadd_rn(s, W[(int64_t)classes * in_dim + c]);
  }
  __syncthreads();
  if (threadIdx.x < 32)  // max-subtracted softmax of this row, e = p - onehot(y_t)
    warp_softmax_grad(lg, classes, __shfl_sync(0xffffffffu, yt0, 0),
                      E + ((int64_t)slot * b + t) * classes);
}

__global__ void __launch_bounds__(256) softmax_wgrad_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ perm, int64_t pos0, int b, int in_dim,
    int classes, int j0, int64_t ld, const float* __restrict__ E, float* __restrict__ Gall) {
  extern __shared__ float sm[];
  float* xs = sm;                  // [b][kFeat]
  float* e = xs + b * kFeat;       // [b][classes]
  __shared__ int rows[64];
  const int slot = blockIdx.x, f0 = blockIdx.y * kFeat;
  const int nf = min(kFeat, in_dim - f0);
  float* G = Gall + (int64_t)slot * ld;
  if (threadIdx.x < b) rows[threadIdx.x] = perm[pos0 + (int64_t)(j0 + slot) * b + threadIdx.x];
  __syncthreads();
  // X[rows][f0, f0 + nf) -> xs [b][nf] (one 16-byte load per thread), while the
  // logits kernel drains (PDL); E (its output) only after the wait
  bulk::load_tile(xs, X, rows, b, nf, in_dim, f0);
  pdl::wait_and_release();
  for (int q = threadIdx.x; q < b * classes; q += blockDim.x) e[q] = E[(int64_t)slot * b * classes + q];
  __syncthreads();
  const float fb = (float)b;
  for (int q = threadIdx.x; q < classes * nf; q += blockDim.x) {
    const int c = q / nf, f = q - c * nf;
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fmaf_rn(e[t * classes + c], xs[t * nf + f], s);
    G[(int64_t)c * in_dim + f0 + f] = __fdiv_rn(s, fb);
  }
  if (blockIdx.y == 0 && threadIdx.x < classes) {
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, e[t * classes + threadIdx.x]);
    G[(int64_t)classes * in_dim + threadIdx.x] = __fdiv_rn(s, fb);
  }
}

// Learner-fused round (n = 1, softmax learner): the dW slice computation of
// softmax_wgrad_kernel followed directly by a3-a5 + a7 for the same parameters
// of ALL r replicas, so the gradient never makes an HBM round trip and the
// round needs no separate replica kernel.  CTA x < nfs owns features
// [32x, 32x + 32) of every class; CTA nfs owns the biases.  All r learners'
// batch tiles are staged at once; each thread then walks its parameters and,
// per parameter, the learners in ascending j (4 replica loads in flight).  The
// arithmetic per element is exactly that of softmax_wgrad_kernel then
// replica_step_ldg<kFused> (same operation order: bitwise identical to that
// pair; the small-round split kernel sums the corrections per lane group, so
// against it the results agree to rounding).  The gradient is still written to G.
constexpr int kFeatF = 32;
constexpr int kFusedPerThread = 2;  // ceil(classes * kFeatF / 256) for classes <= 16
__global__ void __launch_bounds__(256) softmax_round_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ perm, int64_t pos0, int b, int in_dim,
    int classes, int j0, const float* __restrict__ E, float* __restrict__ Gall, const ReplicaArgs a) {
  extern __shared__ float sm[];
  pdl::wait_and_release();
  const int r = a.r;
  float* xs = sm;                              // [r][b][kFeatF]
  float* e = xs + (int64_t)r * b * kFeatF;     // [r][b][classes]
  int* rows = (int*)(e + (int64_t)r * b * classes);  // [r][b]
  const int nfs = (in_dim + kFeatF - 1) / kFeatF;
  const bool bias = blockIdx.x == nfs;
  const int f0 = blockIdx.x * kFeatF;
  const int nf = bias ? 0 : min(kFeatF, in_dim - f0);
  for (int q = threadIdx.x; q < r * b; q += blockDim.x) {
    const int j = q / b, t = q - j * b;
    rows[q] = perm[pos0 + (int64_t)(j0 + j) * b + t];
  }
  for (int q = threadIdx.x; q < r * b * classes; q += blockDim.x) e[q] = E[q];
  __shared__ __align__(8) uint64_t bar;
  __syncthreads();
  // every learner's X[rows][f0, f0 + nf) -> xs [r*b][nf] in one TMA bulk transaction
  if (!bias) bulk::stage_rows_span(xs, X, rows, r * b, nf, in_dim, f0, nullptr, nullptr, 0, &bar, 0, true);
  const int nparam = bias ? classes : classes * kFeatF;
  const float fb = (float)b;
  bool bad = false;
#pragma unroll
  for (int uu = 0; uu < kFusedPerThread; ++uu) {
    const int q = threadIdx.x + uu * 256;
    if (q >= nparam) continue;
    const int c = bias ? q : q / kFeatF, f = bias ? 0 : q - c * kFeatF;
    if (!bias && f >= nf) continue;
    const int64_t p = bias ? (int64_t)classes * in_dim + c : (int64_t)c * in_dim + f0 + f;
    const float z = a.z[p];
    float acc = 0.f;
    for (int j0c = 0; j0c < r; j0c += 4) {
      float w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = (j0c + u < r) ? a.W[(int64_t)(j0c + u) * a.ld + p] : 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0c + u;
        if (j >= r) break;
        const float* ej = e + (int64_t)j * b * classes;
        float s = 0.f;
        if (bias) {
          for (int t = 0; t < b; ++t) s = __fadd_rn(s, ej[t * classes + c]);
        } else {
          const float* xj = xs + (int64_t)j * b * nf;
          for (int t = 0; t < b; ++t) s = __fmaf_rn(ej[t * classes + c], xj[t * nf + f], s);
        }
        const float g = __fdiv_rn(s, fb);
        Gall[(int64_t)j * a.ld + p] = g;
        const StepOut o = sma_elem(w[u], g, z, a.alpha, a.gamma);
        a.W[(int64_t)j * a.ld + p] = o.wn;
        acc = __fadd_rn(acc, o.c);
        bad |= !isfinite(o.wn);
      }
    }
    const float zn = central_elem(z, acc, a.zprev_next[p], a.mu);
    a.zprev_next[p] = zn;
    bad |= !isfinite(zn);
  }
  if (a.nonfinite && bad) atomicOr(a.nonfinite, 1);
}

__global__ void __launch_bounds__(kThreads) broadcast_rows_kernel(float* __restrict__ dst, int64_t ld,
                                                                  int r, const float* __restrict__ src,
                                                                  int64_t n4) {
  const int64_t total = n4 * r;
  for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * kThreads) {
    const int slot = (int)(t / n4);
    const int64_t p0 = (t - (int64_t)slot * n4) << 2;
    st4(dst + (int64_t)slot * ld + p0, ld_ro(src + p0));
  }
}

template <typename K>
cudaError_t launch_pdl(K kernel, int grid, cudaStream_t s, const ReplicaArgs& a) {
  return pdl::launch(kernel, dim3(grid), dim3(kThreads), 0, s, 1, a);
}

template <typename K>
int grid_for(K kernel, int threads, size_t smem, int64_t work_items, int num_sms) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess ||
      occ < 1)
    occ = 1;
  const int64_t want = (work_items + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms * occ;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

// LDG launch geometry (measured, profiles/r01_ldg_variants.jsonl): one thread
// per float4 column over a full (non-persistent) grid, replicas loaded two at a
// time, is the fastest at every size (C4 k = 16: 6.71 TB/s vs 6.14 persistent
// and 6.33 for the TMA ring): the hardware CTA scheduler keeps more independent
// requests in flight than a grid-stride loop.  Knobs for experiments:
// SMA_LDG_UNROLL = 2|4|8, SMA_LDG_GRID = full|persistent.
int ldg_unroll() {
  static int u = [] {
    const char* e = getenv("SMA_LDG_UNROLL");
    const int v = e ? atoi(e) : 2;
    return (v == 4 || v == 8) ? v : 2;
  }();
  return u;
}
bool ldg_full_grid() {
  static bool f = [] {
    const char* e = getenv("SMA_LDG_GRID");
    return !(e && e[0] == 'p');
  }();
  return f;
}

int ldg_minblocks() {
  static int m = [] {
    const char* e = getenv("SMA_LDG_MINB");
    return e ? atoi(e) : 0;
  }();
  return m;
}

int ldg_policy() {
  static int p = [] {
    const char* e = getenv("SMA_LDG_POLICY");
    return e ? atoi(e) : 0;
  }();
  return p;
}

template <int MODE, int UJ>
cudaError_t launch_ldg_uj(const ReplicaArgs& a, int64_t work, int num_sms, cudaStream_t s) {
  auto k = replica_step_ldg<MODE, UJ>;
  if (UJ == 2 && ldg_policy() == 1) k = replica_step_ldg<MODE, 2, 4, 1>;
  if (UJ == 2 && ldg_policy() == 2) k = replica_step_ldg<MODE, 2, 4, 2>;
  if (UJ == 2 && ldg_minblocks() == 6) k = replica_step_ldg<MODE, 2, 6>;
  if (UJ == 2 && ldg_minblocks() == 8) k = replica_step_ldg<MODE, 2, 8>;
  const int grid = ldg_full_grid() ? (int)((work + kThreads - 1) / kThreads)
                                   : grid_for(k, kThreads, 0, work, num_sms);
  return launch_pdl(k, grid < 1 ? 1 : grid, s, a);
}

template <int MODE>
cudaError_t launch_ldg_default(const ReplicaArgs& a, int64_t work, cudaStream_t s) {
  const int grid = (int)((work + kThreads - 1) / kThreads);
  return launch_pdl(replica_step_ldg<MODE, 2>, grid < 1 ? 1 : grid, s, a);
}

template <int MODE>
cudaError_t launch_ldg(const ReplicaArgs& a, int64_t work, int num_sms, cudaStream_t s) {
  switch (ldg_unroll()) {
    case 2: return launch_ldg_uj<MODE, 2>(a, work, num_sms, s);
    case 8: return launch_ldg_uj<MODE, 8>(a, work, num_sms, s);
    default: return launch_ldg_uj<MODE, 4>(a, work, num_sms, s);
  }
}

}  // namespace

// ----------------------------------------------------------------- launchers
cudaError_t launch_replica_step(int mode, bool tma, const ReplicaArgs& a0, int num_sms,
                                cudaStream_t s) {
  ReplicaArgs a = a0;
  a.c0 = 0;
  if (tma && (mode == kFused || mode == kPartialA || mode == kPartialB)) {  // TMA-staged full tiles, then the LDG kernel for the rest
    const int64_t nt = tma_full_tiles(a.d);
    cudaError_t e = launch_replica_step_tma(mode, a, nt, num_sms, s);
    if (e != cudaSuccess) return e;
    a.c0 = nt * tma_tile_floats() / 4;
    if (a.c0 >= a.n4) return cudaSuccess;
  }
  const int64_t work = a.n4 - a.c0;
  // small rounds: lanes split the replicas of a column (see replica_step_split)
  static const int64_t split_below = [] {
    const char* e = getenv("SMA_SPLIT_BELOW");   // float4 chunks; 0 disables
    return e ? atoll(e) : 148ll * 1024;
  }();
  // measured (profiles/r01_split.jsonl): splitting pays when the column count
  // cannot fill the GPU (d < ~150k) or when r >= 8 replicas lengthen each
  // thread's chain; at medium d with r = 4 it is slower
  const bool split = a.c0 == 0 && mode != kLocal && a.r >= 2 &&
                     (a.n4 < split_below / 4 || (a.n4 < split_below && a.r >= 8));
  if (split) {
    static const int g_knob = [] {  // SMA_SPLIT_G = 2|4|8|16: experiments only
      const char* e = getenv("SMA_SPLIT_G");
      const int v = e ? atoi(e) : 0;
      return (v == 2 || v == 4 || v == 8 || v == 16) ? v : 0;
    }();
    // lanes per column: 2 once two lanes per column already give ~100k threads
    // and r <= 16 (more replicas per lane in flight), else 4 (more parallelism);
    // measured with PDL (profiles/r01_split.jsonl): C2 153k -> 169k rounds/s, C3
    // 98k -> 102k with G = 2; C1 (d = 8k) and r = 32 are better with G = 4
    int G = (a.n4 * 2 >= 100000 && a.r <= 16) ? 2 : (a.r >= 4 ? 4 : 2);
    if (g_knob) G = g_knob;
    // replicas per lane in flight: 4 when a lane has >= 4 of them (C2 k = 8:
    // 161k -> 174k rounds/s, k = 16: 108k -> 118k; profiles/r01_split.jsonl),
    // else 2; SMA_SPLIT_UJ = 2|4 forces it
    static const int uj_knob = [] {
      const char* e = getenv("SMA_SPLIT_UJ");
      const int v = e ? atoi(e) : 0;
      return (v == 2 || v == 4) ? v : 0;
    }();
    const int uj = uj_knob ? uj_knob : (a.r >= 4 * G ? 4 : 2);
    const int64_t cols_per_block = (kThreads / 32) * (32 / G);
    const int grid = (int)((a.n4 + cols_per_block - 1) / cols_per_block);
#define SMA_SPLIT_LAUNCH(M)                                                                  \
  if (G == 16) e = launch_pdl(replica_step_split<M, 16>, grid, s, a);                         \
  else if (G == 8) e = launch_pdl(replica_step_split<M, 8>, grid, s, a);                      \
  else if (G == 4) e = uj == 4 ? launch_pdl(replica_step_split<M, 4, 4>, grid, s, a)          \
                               : launch_pdl(replica_step_split<M, 4>, grid, s, a);            \
  else e = uj == 4 ? launch_pdl(replica_step_split<M, 2, 4>, grid, s, a)                      \
                   : launch_pdl(replica_step_split<M, 2>, grid, s, a);
    cudaError_t e = cudaSuccess;
    switch (mode) {
      case kFused: SMA_SPLIT_LAUNCH(kFused) break;
      case kPartialA: SMA_SPLIT_LAUNCH(kPartialA) break;
      case kPartialB: SMA_SPLIT_LAUNCH(kPartialB) break;
      case kHierA: SMA_SPLIT_LAUNCH(kHierA) break;
      case kHierB: SMA_SPLIT_LAUNCH(kHierB) break;
      case kHierB0: SMA_SPLIT_LAUNCH(kHierB0) break;
      default: return cudaErrorInvalidValue;
    }
#undef SMA_SPLIT_LAUNCH
    return e;
  }
  switch (mode) {
    case kFused: return launch_ldg<kFused>(a, work, num_sms, s);
    case kPartialA: return launch_ldg<kPartialA>(a, work, num_sms, s);
    case kPartialB: return launch_ldg<kPartialB>(a, work, num_sms, s);
    case kLocal: return launch_ldg<kLocal>(a, work, num_sms, s);
    // two-level rule: the default geometry only (no experiment-knob variants)
    case kHierA: return launch_ldg_default<kHierA>(a, work, s);
    case kHierB: return launch_ldg_default<kHierB>(a, work, s);
    case kHierB0: return launch_ldg_default<kHierB0>(a, work, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_reduce_corrections(int mode, const ReplicaArgs& a, int num_sms,
                                      cudaStream_t s) {
  // replica slices per column set: 1 (no block tree) up to r = 32, so each lane
  // sums r/4 replicas with its loads in flight; the shared-memory tree over
  // slices is used beyond that (measured: with a slice per 4 replicas each lane
  // made one load and the kernel ran at 2.3 TB/s)
  int wr = 1;
  while (wr < kRedWarps && 32 * wr < a.r) wr <<= 1;
  const int64_t cols = 8 * (kRedWarps / wr);
  const int64_t blocks = (a.n4 + cols - 1) / cols;
  // full grid (one tile per CTA), like the replica kernel: more requests in flight
  const int grid = (int)(blocks < INT32_MAX ? blocks : INT32_MAX);
  (void)num_sms;
  if (mode == kFused)
    reduce_corrections<kFused><<<grid, kRedWarps * 32, 0, s>>>(a, wr);
  else if (mode == kPartialA)
    reduce_corrections<kPartialA><<<grid, kRedWarps * 32, 0, s>>>(a, wr);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_zsync(int mode, const float* S, const float* z, float* zprev_next, int64_t n4,
                         float alpha, float mu, float coef_b, int* nonfinite, int num_sms,
                         cudaStream_t s) {
  if (mode == kPartialA) {
    auto k = zsync_kernel<kPartialA>;
    k<<<grid_for(k, kThreads, 0, n4, num_sms), kThreads, 0, s>>>(S, z, zprev_next, n4, alpha, mu,
                                                                 coef_b, nonfinite);
  } else {
    auto k = zsync_kernel<kPartialB>;
    k<<<grid_for(k, kThreads, 0, n4, num_sms), kThreads, 0, s>>>(S, z, zprev_next, n4, alpha, mu,
                                                                 coef_b, nonfinite);
  }
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kThreads) push_partial_kernel(const float* __restrict__ src,
                                                                const ReplicaArgs a) {
  for (int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x; c < a.n4;
       c += (int64_t)gridDim.x * kThreads)
    store_partial(a, c << 2, ld_ro(src + (c << 2)));
}

cudaError_t launch_push_partial(const float* src, const ReplicaArgs& a, int num_sms, cudaStream_t s) {
  push_partial_kernel<<<grid_for(push_partial_kernel, kThreads, 0, a.n4, num_sms), kThreads, 0, s>>>(
      src, a);
  return cudaGetLastError();
}

cudaError_t launch_q_prologue(const float* W, int64_t ld, int r, const float* zprev, float* Q,
                              int64_t n4, const float* U, float scale, int num_sms,
                              cudaStream_t s) {
  q_prologue_kernel<<<grid_for(q_prologue_kernel, kThreads, 0, n4, num_sms), kThreads, 0, s>>>(
      W, ld, r, zprev, Q, n4, U, scale);
  return cudaGetLastError();
}

cudaError_t launch_synth_grads(float* G, int64_t ld, int r, int j0, int k, int64_t d,
                               int64_t round, uint64_t seed, int num_sms, cudaStream_t s) {
  // key(seed) = splitmix64(seed), computed on the host side of the launch
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const uint64_t key = z ^ (z >> 31);
  synth_grads_kernel<<<grid_for(synth_grads_kernel, kThreads, 0, (ld >> 2) * r, num_sms), kThreads,
                       0, s>>>(G, ld, r, j0, k, d, round, key);
  return cudaGetLastError();
}

cudaError_t launch_softmax_grad(const float* X, const int32_t* y, const int32_t* perm, int64_t pos0,
                                int b, int in_dim, int classes, const float* W, int64_t ld, int r,
                                int j0, float* E, float* G, cudaStream_t s) {
  if (classes > kMaxClasses || b > 64) return cudaErrorInvalidValue;
  const size_t sm1 = sizeof(float) * (size_t)in_dim;
  const size_t sm2 = sizeof(float) * ((size_t)b * kFeat + (size_t)b * classes);
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(softmax_logits_kernel), (int)sm1);
  if (e != cudaSuccess) return e;
  e = pdl::launch(softmax_logits_kernel, dim3(r, b), dim3(classes * 32), sm1, s, 1, X, y, perm, pos0,
                  b, in_dim, classes, W, ld, j0, E);
  if (e != cudaSuccess) return e;
  return pdl::launch(softmax_wgrad_kernel, dim3(r, (in_dim + kFeat - 1) / kFeat), dim3(256), sm2, s,
                     1, X, perm, pos0, b, in_dim, classes, j0, ld, E, G);
}

cudaError_t launch_softmax_round(const float* X, const int32_t* y, const int32_t* perm,
                                 int64_t pos0, int b, int in_dim, int classes, int j0, float* E,
                                 float* G, const ReplicaArgs& a, cudaStream_t s) {
  if (classes > kMaxClasses || b > 64 || classes * kFeatF > kFusedPerThread * 256)
    return cudaErrorInvalidValue;
  const size_t sm1 = sizeof(float) * (size_t)in_dim;
  const size_t sm2 = sizeof(float) * ((size_t)a.r * b * kFeatF + (size_t)a.r * b * classes) +
                     sizeof(int) * (size_t)a.r * b;
  if (sm2 > 200 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(softmax_logits_kernel), (int)sm1);
  if (e != cudaSuccess) return e;
  if ((e = ensure_dyn_smem(reinterpret_cast<const void*>(softmax_round_kernel), (int)sm2)) != cudaSuccess)
    return e;
  e = pdl::launch(softmax_logits_kernel, dim3(a.r, b), dim3(classes * 32), sm1, s, 1, X, y, perm,
                  pos0, b, in_dim, classes, (const float*)a.W, a.ld, j0, E);
  if (e != cudaSuccess) return e;
  const int nfs = (in_dim + kFeatF - 1) / kFeatF;
  return pdl::launch(softmax_round_kernel, dim3(nfs + 1), dim3(256), sm2, s, 1, X, perm, pos0, b,
                     in_dim, classes, j0, (const float*)E, G, a);
}

cudaError_t launch_broadcast_rows(float* dst, int64_t ld, int r, const float* src, int64_t n4,
                                  int num_sms, cudaStream_t s) {
  broadcast_rows_kernel<<<grid_for(broadcast_rows_kernel, kThreads, 0, n4 * r, num_sms), kThreads,
                          0, s>>>(dst, ld, r, src, n4);
  return cudaGetLastError();
}

}  // namespace sma
