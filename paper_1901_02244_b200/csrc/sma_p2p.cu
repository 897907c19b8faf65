// sma_p2p.cu -- the inter-GPU z-sync (a6 + a7 + a8) as ONE kernel over peer
// memory (CUDA IPC mappings of every rank's buffers), no NCCL on the data path.
//
// Every rank owns one cudaMalloc region [flags | partial(s) | z[2]] and maps the
// regions of all other ranks (cudaIpcOpenMemHandle; handles exchanged by the
// caller, e.g. with torch.distributed).  Rank g then, for each float4 chunk of
// ITS shard of z:
//   S  = sum over ranks g' = 0..n-1 (ascending) of partial_{g'}[chunk]   (a6: peer loads)
//   z' = z + S + mu (z - z_prev)                 (Mode A)                 (a7)
//   z' = (z + alpha S) + (mu - alpha k)(z - z_prev)  (Mode B)
//   store z' into z[1-cur][chunk] of every rank                          (a8: peer stores)
// so the reduce-scatter, the shard update and the all-gather are one pass that
// overlaps loads from peers with stores to peers tile by tile.  Two barriers
// (release stores of a per-source flag into every peer's flag array, acquire
// spins on the local array; targets kept in device memory so CUDA graphs can
// replay the kernel) order "every partial is complete" before the loads and
// "every shard has landed" before the next round.  Barrier A is taken at
// system scope by ONE thread (CTA 0), which then releases the rest of the
// grid through a device-scope flag in local memory: the other CTAs spin on an
// L2-resident ld.acquire.gpu instead of n system-scope acquires each (the
// release -> acquire chain is transitive, so every CTA's later loads of the
// peers' partials are ordered after the peers' writes).  A barrier that does
// not complete within ~30 s traps, so a broken peer fails the process loudly.
//
// Because no NCCL communicator is involved, several processes may share one
// GPU (cudaIpc works within a device), which is how the multi-rank path is
// tested on a single B200 (tests/test_p2p_multiprocess.py).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "sma_internal.h"

namespace sma {
namespace {
constexpr int kP2PThreads = 256;

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Wait until flags[0..n) (written by the n ranks) all reached `target`.
__device__ __forceinline__ void wait_all(const unsigned* flags, int n, unsigned target) {
  const long long t0 = clock64();
  for (int g = 0; g < n; ++g)
    while ((int)(ld_acquire_sys(flags + g) - target) < 0) {
      if (clock64() - t0 > 60000000000ll) __trap();  // ~30 s: a peer never arrived
      __nanosleep(64);
    }
}
// z[cur] is read-only for the whole kernel on every rank (its last writer is
// the previous round's z-sync, complete before this launch), so the
// non-coherent path is legal for it.  The partials are NOT: a peer's replica
// kernel (Mode A), or its push epilogue (SMA_FLAG_P2P_PUSH, into this rank's
// slots), may still be writing them while this kernel is already resident and
// spinning at barrier A, and PTX requires .nc data to be read-only for the
// kernel's whole lifetime.  They are loaded with weak coherent loads after the
// barrier (ordered by its acquire + bar.sync), no L1 allocation: peer data is
// never reused.  z[1-cur] of this rank's chunk is read then written by the same
// thread (coherent path).  (.cg loads here measured ~half the bandwidth at n = 1.)
__device__ __forceinline__ float4 ld_ro4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_rw4(const float* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st4(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

template <int MODE>
__device__ __forceinline__ float4 shard_update(float4 zc, float4 s, float4 zp, const P2PArgs& a) {
  float4 zn;
  if (MODE == kPartialA) {  // z' = (z + S) + mu (z - z_prev)
    zn.x = __fadd_rn(__fadd_rn(zc.x, s.x), __fmul_rn(a.mu, __fsub_rn(zc.x, zp.x)));
    zn.y = __fadd_rn(__fadd_rn(zc.y, s.y), __fmul_rn(a.mu, __fsub_rn(zc.y, zp.y)));
    zn.z = __fadd_rn(__fadd_rn(zc.z, s.z), __fmul_rn(a.mu, __fsub_rn(zc.z, zp.z)));
    zn.w = __fadd_rn(__fadd_rn(zc.w, s.w), __fmul_rn(a.mu, __fsub_rn(zc.w, zp.w)));
  } else {                  // z' = (z + alpha S) + (mu - alpha k)(z - z_prev)
    zn.x = __fadd_rn(__fmaf_rn(a.alpha, s.x, zc.x), __fmul_rn(a.coef_b, __fsub_rn(zc.x, zp.x)));
    zn.y = __fadd_rn(__fmaf_rn(a.alpha, s.y, zc.y), __fmul_rn(a.coef_b, __fsub_rn(zc.y, zp.y)));
    zn.z = __fadd_rn(__fmaf_rn(a.alpha, s.z, zc.z), __fmul_rn(a.coef_b, __fsub_rn(zc.z, zp.z)));
    zn.w = __fadd_rn(__fmaf_rn(a.alpha, s.w, zc.w), __fmul_rn(a.coef_b, __fsub_rn(zc.w, zp.w)));
  }
  return zn;
}

// BAR = 1: barrier A at system scope in CTA 0 only, the grid released through
// the device-scope flag ctl[3]; BAR = 0 (SMA_P2P_BARRIER=0, measurement only):
// every CTA's thread 0 takes the n system-scope acquires itself (round 1).
template <int MODE, int BAR>
__global__ void __launch_bounds__(kP2PThreads) zsync_p2p_kernel(const P2PArgs a) {
  __shared__ unsigned s_targetA;
  const int n = a.n;
  if (threadIdx.x == 0) {
    const unsigned tA = a.ctl[0] + 1u;
    if (blockIdx.x == 0) {  // barrier A: my partial is complete -> tell every rank
      for (int g = 0; g < n; ++g)
        st_release_sys(reinterpret_cast<unsigned*>(a.base[g] + a.off_flags) + a.rank, tA);
      wait_all(reinterpret_cast<const unsigned*>(a.base[a.rank] + a.off_flags), n, tA);
      if (BAR) st_release_gpu(a.ctl + 3, tA);  // every rank's partial is complete
    } else if (BAR) {
      const long long t0 = clock64();
      while ((int)(ld_acquire_gpu(a.ctl + 3) - tA) < 0) {
        if (clock64() - t0 > 60000000000ll) __trap();
        __nanosleep(32);
      }
    } else {
      wait_all(reinterpret_cast<const unsigned*>(a.base[a.rank] + a.off_flags), n, tA);
    }
    s_targetA = tA;
  }
  __syncthreads();
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * kP2PThreads;
  const float* zl = reinterpret_cast<const float*>(a.base[a.rank] + a.off_z);
  const float* zpl = reinterpret_cast<const float*>(a.base[a.rank] + a.off_zprev);
  // source g's contribution to element e of this rank's shard: a peer load of
  // g's partial, or (SMA_FLAG_P2P_PUSH: g's replica kernel already stored it into
  // slot g of this rank's buffer) a local load
  const float* mine = reinterpret_cast<const float*>(a.base[a.rank] + a.off_part);
  const int64_t shard = a.len4 << 2, soff = a.off4 << 2;
  auto part_ptr = [&](int g, int64_t e) -> const float* {
    return a.push ? mine + (int64_t)g * shard + (e - soff)
                  : reinterpret_cast<const float*>(a.base[g] + a.off_part) + e;
  };
  // SMA_P2P_EMULATE_N = N on a 1-rank handle (bench.py --emulate-n; measurement
  // only, the z it produces is WRONG outside the first 1/N of the vector): the
  // kernel moves the HBM traffic that ONE GPU of an N-rank job sees -- its whole
  // partial read (its own shard by itself, the others by the peers' loads), the
  // whole z[1-cur] written (every owner's all-gather stores land here), but z and
  // z_prev read only on its own 1/N shard -- so the overlapped replica kernel can
  // be measured against that load on one GPU.
  const int64_t own4 = a.emu_n ? a.len4 / a.emu_n : a.len4;
  // two chunks per iteration: 2n peer loads + 4 local loads in flight
  int64_t c = (int64_t)blockIdx.x * kP2PThreads + threadIdx.x;
  for (; c + stride < a.len4; c += 2 * stride) {
    const int64_t e0 = (a.off4 + c) << 2, e1 = (a.off4 + c + stride) << 2;
    float4 s0 = make_float4(0.f, 0.f, 0.f, 0.f), s1 = s0;
    for (int g = 0; g < n; ++g) {  // a6: the shard's sum over ranks, ascending rank
      const float4 v0 = ld_rw4(part_ptr(g, e0)), v1 = ld_rw4(part_ptr(g, e1));
      s0.x = __fadd_rn(s0.x, v0.x); s0.y = __fadd_rn(s0.y, v0.y);
      s0.z = __fadd_rn(s0.z, v0.z); s0.w = __fadd_rn(s0.w, v0.w);
      s1.x = __fadd_rn(s1.x, v1.x); s1.y = __fadd_rn(s1.y, v1.y);
      s1.z = __fadd_rn(s1.z, v1.z); s1.w = __fadd_rn(s1.w, v1.w);
    }
    const float4 f0 = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool o0 = c < own4, o1 = c + stride < own4;
    const float4 zn0 = shard_update<MODE>(o0 ? ld_ro4(zl + e0) : f0, s0, o0 ? ld_rw4(zpl + e0) : f0, a);  // a7
    const float4 zn1 = shard_update<MODE>(o1 ? ld_ro4(zl + e1) : f0, s1, o1 ? ld_rw4(zpl + e1) : f0, a);
    for (int g = 0; g < n; ++g) {  // a8: broadcast the updated shard chunks
      float* zg = reinterpret_cast<float*>(a.base[g] + a.off_zprev);
      st4(zg + e0, zn0);
      st4(zg + e1, zn1);
    }
    bad |= !(isfinite(zn0.x) && isfinite(zn0.y) && isfinite(zn0.z) && isfinite(zn0.w));
    bad |= !(isfinite(zn1.x) && isfinite(zn1.y) && isfinite(zn1.z) && isfinite(zn1.w));
  }
  for (; c < a.len4; c += stride) {
    const int64_t e = (a.off4 + c) << 2;  // element offset in the padded vector
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int g = 0; g < n; ++g) {
      const float4 v = ld_rw4(part_ptr(g, e));
      sum.x = __fadd_rn(sum.x, v.x); sum.y = __fadd_rn(sum.y, v.y);
      sum.z = __fadd_rn(sum.z, v.z); sum.w = __fadd_rn(sum.w, v.w);
    }
    const float4 f0 = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool o = c < own4;
    const float4 zn = shard_update<MODE>(o ? ld_ro4(zl + e) : f0, sum, o ? ld_rw4(zpl + e) : f0, a);
    for (int g = 0; g < n; ++g) st4(reinterpret_cast<float*>(a.base[g] + a.off_zprev) + e, zn);
    bad |= !(isfinite(zn.x) && isfinite(zn.y) && isfinite(zn.z) && isfinite(zn.w));
  }
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.nonfinite, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    // Barrier B.  Each CTA's arrival is a gpu-scope release (it orders the CTA's
    // peer stores, made visible to thread 0 by the bar.sync above) and the last
    // arrival's acquire sees them all; its system-scope release to every peer is
    // cumulative, so a peer that acquires the flag sees every store of this
    // rank's grid (PTX causality order is transitive across the two scopes).
    // Round 1 ran a __threadfence_system per CTA instead: 53 % of the stall
    // samples of the C3 z-sync (profiles/r02_ncu_p2p_c3.txt).
    const unsigned prev = BAR ? atom_add_acq_rel_gpu(a.ctl + 2, 1u)
                              : (__threadfence_system(), atomicAdd(a.ctl + 2, 1u));
    if (prev == gridDim.x - 1) {  // the last CTA of this rank closes the round
      if (!BAR) __threadfence_system();
      a.ctl[2] = 0;
      const unsigned tB = a.ctl[1] + 1u;
      if (BAR) asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int g = 0; g < n; ++g) {  // barrier B: my shard has landed everywhere
        unsigned* f = reinterpret_cast<unsigned*>(a.base[g] + a.off_flags) + 64 + a.rank;
        if (BAR) st_relaxed_sys(f, tB);   // fence.release + strong write = release pattern
        else st_release_sys(f, tB);
      }
      wait_all(reinterpret_cast<const unsigned*>(a.base[a.rank] + a.off_flags) + 64, n, tB);
      a.ctl[0] = s_targetA;
      a.ctl[1] = tB;
      __threadfence();
    }
  }
}
}  // namespace

cudaError_t launch_zsync_p2p(int mode, const P2PArgs& a, int num_ctas, cudaStream_t s) {
  // A persistent grid (at most num_ctas: #SMs x 4) sized so every thread has
  // >= 4 float4 chunks of the shard (2 per loop iteration): the per-CTA barrier
  // work (one device-scope wait, one arrival) is then amortised, and a small
  // shard (C3 at n = 8: 14.5k chunks) runs on a few CTAs instead of ~450.
  const int64_t want = (a.len4 + 4 * kP2PThreads - 1) / (4 * kP2PThreads);
  int grid = (int)((num_ctas > 0 && want > num_ctas) ? num_ctas : want);
  if (grid < 1) grid = 1;
  // Launched without PDL (no measurable gain on one GPU: C3 Mode A 41-46k rounds/s
  // either way, within the run-to-run spread of the barrier spin; profiles/r01_pdl.txt),
  // so the next replica kernel starts only after this kernel has completed.
  static const int bar = [] {
    const char* e = getenv("SMA_P2P_BARRIER");
    return e && e[0] == '0' ? 0 : 1;
  }();
  if (mode == kPartialA) {
    if (bar) zsync_p2p_kernel<kPartialA, 1><<<grid, kP2PThreads, 0, s>>>(a);
    else zsync_p2p_kernel<kPartialA, 0><<<grid, kP2PThreads, 0, s>>>(a);
  } else {
    if (bar) zsync_p2p_kernel<kPartialB, 1><<<grid, kP2PThreads, 0, s>>>(a);
    else zsync_p2p_kernel<kPartialB, 0><<<grid, kP2PThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace sma
