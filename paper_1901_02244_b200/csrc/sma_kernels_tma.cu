// sma_kernels_tma.cu -- the replica kernel with TMA bulk-copy staging (sm_100a).
//
// Same arithmetic as replica_step_ldg (sma_kernels.cu), different data movement:
// one persistent CTA per SM; a producer warp streams (w_j, g_j) column tiles of
// kTile floats from HBM into a ring of kStages shared-memory slots with 1-D
// `cp.async.bulk` (TMA) completing on per-slot mbarriers; 8 consumer warps read
// the tiles from shared memory, update the replicas, store w' with 128-bit
// stores and accumulate the cross-replica sum in registers.  The z (and z_prev)
// tile of a column block is loaded once into its own double-buffered slot.
// Tiles that straddle d and the padding are left to the LDG kernel (tail launch).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "sma_internal.h"

namespace sma {
namespace {

// Tile (floats per stream per TMA op) and ring depth; the default
// (2048 floats = 8 KB, 8 stages = 128 KB of (w, g) in flight per SM) was the
// best of the sweep in profiles/r01_sweep_tma.jsonl.  SMA_TMA_CONFIG=<i>
// selects another entry of kTmaConfigs (tuning knob, documented in DESIGN.md).
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreadsTma = kConsumers + 32;  // + 1 producer warp

template <int TILE, int STAGES>
struct __align__(128) TmaSmem {
  float w[STAGES][TILE];
  float g[STAGES][TILE];
  float z[2][TILE];
  float zp[2][TILE];
  uint64_t full[STAGES], empty[STAGES];
  uint64_t zfull[2], zempty[2];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// 1-D TMA: global -> shared, completion counted in bytes on the mbarrier.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st4(float* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ bool finite4(float4 v) {
  return isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w);
}
__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// Alg. 1 lines 9-10 and 13, the same fixed fp32 sequence as sma_kernels.cu.
__device__ __forceinline__ void upd(float& w, float g, float z, float alpha, float gamma, float& c) {
  c = __fmul_rn(alpha, __fsub_rn(w, z));
  w = __fsub_rn(__fmaf_rn(-gamma, g, w), c);
}
__device__ __forceinline__ float central(float z, float s, float zp, float mu) {
  return __fadd_rn(__fadd_rn(z, s), __fmul_rn(mu, __fsub_rn(z, zp)));
}

template <int MODE, int TILE, int STAGES>
__global__ void __launch_bounds__(kThreadsTma, 1)
    replica_step_tma(const ReplicaArgs a, int64_t ntiles) {
  constexpr int kTile = TILE, kStages = STAGES;
  constexpr int kVecPerThread = kTile / 4 / kConsumers;  // float4s per consumer thread
  static_assert(kTile % (4 * kConsumers) == 0, "tile must split evenly");
  extern __shared__ __align__(128) uint8_t smem_raw[];
  TmaSmem<TILE, STAGES>& sm = *reinterpret_cast<TmaSmem<TILE, STAGES>*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool need_zp = (MODE == kFused);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], kConsumerWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.zfull[s], 1);
      mbar_init(&sm.zempty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int slot = 0;
      uint32_t phase = 0;
      int zb = 0;
      uint32_t zphase = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t p0 = t * kTile;
        mbar_wait(&sm.zempty[zb], zphase ^ 1);
        mbar_expect_tx(&sm.zfull[zb], (need_zp ? 2u : 1u) * kTile * 4u);
        tma_load_1d(sm.z[zb], a.z + p0, kTile * 4u, &sm.zfull[zb], pol);
        if (need_zp) tma_load_1d(sm.zp[zb], a.zprev_next + p0, kTile * 4u, &sm.zfull[zb], pol);
        if (++zb == 2) { zb = 0; zphase ^= 1; }
        for (int j = 0; j < a.r; ++j) {
          mbar_wait(&sm.empty[slot], phase ^ 1);
          mbar_expect_tx(&sm.full[slot], 2u * kTile * 4u);
          tma_load_1d(sm.w[slot], a.W + (int64_t)j * a.ld + p0, kTile * 4u, &sm.full[slot], pol);
          tma_load_1d(sm.g[slot], a.g.p[j] + p0, kTile * 4u, &sm.full[slot], pol);
          if (++slot == kStages) { slot = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const bool matc = a.C != nullptr;
  bool bad = false;
  int slot = 0;
  uint32_t phase = 0;
  int zb = 0;
  uint32_t zphase = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t p0 = t * kTile;
    mbar_wait(&sm.zfull[zb], zphase);
    float4 z[kVecPerThread], acc[kVecPerThread];
#pragma unroll
    for (int v = 0; v < kVecPerThread; ++v) {
      z[v] = lds4(&sm.z[zb][(v * kConsumers + threadIdx.x) * 4]);
      acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int j = 0; j < a.r; ++j) {
      mbar_wait(&sm.full[slot], phase);
#pragma unroll
      for (int v = 0; v < kVecPerThread; ++v) {
        const int e = (v * kConsumers + threadIdx.x) * 4;
        float4 w = lds4(&sm.w[slot][e]);
        const float4 g = lds4(&sm.g[slot][e]);
        float4 c;
        upd(w.x, g.x, z[v].x, a.alpha, a.gamma, c.x);
        upd(w.y, g.y, z[v].y, a.alpha, a.gamma, c.y);
        upd(w.z, g.z, z[v].z, a.alpha, a.gamma, c.z);
        upd(w.w, g.w, z[v].w, a.alpha, a.gamma, c.w);
        if (MODE == kPartialB) {
          acc[v].x = __fadd_rn(acc[v].x, __fsub_rn(w.x, z[v].x));
          acc[v].y = __fadd_rn(acc[v].y, __fsub_rn(w.y, z[v].y));
          acc[v].z = __fadd_rn(acc[v].z, __fsub_rn(w.z, z[v].z));
          acc[v].w = __fadd_rn(acc[v].w, __fsub_rn(w.w, z[v].w));
        } else {
          acc[v].x = __fadd_rn(acc[v].x, c.x);
          acc[v].y = __fadd_rn(acc[v].y, c.y);
          acc[v].z = __fadd_rn(acc[v].z, c.z);
          acc[v].w = __fadd_rn(acc[v].w, c.w);
        }
        st4(a.W + (int64_t)j * a.ld + p0 + e, w);
        if (matc) st4(a.C + (int64_t)j * a.ld + p0 + e, c);
        bad |= !finite4(w);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.empty[slot]);
      if (++slot == kStages) { slot = 0; phase ^= 1; }
    }
    if (!matc) {
#pragma unroll
      for (int v = 0; v < kVecPerThread; ++v) {
        const int e = (v * kConsumers + threadIdx.x) * 4;
        if (MODE == kFused) {
          const float4 zp = lds4(&sm.zp[zb][e]);
          float4 zn;
          zn.x = central(z[v].x, acc[v].x, zp.x, a.mu);
          zn.y = central(z[v].y, acc[v].y, zp.y, a.mu);
          zn.z = central(z[v].z, acc[v].z, zp.z, a.mu);
          zn.w = central(z[v].w, acc[v].w, zp.w, a.mu);
          st4(a.zprev_next + p0 + e, zn);
          bad |= !finite4(zn);
        } else {
          st4(a.out + p0 + e, acc[v]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.zempty[zb]);
    if (++zb == 2) { zb = 0; zphase ^= 1; }
  }
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.nonfinite, 1);
}

template <int MODE, int TILE, int STAGES>
cudaError_t launch_mode(const ReplicaArgs& a, int64_t ntiles, int num_sms, cudaStream_t s) {
  auto k = replica_step_tma<MODE, TILE, STAGES>;
  const int smem = (int)sizeof(TmaSmem<TILE, STAGES>);
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(k), smem);
  if (e != cudaSuccess) return e;
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreadsTma, smem) != cudaSuccess ||
      occ < 1)
    occ = 1;
  const int64_t cap = (int64_t)num_sms * occ;
  const int grid = (int)(ntiles < cap ? ntiles : cap);
  k<<<grid, kThreadsTma, smem, s>>>(a, ntiles);
  return cudaGetLastError();
}

struct TmaConfig { int tile, stages; };
// index 0 is the default
constexpr TmaConfig kTmaConfigs[] = {{2048, 8}, {4096, 4}, {1024, 16}, {2048, 4}, {1024, 6},
                                     {4096, 2}, {2048, 12}};
constexpr int kNumTmaConfigs = sizeof(kTmaConfigs) / sizeof(kTmaConfigs[0]);

int tma_config() {
  static int cfg = [] {
    const char* e = getenv("SMA_TMA_CONFIG");
    int v = e ? atoi(e) : 0;
    return (v >= 0 && v < kNumTmaConfigs) ? v : 0;
  }();
  return cfg;
}

template <int MODE>
cudaError_t launch_cfg(const ReplicaArgs& a, int64_t ntiles, int num_sms, cudaStream_t s) {
  switch (tma_config()) {
    case 1: return launch_mode<MODE, 4096, 4>(a, ntiles, num_sms, s);
    case 2: return launch_mode<MODE, 1024, 16>(a, ntiles, num_sms, s);
    case 3: return launch_mode<MODE, 2048, 4>(a, ntiles, num_sms, s);
    case 4: return launch_mode<MODE, 1024, 6>(a, ntiles, num_sms, s);
    case 5: return launch_mode<MODE, 4096, 2>(a, ntiles, num_sms, s);
    case 6: return launch_mode<MODE, 2048, 12>(a, ntiles, num_sms, s);
    default: return launch_mode<MODE, 2048, 8>(a, ntiles, num_sms, s);
  }
}

}  // namespace

int64_t tma_tile_floats() { return kTmaConfigs[tma_config()].tile; }
int64_t tma_full_tiles(int64_t d) { return d / tma_tile_floats(); }

cudaError_t launch_replica_step_tma(int mode, const ReplicaArgs& a, int64_t ntiles, int num_sms,
                                    cudaStream_t s) {
  if (ntiles <= 0) return cudaSuccess;
  switch (mode) {
    case kFused: return launch_cfg<kFused>(a, ntiles, num_sms, s);
    case kPartialA: return launch_cfg<kPartialA>(a, ntiles, num_sms, s);
    case kPartialB: return launch_cfg<kPartialB>(a, ntiles, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sma
