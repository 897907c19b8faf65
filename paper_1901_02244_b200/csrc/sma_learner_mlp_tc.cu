// sma_learner_mlp_tc.cu -- NEXT-2: the MLP learner's first-layer GEMM on the
// 5th-generation tensor cores (tcgen05 + TMEM + TMA + a thread-block cluster).
//
// a1[t][u] = sum_f W1[u][f] x_t[f] + b1[u] for every local learner, hidden
// unit u and batch row t (forward layer 1 of back-propagation, PAPER.md:249-256;
// SPEC S:104's 784-256-10 MLP).  As a GEMM per learner: D[u][t] = A[u][:] . B[t][:]
// with A = W1 (hidden x in_dim, K-major, the replica itself) and B = the batch
// rows of X (b x in_dim, K-major, gathered by the batch permutation, R10).
//
// fp32 accuracy from TF32 tensor cores ("3xTF32"): every operand is split as
// x = hi + lo with hi = rna_tf32(x), lo = rna_tf32(x - hi), and
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi  (error per product <= ~2^-20.4 |a b|;
// the dropped lo*lo term and both lo roundings).  A fourth MMA accumulates
// |A_hi| |B_hi|, the bound sum |w x| that R18's ReLU-mask decision needs: where
// |a1| <= 2^-12 * 1.004 * (sum |w x| + |b1|) the sign is not certain at this
// accuracy and the pre-activation is recomputed with the double-float Dot2 of
// the SIMT kernel (warp-cooperative, rare), exactly as mlp_hidden_kernel does.
//
// Launch: one cluster of nks <= 8 CTAs per (learner, 128-unit M tile); CTA q of
// the cluster owns K range [128 q, 128 q + 128).  Per CTA:
//   1. TMA (3-D tensor map over W [r][hidden][in_dim], SWIZZLE_128B) brings its
//      128 x 128 fp32 W1 tile into shared memory as four 128 x 32 boxes, while
//      the threads gather the 16 batch rows' K slice from global memory and
//      write B_hi / B_lo / |B_hi| in the same swizzled K-major layout;
//   2. the threads split A in place (hi) and into A_lo / |A_hi|;
//   3. one thread issues 4 tcgen05.mma.kind::tf32 (M128 N16 K8) per K step into
//      two TMEM accumulators (D: 16 columns, |.| bound: 16 columns) and commits
//      to an mbarrier;
//   4. warps 0-3 read their 32 TMEM lanes (tcgen05.ld.32x32b.x16) and park the
//      partial tiles in shared memory; after a cluster barrier, each CTA sums
//      1/nks of the tile's nks partials in rank order through distributed shared
//      memory (fixed order: deterministic), adds b1, decides the mask certainty
//      and writes A1
//      [r][b][hidden] (double-float, lo = 0 unless recomputed) -- the same output
//      contract as mlp_hidden_kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <mutex>

#include "sma_dot2.cuh"
#include "sma_pdl.cuh"
#include "sma_internal.h"

namespace sma {
namespace {

constexpr int kTcThreads = 256;
constexpr int kTcM = 128;          // UMMA M (hidden units per CTA)
constexpr int kTcN = 16;           // UMMA N (batch rows, zero-padded)
constexpr int kTcKC = 128;         // K per CTA of the cluster
constexpr int kBoxK = 32;          // 128-byte swizzle atom width in fp32
constexpr int kABox = kTcM * kBoxK * 4;    // 16 KB
constexpr int kBBox = kTcN * kBoxK * 4;    // 2 KB
constexpr int kABytes = 4 * kABox;         // 64 KB per A variant
constexpr int kBBytes = 4 * kBBox;         // 8 KB per B variant
constexpr int kSmemBytes = 3 * kABytes + 3 * kBBytes + 1024 /* align */ + 256 /* ctl */;
constexpr int kMaxCluster = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// mbarrier wait with a watchdog: traps after ~5 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint64_t t0 = global_ns();
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) break;
    if (global_ns() - t0 > 5000000000ull) __trap();
  }
}
// UMMA shared-memory descriptor: K-major, SWIZZLE_128B (8-row x 128-byte atoms,
// SBO = 1024 B between 8-row groups, LBO unused = 1), sm_100 version bit.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
// Instruction descriptor: kind::tf32, D fp32, A/B tf32, both K-major, M = 128, N = 16.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                            ((uint32_t)(kTcM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
// Byte offset of element (row, k) of a [rows][32] fp32 box in the 128-byte
// swizzle (Swizzle<3,4,3>: 16-byte chunk index XOR row mod 8).
__device__ __forceinline__ uint32_t sw128_off(int row, int k) {
  return (uint32_t)row * 128u + ((uint32_t)(((k >> 2) ^ (row & 7))) << 4) + (uint32_t)(k & 3) * 4u;
}

using dot2::f2;
using dot2::dot2_step;
using dot2::f2_add;

__global__ void __launch_bounds__(kTcThreads, 1) mlp_hidden_tc_kernel(
    const __grid_constant__ CUtensorMap tmW1, const float* __restrict__ X,
    const int32_t* __restrict__ perm, int64_t pos0, int b, int in_dim, int hidden,
    const float* __restrict__ Wall, int64_t ld, int j0, float2* __restrict__ A1) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128-byte swizzle atoms, keeping the pointer
  // derived from smem_raw (so accesses compile to LDS/STS, not generic LD/ST)
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* Ahi = reinterpret_cast<float*>(sm);
  float* Alo = reinterpret_cast<float*>(sm + kABytes);
  float* Aab = reinterpret_cast<float*>(sm + 2 * kABytes);
  uint8_t* Bb = sm + 3 * kABytes;                      // B_hi | B_lo | |B_hi|
  uint8_t* ctl = Bb + 3 * kBBytes;
  uint64_t* bar_tma = reinterpret_cast<uint64_t*>(ctl);
  uint64_t* bar_mma = bar_tma + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ctl + 16);
  int* rows = reinterpret_cast<int*>(ctl + 32);        // [kTcN]
  int* nfb = reinterpret_cast<int*>(ctl + 32 + 4 * kTcN);
  int* fb = reinterpret_cast<int*>(Bb);                // fallback list (B is free after the MMAs)

  const int q = blockIdx.x;                 // cluster rank = K slice
  const int nks = gridDim.x;
  const int mt = blockIdx.y, slot = blockIdx.z;
  const int k0 = q * kTcKC;
  const int kb = min(kTcKC, in_dim - k0);
  const int nbox = (kb + kBoxK - 1) / kBoxK;
  const int nstep = (kb + 7) / 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // PDL: wait for the previous kernel first (W1 is the replica it wrote; moving
  // the X loads before the wait measured ~3 % slower at k = 16).  Prologue,
  // overlapped: lane 0 of warp 1 initialises the barriers and issues the TMA
  // boxes of W1 at once; every thread starts its X loads (reading the batch
  // permutation itself); warp 0 allocates TMEM meanwhile.
  pdl::wait_and_release();
  if (threadIdx.x == 32) {  // 1. the W1 tile: nbox TMA boxes of 128 rows x 32 fp32
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar_tma)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar_mma)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar_tma)),
                 "r"((uint32_t)(nbox * kABox))
                 : "memory");
    for (int bx = 0; bx < nbox; ++bx)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
          "%3, %4}], [%5];" ::"r"(smem_u32(Ahi) + (uint32_t)(bx * kABox)),
          "l"(&tmW1), "r"(k0 + bx * kBoxK), "r"(mt * kTcM), "r"(slot), "r"(smem_u32(bar_tma))
          : "memory");
  }
  if (threadIdx.x == 0) *nfb = 0;
  const int32_t* prow = perm + pos0 + (int64_t)(j0 + slot) * b;
  if (threadIdx.x < kTcN) rows[threadIdx.x] = threadIdx.x < b ? prow[threadIdx.x] : -1;
  // 1b. B = the batch rows' K slice, split and swizzled by the threads: the
  //     16 x 128 slice is 512 float4, two per thread, both loads in flight
  //     before any use (the rows are scattered over X: one HBM latency)
  constexpr int kB4 = kTcN * kTcKC / 4 / kTcThreads;
  float4 xv[kB4];
#pragma unroll
  for (int i = 0; i < kB4; ++i) {
    const int e4 = threadIdx.x + i * kTcThreads;
    const int n = e4 / (kTcKC / 4), kk = (e4 - n * (kTcKC / 4)) * 4;
    const int row = n < b ? __ldg(prow + n) : -1;
    xv[i] = (row >= 0 && kk < kb)
                ? __ldg(reinterpret_cast<const float4*>(X + (int64_t)row * in_dim + k0 + kk))
                : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (warp == 0) {  // 32 TMEM columns: D at +0, the |.| bound at +16
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
#pragma unroll
  for (int i = 0; i < kB4; ++i) {
    const int e4 = threadIdx.x + i * kTcThreads;
    const int n = e4 / (kTcKC / 4), kk = (e4 - n * (kTcKC / 4)) * 4;
    // 4 consecutive k of one row stay in one 16-byte chunk of the swizzle
    const uint32_t off = (uint32_t)(kk / kBoxK) * kBBox + sw128_off(n, kk % kBoxK);
    const float x[4] = {xv[i].x, xv[i].y, xv[i].z, xv[i].w};
    float4 h, l, a;
    float* hp = &h.x; float* lp = &l.x; float* ap = &a.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      hp[c] = rna_tf32(x[c]);
      lp[c] = rna_tf32(__fsub_rn(x[c], hp[c]));
      ap[c] = fabsf(hp[c]);
    }
    *reinterpret_cast<float4*>(Bb + off) = h;
    *reinterpret_cast<float4*>(Bb + kBBytes + off) = l;
    *reinterpret_cast<float4*>(Bb + 2 * kBBytes + off) = a;
  }
  // 2. split A in place (the swizzle is a function of the address, so the
  //    element-wise transform keeps the layout)
  mbar_wait(bar_tma, 0);
  for (int i = threadIdx.x; i < nbox * (kABox / 16); i += kTcThreads) {
    const float4 x = reinterpret_cast<const float4*>(Ahi)[i];
    float4 h, l, a;
    h.x = rna_tf32(x.x); h.y = rna_tf32(x.y); h.z = rna_tf32(x.z); h.w = rna_tf32(x.w);
    l.x = rna_tf32(__fsub_rn(x.x, h.x)); l.y = rna_tf32(__fsub_rn(x.y, h.y));
    l.z = rna_tf32(__fsub_rn(x.z, h.z)); l.w = rna_tf32(__fsub_rn(x.w, h.w));
    a.x = fabsf(h.x); a.y = fabsf(h.y); a.z = fabsf(h.z); a.w = fabsf(h.w);
    reinterpret_cast<float4*>(Ahi)[i] = h;
    reinterpret_cast<float4*>(Alo)[i] = l;
    reinterpret_cast<float4*>(Aab)[i] = a;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
  __syncthreads();

  if (threadIdx.x == 0) {  // 3. the MMAs of this K slice
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t a0 = smem_u32(Ahi), al0 = smem_u32(Alo), aa0 = smem_u32(Aab);
    const uint32_t b0 = smem_u32(Bb), bl0 = b0 + kBBytes, ba0 = b0 + 2 * kBBytes;
    for (int s = 0; s < nstep; ++s) {
      const uint32_t oa = (uint32_t)(s >> 2) * kABox + (uint32_t)(s & 3) * 32u;
      const uint32_t ob = (uint32_t)(s >> 2) * kBBox + (uint32_t)(s & 3) * 32u;
      const uint32_t acc = s > 0;
      mma_tf32(tmem, sw128_desc(a0 + oa), sw128_desc(b0 + ob), acc);       // hi hi
      mma_tf32(tmem, sw128_desc(a0 + oa), sw128_desc(bl0 + ob), 1u);       // hi lo
      mma_tf32(tmem, sw128_desc(al0 + oa), sw128_desc(b0 + ob), 1u);       // lo hi
      mma_tf32(tmem + 16, sw128_desc(aa0 + oa), sw128_desc(ba0 + ob), acc);  // |hi| |hi|
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar_mma))
                 : "memory");
  }
  mbar_wait(bar_mma, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // 4. TMEM -> registers -> this CTA's partial tile red[2][128][16] (A_hi region)
  float* red = Ahi;
  if (warp < 4) {
    uint32_t v[32];
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(ta));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
          "=r"(v[30]), "=r"(v[31])
        : "r"(ta + 16u));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = warp * 32 + lane;
#pragma unroll
    for (int t = 0; t < kTcN; ++t) {
      red[m * kTcN + t] = __uint_as_float(v[t]);
      red[kTcM * kTcN + m * kTcN + t] = __uint_as_float(v[16 + t]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");

  // every CTA of the cluster reduces an equal share of the 128 x 16 tile: for
  // each element, the nks partials are loaded from the peers' shared memory
  // (all loads in flight, then summed in rank order: deterministic), then the
  // bias, R18's certainty test, and A1
  {
    const float* W1 = Wall + (int64_t)slot * ld;
    const float* b1 = W1 + (int64_t)hidden * in_dim;
    const uint32_t red_l = smem_u32(red);
    const int per = (kTcM * kTcN + nks - 1) / nks;
    const int e1 = min((q + 1) * per, kTcM * kTcN);
    for (int e = q * per + threadIdx.x; e < e1; e += kTcThreads) {
      float v[kMaxCluster], va[kMaxCluster];
#pragma unroll
      for (int p = 0; p < kMaxCluster; ++p) {
        if (p < nks) {
          uint32_t ra;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(red_l + 4u * e), "r"(p));
          asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v[p]) : "r"(ra) : "memory");
          asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(va[p]) : "r"(ra + 4u * kTcM * kTcN)
                       : "memory");
        }
      }
      float s = 0.f, sa = 0.f;
#pragma unroll
      for (int p = 0; p < kMaxCluster; ++p) {
        if (p < nks) {
          s = __fadd_rn(s, v[p]);
          sa = __fadd_rn(sa, va[p]);
        }
      }
      const int m = e / kTcN, t = e - m * kTcN;
      if (t >= b) continue;
      const int u = mt * kTcM + m;
      const float bias = b1[u];
      const float a = __fadd_rn(s, bias);
      const float bound = ldexpf(__fmul_rn(__fadd_rn(sa, fabsf(bias)), 1.004f), -12);
      if (fabsf(a) <= bound) {
        const int i = atomicAdd(nfb, 1);
        fb[i] = (t << 16) | u;
      } else {
        A1[((int64_t)slot * b + t) * hidden + u] = make_float2(a, 0.f);
      }
    }
  }
  // no CTA may leave (or reuse its partial tile) while a peer still reads it
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  {  // near a ReLU kink: the Dot2 pre-activation (~2^-48), one warp per entry
    const float* W1 = Wall + (int64_t)slot * ld;
    const float* b1 = W1 + (int64_t)hidden * in_dim;
    const int n = *nfb;
    for (int i = warp; i < n; i += kTcThreads / 32) {
      const int t = fb[i] >> 16, u = fb[i] & 0xFFFF;
      const float* w = W1 + (int64_t)u * in_dim;
      const float* x = X + (int64_t)rows[t] * in_dim;
      f2 acc = {0.f, 0.f};
      for (int f = lane; f < in_dim; f += 32) dot2_step(acc, __ldg(w + f), __ldg(x + f));
      acc = f2_add(dot2::warp_sum(acc), f2{b1[u], 0.f});
      if (lane == 0) A1[((int64_t)slot * b + t) * hidden + u] = make_float2(acc.hi, acc.lo);
    }
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}


// ------------------------------------------------------------------- dW1
// dW1[u][f] = (1/b) sum_t da1[t][u] x_t[f] (back-propagation into layer 1,
// PAPER.md:249-256; batch mean, Eq. 2) as D[u][f] = A[u][:] . B[f][:] with
// M = 128 units, N = 112 features, K = the batch (zero-padded to 32, one
// 128-byte swizzle atom): A[u][t] = da1[t][u], B[f][t] = x_t[f], both staged
// K-major by the threads (a transpose of the tiny da1 / X tiles), 3xTF32 split,
// three tcgen05.mma per K step into 112 TMEM columns; the epilogue reads 16
// columns per tcgen05.ld and writes rows of dW1 with 128-bit stores.  No cluster:
// K is the batch, so each CTA owns a whole output tile.  db1 on the f0 = 0 CTAs.
constexpr int kW1N = 112;                              // UMMA N (features per CTA)
constexpr int kW1ABytes = kTcM * kBoxK * 4;            // 16 KB
constexpr int kW1BBytes = kW1N * kBoxK * 4;            // 14 KB
constexpr int kW1Smem = 2 * kW1ABytes + 2 * kW1BBytes + 1024 + 64;
constexpr uint32_t kIdescW1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kW1N >> 3) << 17) |
                              ((uint32_t)(kTcM >> 4) << 24);

__global__ void __launch_bounds__(kTcThreads) mlp_w1_tc_kernel(
    const float* __restrict__ X, const int32_t* __restrict__ perm, int64_t pos0, int b, int in_dim,
    int hidden, int j0, int64_t ld, const float* __restrict__ DA, float* __restrict__ Gall) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* Ah = sm;
  uint8_t* Al = sm + kW1ABytes;
  uint8_t* Bh = sm + 2 * kW1ABytes;
  uint8_t* Bl = Bh + kW1BBytes;
  uint8_t* ctl = Bl + kW1BBytes;
  uint64_t* bar_mma = reinterpret_cast<uint64_t*>(ctl);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ctl + 8);
  const int f0 = blockIdx.x * kW1N, mt = blockIdx.y, slot = blockIdx.z;
  const int u0 = mt * kTcM;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* prow = perm + pos0 + (int64_t)(j0 + slot) * b;
  const float* da = DA + (int64_t)slot * b * hidden;

  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar_mma)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // 128 TMEM columns (>= N = 112)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // A[u][t] = da1[t][u0 + u] (coalesced along u), B[f][t] = x_t[f0 + f]; every
  // thread issues all of its loads before the first use (one memory latency)
  constexpr int kAE = kTcM * kBoxK / kTcThreads, kBE = kW1N * kBoxK / kTcThreads;
  static_assert(kAE * kTcThreads == kTcM * kBoxK && kBE * kTcThreads == kW1N * kBoxK, "tiling");
  // all loads after the PDL wait, in flight together (da1 is the head kernel's
  // output; issuing the X loads before the wait measured slower: a second
  // serialised latency once the head kernel has already completed)
  pdl::wait_and_release();
  float av[kAE], bv[kBE];
#pragma unroll
  for (int i = 0; i < kAE; ++i) {
    const int e = threadIdx.x + i * kTcThreads;
    const int t = e / kTcM, u = e - t * kTcM;
    av[i] = t < b ? da[(int64_t)t * hidden + u0 + u] : 0.f;
  }
#pragma unroll
  for (int i = 0; i < kBE; ++i) {
    const int e = threadIdx.x + i * kTcThreads;
    const int t = e / kW1N, f = e - t * kW1N;
    bv[i] = (t < b && f0 + f < in_dim) ? __ldg(X + (int64_t)__ldg(prow + t) * in_dim + f0 + f) : 0.f;
  }
#pragma unroll
  for (int i = 0; i < kAE; ++i) {
    const int e = threadIdx.x + i * kTcThreads;
    const int t = e / kTcM, u = e - t * kTcM;
    const float h = rna_tf32(av[i]);
    const uint32_t off = sw128_off(u, t);
    *reinterpret_cast<float*>(Ah + off) = h;
    *reinterpret_cast<float*>(Al + off) = rna_tf32(__fsub_rn(av[i], h));
  }
#pragma unroll
  for (int i = 0; i < kBE; ++i) {
    const int e = threadIdx.x + i * kTcThreads;
    const int t = e / kW1N, f = e - t * kW1N;
    const float h = rna_tf32(bv[i]);
    const uint32_t off = sw128_off(f, t);
    *reinterpret_cast<float*>(Bh + off) = h;
    *reinterpret_cast<float*>(Bl + off) = rna_tf32(__fsub_rn(bv[i], h));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(Ah), al0 = smem_u32(Al), b0 = smem_u32(Bh), bl0 = smem_u32(Bl);
    const int nstep = (b + 7) / 8;
    for (int s = 0; s < nstep; ++s) {
      const uint32_t o = (uint32_t)s * 32u;
      const uint32_t acc = s > 0;
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                   "l"(sw128_desc(a0 + o)), "l"(sw128_desc(b0 + o)), "r"(kIdescW1), "r"(acc));
      asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(tmem),
                   "l"(sw128_desc(a0 + o)), "l"(sw128_desc(bl0 + o)), "r"(kIdescW1));
      asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n" ::"r"(tmem),
                   "l"(sw128_desc(al0 + o)), "l"(sw128_desc(b0 + o)), "r"(kIdescW1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar_mma))
                 : "memory");
  }
  float* G = Gall + (int64_t)slot * ld;
  const float fb = (float)b;
  if (blockIdx.x == 0 && threadIdx.x < kTcM) {  // db1 = (1/b) sum_t da1[t][u]
    float s = 0.f;
    for (int t = 0; t < b; ++t) s = __fadd_rn(s, da[(int64_t)t * hidden + u0 + threadIdx.x]);
    G[(int64_t)hidden * in_dim + u0 + threadIdx.x] = __fdiv_rn(s, fb);
  }
  mbar_wait(bar_mma, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads TMEM lanes 32 (w % 4) .. +31 (one unit row per lane), column
  // chunks w / 4, w / 4 + 2, ... of 16
  const int u = u0 + (warp & 3) * 32 + lane;
  float* grow = G + (int64_t)u * in_dim;
  for (int c = warp >> 2; c < kW1N / 16; c += 2) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(c * 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int fc = f0 + c * 16;
    if (fc + 16 <= in_dim) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        reinterpret_cast<float4*>(grow + fc)[i] =
            make_float4(__fdiv_rn(__uint_as_float(v[4 * i + 0]), fb),
                        __fdiv_rn(__uint_as_float(v[4 * i + 1]), fb),
                        __fdiv_rn(__uint_as_float(v[4 * i + 2]), fb),
                        __fdiv_rn(__uint_as_float(v[4 * i + 3]), fb));
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (fc + i < in_dim) grow[fc + i] = __fdiv_rn(__uint_as_float(v[i]), fb);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// ---------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

// SMA_MLP_TC: 0 = SIMT kernels, 1 = both GEMMs on the tensor cores, "hidden" =
// layer 1 only, "w1" = dW1 only; unset = by learners per GPU (tc_wanted()).
// Bits: 1 = layer 1, 2 = dW1; -1 = unset.
int tc_policy() {
  static const int p = [] {
    const char* e = getenv("SMA_MLP_TC");
    if (!e) return -1;
    if (e[0] == 'h') return 1;
    if (e[0] == 'w') return 2;
    return e[0] == '0' ? 0 : 3;
  }();
  return p;
}

// Default thresholds, measured (profiles/r01_mlp_tc_sweep2.txt, MLP rounds/s,
// b = 16, PDL on, SIMT vs tensor cores per GEMM): layer 1 on tcgen05 loses while
// the SIMT kernel's 64 CTAs per learner still fit one wave (k = 4: 38.7k SIMT vs
// 34.4k; k = 8: 27.1k vs 24.2k) and wins from r = 12 on (20.9k vs 20.6k; k = 16:
// 16.8k vs 16.5k; k = 32: 10.2k vs 9.8k). The SIMT dW1 kernel (4 features per
// thread) is at least as fast as the tensor-core one at every k measured (4-32),
// so dW1 takes the tensor cores only when forced (SMA_MLP_TC=1 / w1).
constexpr int kTcHiddenMinR = 12;         // layer 1 (launch_mlp_grad also keeps the SIMT
                                          // kernel when its grid fills >= 85 % of a wave)
constexpr int kTcW1MinR = 1 << 30;        // dW1: never by default
bool tc_wanted(int bit, int r) {
  const int pol = tc_policy();
  if (pol >= 0) return (pol & bit) != 0;
  return r >= (bit == 1 ? kTcHiddenMinR : kTcW1MinR);
}
}  // namespace

int mlp_tc_policy() { return tc_policy(); }

// Returns cudaErrorNotSupported (nothing launched) when the policy or the shape
// keeps layer 1 on the SIMT kernel (tc_policy(); b > 16, hidden % 128, in_dim % 4,
// in_dim > 1024, or no tensor-map encoder); the caller then launches that kernel.
cudaError_t launch_mlp_hidden_tc(const float* X, const int32_t* perm, int64_t pos0, int b,
                                 int in_dim, int hidden, const float* W, int64_t ld, int r, int j0,
                                 float2* A1, cudaStream_t s) {
  if (!tc_wanted(1, r) || b > kTcN || b < 1 || hidden % kTcM != 0 || hidden > 65535 ||
      (in_dim & 3) != 0 || in_dim > kMaxCluster * kTcKC || r < 1)
    return cudaErrorNotSupported;
  std::call_once(g_encode_once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
            cudaSuccess && qr == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!g_encode) return cudaErrorNotSupported;
  // W [r][ld] with W1 = [hidden][in_dim] at the start of each replica; the
  // encoded map is cached per issuing thread (re-encoded when W or a shape changes)
  struct MapCache {
    const float* W = nullptr;
    int64_t ld = 0;
    int r = 0, in_dim = 0, hidden = 0;
    CUtensorMap tm;
  };
  thread_local MapCache mc;
  if (mc.W != W || mc.ld != ld || mc.r != r || mc.in_dim != in_dim || mc.hidden != hidden) {
    const cuuint64_t dims[3] = {(cuuint64_t)in_dim, (cuuint64_t)hidden, (cuuint64_t)r};
    const cuuint64_t strides[2] = {(cuuint64_t)in_dim * 4, (cuuint64_t)ld * 4};
    const cuuint32_t box[3] = {kBoxK, kTcM, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    mc.W = nullptr;
    if (g_encode(&mc.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(W), dims, strides,
                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorNotSupported;
    mc.W = W;
    mc.ld = ld;
    mc.r = r;
    mc.in_dim = in_dim;
    mc.hidden = hidden;
  }
  const CUtensorMap& tm = mc.tm;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(mlp_hidden_tc_kernel), kSmemBytes);
  if (e != cudaSuccess) return e;
  const int nks = (in_dim + kTcKC - 1) / kTcKC;
  return pdl::launch(mlp_hidden_tc_kernel, dim3(nks, hidden / kTcM, r), dim3(kTcThreads),
                     (size_t)kSmemBytes, s, nks, tm, X, perm, pos0, b, in_dim, hidden, W, ld, j0, A1);
}

}  // namespace sma

namespace sma {
// dW1 on tcgen05; cudaErrorNotSupported (nothing launched) when the policy or
// the shape keeps it on the SIMT kernel (b > 32, hidden % 128, in_dim % 4).
cudaError_t launch_mlp_w1_tc(const float* X, const int32_t* perm, int64_t pos0, int b, int in_dim,
                             int hidden, int j0, int64_t ld, int r, const float* DA, float* G,
                             cudaStream_t s) {
  if (!tc_wanted(2, r) || b < 1 || b > kBoxK || hidden % kTcM != 0 ||
      (in_dim & 3) != 0 || r < 1)
    return cudaErrorNotSupported;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(mlp_w1_tc_kernel), kW1Smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((in_dim + kW1N - 1) / kW1N, hidden / kTcM, r);
  return pdl::launch(mlp_w1_tc_kernel, grid, dim3(kTcThreads), (size_t)kW1Smem, s, 1, X, perm, pos0, b,
                     in_dim, hidden, j0, ld, DA, G);
}
}  // namespace sma
