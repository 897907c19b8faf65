// sma_bulk.cuh -- shared-memory staging with 1-D TMA bulk copies (sm_90+/sm_100a).
//
// The learner kernels stage a handful of contiguous spans (batch rows of X, a
// block of weight rows, a scratch tile) into shared memory before computing.
// A thread-per-element copy loop serialises one global round trip per
// iteration (ncu: the stall sits on the STS after each load); here one thread
// issues every span as `cp.async.bulk` (SASS UBLKCP) completing on a single
// mbarrier, and the CTA waits once.  Spans that are not 16-byte aligned (or not
// a multiple of 16 bytes) fall back to a cooperative copy.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sma {
namespace bulk {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ bool aligned16(const void* p, size_t bytes) {
  return ((reinterpret_cast<uintptr_t>(p) | bytes) & 15u) == 0;
}
__device__ __forceinline__ void bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void copy(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Stage, by the whole CTA (every thread must call; it synchronises):
//   rows:  nrows rows of `row_floats` floats, row t taken from
//          src + row_idx[t] * stride + col   (row_idx in shared memory)
//          into dst_rows + t * row_floats;
//   span:  n_span contiguous floats src_span -> dst_span (n_span may be 0).
// `bar` is a shared mbarrier used once per call; pass init = true on its first
// use and alternate `phase` (0, 1, 0, ...) on later ones.  Falls back to a
// cooperative copy when a span is not 16-byte aligned / sized.  Returns whether
// the barrier was used (uniform across the CTA), so a caller staging twice
// knows the next call's phase / init.
__device__ __forceinline__ bool stage_rows_span(float* dst_rows, const float* src, const int* row_idx,
                                                int nrows, int row_floats, int64_t stride, int col,
                                                float* dst_span, const float* src_span, int n_span,
                                                uint64_t* bar, uint32_t phase, bool init) {
  const uint32_t rb = 4u * (uint32_t)row_floats, sb = 4u * (uint32_t)n_span;
  const bool ok = nrows == 0 ||
                  (aligned16(src + col, rb) && ((stride * 4) & 15) == 0 && aligned16(dst_rows, 0));
  const bool ok2 = n_span == 0 || (aligned16(src_span, sb) && aligned16(dst_span, 0));
  if (ok && ok2) {
    if (threadIdx.x == 0) {
      if (init) bar_init(bar);
      expect_tx(bar, rb * (uint32_t)nrows + sb);
      for (int t = 0; t < nrows; ++t)
        copy(dst_rows + (int64_t)t * row_floats, src + (int64_t)row_idx[t] * stride + col, rb, bar);
      if (n_span) copy(dst_span, src_span, sb, bar);
    }
    __syncthreads();
    wait(bar, phase);
    return true;
  } else {
    for (int q = threadIdx.x; q < nrows * row_floats; q += blockDim.x) {
      const int t = q / row_floats, f = q - t * row_floats;
      dst_rows[q] = src[(int64_t)row_idx[t] * stride + col + f];
    }
    for (int q = threadIdx.x; q < n_span; q += blockDim.x) dst_span[q] = src_span[q];
    __syncthreads();
    return false;
  }
}

// Stage a [nrows][nf] tile of rows row_idx[t] (shared memory), columns
// [col, col + nf), of a row-major matrix with `stride` floats per row into
// dst [nrows][nf], by the whole CTA with one 16-byte load per thread and
// element group (no synchronisation inside; the caller syncs).  For narrow
// tiles this beats one TMA bulk copy per short row issued by a single thread
// (MLP dW1: 16 rows x 256 B per CTA).  Scalar fallback when not 16-byte aligned.
__device__ __forceinline__ void load_tile(float* dst, const float* src, const int* row_idx,
                                          int nrows, int nf, int64_t stride, int col) {
  const bool vec = ((nf | col) & 3) == 0 && ((stride & 3) == 0) &&
                   ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (vec) {
    const int n4 = nf >> 2;
    for (int q = threadIdx.x; q < nrows * n4; q += blockDim.x) {
      const int t = q / n4, c = q - t * n4;
      reinterpret_cast<float4*>(dst)[q] =
          __ldg(reinterpret_cast<const float4*>(src + (int64_t)row_idx[t] * stride + col) + c);
    }
  } else {
    for (int q = threadIdx.x; q < nrows * nf; q += blockDim.x) {
      const int t = q / nf, f = q - t * nf;
      dst[q] = __ldg(src + (int64_t)row_idx[t] * stride + col + f);
    }
  }
}

}  // namespace bulk
}  // namespace sma
