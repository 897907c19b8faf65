// sma_pdl.cuh -- programmatic dependent launch (PDL, sm_90+) for the kernels of
// a round.  Consecutive kernels on one stream normally start only after the
// front end sees the previous grid complete and launches the next one (~1 us
// per boundary on B200, and back-to-back small rounds were quantised to 4.1 us
// steps).  Launched with cudaLaunchAttributeProgrammaticStreamSerialization, a
// kernel's CTAs become resident while the previous grid drains; each kernel
// calls pdl::wait() before its first access to memory a previous kernel may
// write (griddepcontrol.wait returns once the previous grid has completed and
// its writes are visible; without the attribute it is a no-op) and
// pdl::release() to let the next kernel launch early.
// Measured (bench.py, profiles/r01_pdl.txt): C2 122k -> 154k rounds/s, C3 81k ->
// 96k, C1 60k -> 69k.  SMA_PDL=0 disables it.
#pragma once
#include <cuda_runtime.h>
#include <stdlib.h>

namespace sma {
namespace pdl {

__device__ __forceinline__ void wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void release() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void wait_and_release() {
  wait();
  release();
}

inline bool enabled() {
  static const bool on = [] {
    const char* e = getenv("SMA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// kernel<<<grid, block, smem, s>>>(args...) with the PDL attribute (and, if
// cluster_x > 1, a (cluster_x, 1, 1) thread-block cluster).
template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = n ? at : nullptr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace pdl
}  // namespace sma
