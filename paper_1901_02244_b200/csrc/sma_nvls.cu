// sma_nvls.cu -- NEXT-1: the inter-GPU z-sync (a6 + a7 + a8) as ONE kernel over
// NVSwitch multicast memory (NVLS), replacing NCCL reduce-scatter -> shard
// update -> all-gather.
//
// Every rank binds one physical allocation [flags | partial(s) | z[2]] to a
// multicast object.  Rank g then, for each float4 chunk of ITS shard:
//   S  = multimem.ld_reduce.add  (partial_mc + chunk)   -- the switch sums the
//                                                          chunk over all GPUs (a6)
//   z' = z + S + mu (z - z_prev)     (Mode A)            -- Alg. 1 line 13 (a7)
//   z' = z + alpha S + (mu - alpha k)(z - z_prev) (Mode B)
//   multimem.st (znext_mc + chunk, z')                  -- broadcast to all GPUs (a8)
// Per GPU and direction the links carry about 4 d bytes instead of the
// 2 x 4 d (n-1)/n of a ring reduce-scatter + all-gather.
// Two device-side barriers (multimem.red on a multicast flag, acquire-spin on
// the local copy) order "all partials written" before the loads and "all
// broadcasts landed" before the next round; the barrier targets are kept in
// device memory so the kernel can be replayed from a CUDA graph.  A barrier
// that does not complete within ~30 s traps (the process fails loudly
// instead of hanging the GPU).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <mutex>
#include <string>

#include "sma_internal.h"

namespace sma {

// ------------------------------------------------------- driver entry points
namespace {
struct DriverApi {
  bool tried = false, ok = false;
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle,
                               size_t, size_t, unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*,
                                      CUmulticastGranularity_flags) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                        unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*,
                                          CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle,
                                         CUmemAllocationHandleType, unsigned long long) = nullptr;
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*,
                                           CUmemAllocationHandleType) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
};
DriverApi g_drv;

template <typename F>
bool bind_sym(F*& f, const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  f = reinterpret_cast<F*>(p);
  return true;
}

void drv_load_once();
std::once_flag g_drv_once;
bool drv_load(std::string* err) {
  std::call_once(g_drv_once, drv_load_once);
  if (!g_drv.ok) *err = "CUDA driver multicast entry points unavailable";
  return g_drv.ok;
}

void drv_load_once() {
  g_drv.tried = true;
  bool ok = bind_sym(g_drv.DeviceGet, "cuDeviceGet") &&
            bind_sym(g_drv.DeviceGetAttribute, "cuDeviceGetAttribute") &&
            bind_sym(g_drv.MulticastCreate, "cuMulticastCreate") &&
            bind_sym(g_drv.MulticastAddDevice, "cuMulticastAddDevice") &&
            bind_sym(g_drv.MulticastBindMem, "cuMulticastBindMem") &&
            bind_sym(g_drv.MulticastUnbind, "cuMulticastUnbind") &&
            bind_sym(g_drv.MulticastGetGranularity, "cuMulticastGetGranularity") &&
            bind_sym(g_drv.MemCreate, "cuMemCreate") && bind_sym(g_drv.MemRelease, "cuMemRelease") &&
            bind_sym(g_drv.MemAddressReserve, "cuMemAddressReserve") &&
            bind_sym(g_drv.MemAddressFree, "cuMemAddressFree") &&
            bind_sym(g_drv.MemMap, "cuMemMap") && bind_sym(g_drv.MemUnmap, "cuMemUnmap") &&
            bind_sym(g_drv.MemSetAccess, "cuMemSetAccess") &&
            bind_sym(g_drv.MemGetAllocationGranularity, "cuMemGetAllocationGranularity") &&
            bind_sym(g_drv.MemExportToShareableHandle, "cuMemExportToShareableHandle") &&
            bind_sym(g_drv.MemImportFromShareableHandle, "cuMemImportFromShareableHandle") &&
            bind_sym(g_drv.GetErrorString, "cuGetErrorString");
  g_drv.ok = ok;
}

std::string cu_err(CUresult r, const char* what) {
  const char* s = nullptr;
  if (g_drv.GetErrorString) g_drv.GetErrorString(r, &s);
  return std::string(what) + " failed: " + (s ? s : "unknown CUDA driver error");
}

#define CU_CHECK(expr, what)                 \
  do {                                       \
    CUresult _r = (expr);                    \
    if (_r != CUDA_SUCCESS) {                \
      *err = cu_err(_r, what);               \
      return false;                          \
    }                                        \
  } while (0)

// ----------------------------------------- POSIX fd passing (SCM_RIGHTS)
// Abstract-namespace Unix sockets named after the rendezvous key: rank 0
// sends the exported multicast fd to every other rank.
std::string sock_name(const std::string& key, int rank) {
  return std::string("\0sma-nvls-", 10) + key + "-" + std::to_string(rank);
}

int uds_listen(const std::string& name) {
  int s = socket(AF_UNIX, SOCK_STREAM, 0);
  if (s < 0) return -1;
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  memcpy(a.sun_path, name.data(), name.size());
  socklen_t len = (socklen_t)(offsetof(sockaddr_un, sun_path) + name.size());
  if (bind(s, (sockaddr*)&a, len) != 0 || listen(s, 4) != 0) {
    close(s);
    return -1;
  }
  return s;
}

bool uds_send_fd(const std::string& name, int fd) {
  for (int attempt = 0; attempt < 600; ++attempt) {  // up to ~60 s for the peer to listen
    int s = socket(AF_UNIX, SOCK_STREAM, 0);
    if (s < 0) return false;
    sockaddr_un a{};
    a.sun_family = AF_UNIX;
    memcpy(a.sun_path, name.data(), name.size());
    socklen_t len = (socklen_t)(offsetof(sockaddr_un, sun_path) + name.size());
    if (connect(s, (sockaddr*)&a, len) == 0) {
      char byte = 'x';
      iovec io{&byte, 1};
      char ctrl[CMSG_SPACE(sizeof(int))] = {};
      msghdr m{};
      m.msg_iov = &io;
      m.msg_iovlen = 1;
      m.msg_control = ctrl;
      m.msg_controllen = sizeof ctrl;
      cmsghdr* c = CMSG_FIRSTHDR(&m);
      c->cmsg_level = SOL_SOCKET;
      c->cmsg_type = SCM_RIGHTS;
      c->cmsg_len = CMSG_LEN(sizeof(int));
      memcpy(CMSG_DATA(c), &fd, sizeof(int));
      const bool ok = sendmsg(s, &m, 0) == 1;
      close(s);
      return ok;
    }
    close(s);
    usleep(100000);
  }
  return false;
}

int uds_recv_fd(int listen_sock) {
  int c = accept(listen_sock, nullptr, nullptr);
  if (c < 0) return -1;
  char byte;
  iovec io{&byte, 1};
  char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof ctrl;
  int fd = -1;
  if (recvmsg(c, &m, 0) == 1) {
    cmsghdr* h = CMSG_FIRSTHDR(&m);
    if (h && h->cmsg_type == SCM_RIGHTS) memcpy(&fd, CMSG_DATA(h), sizeof(int));
  }
  close(c);
  return fd;
}
}  // namespace

// ----------------------------------------------------------------- setup
bool nvls_supported(int device, std::string* err) {
  if (!drv_load(err)) return false;
  CUdevice dev;
  CU_CHECK(g_drv.DeviceGet(&dev, device), "cuDeviceGet");
  int mc = 0;
  CU_CHECK(g_drv.DeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev),
           "cuDeviceGetAttribute(MULTICAST_SUPPORTED)");
  if (!mc) {
    *err = "device does not support NVSwitch multicast (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED=0)";
    return false;
  }
  return true;
}

bool nvls_setup(NvlsRegion* R, int device, int rank, int world, size_t bytes, const std::string& key,
                const std::function<bool(std::string*)>& barrier, std::string* err) {
  if (!nvls_supported(device, err)) return false;
  CUdevice dev;
  CU_CHECK(g_drv.DeviceGet(&dev, device), "cuDeviceGet");
  R->dev = dev;
  CUmulticastObjectProp mp{};
  mp.numDevices = (unsigned)world;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  size_t gmc = 0, gph = 0;
  CU_CHECK(g_drv.MulticastGetGranularity(&gmc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED),
           "cuMulticastGetGranularity");
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  CU_CHECK(g_drv.MemGetAllocationGranularity(&gph, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
           "cuMemGetAllocationGranularity");
  size_t g = gmc > gph ? gmc : gph;
  R->size = (bytes + g - 1) / g * g;
  mp.size = R->size;

  // 1. the multicast object: created on rank 0, its fd sent to the others
  int lsock = -1;
  if (rank != 0 && world > 1) {
    lsock = uds_listen(sock_name(key, rank));
    if (lsock < 0) {
      *err = "cannot open the rendezvous socket";
      return false;
    }
  }
  if (!barrier(err)) {
    if (lsock >= 0) close(lsock);
    return false;
  }
  if (rank == 0) {
    CU_CHECK(g_drv.MulticastCreate(&R->mc, &mp), "cuMulticastCreate");
    R->have_mc = true;
    if (world > 1) {
      int fd = -1;
      CU_CHECK(g_drv.MemExportToShareableHandle(&fd, R->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
               "cuMemExportToShareableHandle");
      for (int p = 1; p < world; ++p)
        if (!uds_send_fd(sock_name(key, p), fd)) {
          close(fd);
          *err = "sending the multicast handle to rank " + std::to_string(p) + " failed";
          return false;
        }
      close(fd);
    }
  } else {
    const int fd = uds_recv_fd(lsock);
    close(lsock);
    if (fd < 0) {
      *err = "receiving the multicast handle failed";
      return false;
    }
    CUresult r = g_drv.MemImportFromShareableHandle(&R->mc, (void*)(uintptr_t)fd,
                                                    CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    close(fd);
    if (r != CUDA_SUCCESS) {
      *err = cu_err(r, "cuMemImportFromShareableHandle");
      return false;
    }
    R->have_mc = true;
  }
  CU_CHECK(g_drv.MulticastAddDevice(R->mc, dev), "cuMulticastAddDevice");
  if (!barrier(err)) return false;  // every device added before any binding

  // 2. local physical memory, mapped at a unicast VA and bound to the object
  CU_CHECK(g_drv.MemCreate(&R->phys, R->size, &ap, 0), "cuMemCreate");
  R->have_phys = true;
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU_CHECK(g_drv.MemAddressReserve(&R->uc, R->size, g, 0, 0), "cuMemAddressReserve");
  CU_CHECK(g_drv.MemMap(R->uc, R->size, 0, R->phys, 0), "cuMemMap");
  R->uc_mapped = true;
  CU_CHECK(g_drv.MemSetAccess(R->uc, R->size, &acc, 1), "cuMemSetAccess");
  CU_CHECK(g_drv.MulticastBindMem(R->mc, 0, R->phys, 0, R->size, 0), "cuMulticastBindMem");
  R->bound = true;
  // 3. the multicast VA
  CU_CHECK(g_drv.MemAddressReserve(&R->mcva, R->size, g, 0, 0), "cuMemAddressReserve(mc)");
  CU_CHECK(g_drv.MemMap(R->mcva, R->size, 0, R->mc, 0), "cuMemMap(mc)");
  R->mc_mapped = true;
  CU_CHECK(g_drv.MemSetAccess(R->mcva, R->size, &acc, 1), "cuMemSetAccess(mc)");
  if (cudaMemset((void*)R->uc, 0, R->size) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    *err = "zeroing the NVLS region failed";
    return false;
  }
  return barrier(err);  // every rank bound and zeroed before first use
}

void nvls_teardown(NvlsRegion* R) {
  if (!g_drv.ok) return;
  if (R->mc_mapped) g_drv.MemUnmap(R->mcva, R->size);
  if (R->mcva) g_drv.MemAddressFree(R->mcva, R->size);
  if (R->bound) g_drv.MulticastUnbind(R->mc, R->dev, 0, R->size);
  if (R->uc_mapped) g_drv.MemUnmap(R->uc, R->size);
  if (R->uc) g_drv.MemAddressFree(R->uc, R->size);
  if (R->have_phys) g_drv.MemRelease(R->phys);
  if (R->have_mc) g_drv.MemRelease(R->mc);
  *R = NvlsRegion{};
}

// ---------------------------------------------------------------- kernel
namespace {
constexpr int kNvlsThreads = 512;
constexpr int kNvlsUnroll = 4;

__device__ __forceinline__ float4 mm_ld_reduce(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void mm_st(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_signal(unsigned* flag_mc) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(flag_mc), "r"(1u) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned target) {
  const long long t0 = clock64();
  while ((int)(ld_acquire_sys(p) - target) < 0) {
    if (clock64() - t0 > 60000000000ll) __trap();  // ~30 s: a peer never arrived
    __nanosleep(64);
  }
}
__device__ __forceinline__ float4 ld_nc4(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ float4 ld_cg4(const float* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

template <int MODE>
__device__ __forceinline__ float4 shard_update(float4 zc, float4 s, float4 zp, const NvlsArgs& a) {
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

template <int MODE>
__global__ void __launch_bounds__(kNvlsThreads) zsync_nvls_kernel(const NvlsArgs a) {
  __shared__ unsigned s_targetA;
  if (threadIdx.x == 0) {
    const unsigned tA = a.expect[0] + (unsigned)a.n;
    if (blockIdx.x == 0) mm_signal(a.flag_mc + 0);  // barrier A: my partial is complete
    wait_geq(a.flag_uc + 0, tA);                     // ... and every GPU's
    s_targetA = tA;
  }
  __syncthreads();
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * kNvlsThreads;
  const int64_t base = a.off4;
  int64_t c = (int64_t)blockIdx.x * kNvlsThreads + threadIdx.x;
  for (; c + (kNvlsUnroll - 1) * stride < a.len4; c += kNvlsUnroll * stride) {
    float4 s[kNvlsUnroll];
#pragma unroll
    for (int u = 0; u < kNvlsUnroll; ++u) s[u] = mm_ld_reduce(a.part_mc + ((base + c + u * stride) << 2));
#pragma unroll
    for (int u = 0; u < kNvlsUnroll; ++u) {
      const int64_t p0 = (base + c + u * stride) << 2;
      const float4 zn = shard_update<MODE>(ld_nc4(a.z + p0), s[u], ld_cg4(a.zprev + p0), a);
      mm_st(a.znext_mc + p0, zn);
      bad |= !(isfinite(zn.x) && isfinite(zn.y) && isfinite(zn.z) && isfinite(zn.w));
    }
  }
  for (; c < a.len4; c += stride) {
    const int64_t p0 = (base + c) << 2;
    const float4 s = mm_ld_reduce(a.part_mc + p0);
    const float4 zn = shard_update<MODE>(ld_nc4(a.z + p0), s, ld_cg4(a.zprev + p0), a);
    mm_st(a.znext_mc + p0, zn);
    bad |= !(isfinite(zn.x) && isfinite(zn.y) && isfinite(zn.z) && isfinite(zn.w));
  }
  if (a.nonfinite && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.nonfinite, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // my broadcasts before my arrival
    const unsigned prev = atomicAdd(a.done_ctr, 1u);
    if (prev == gridDim.x - 1) {  // the last CTA of this GPU closes the round
      __threadfence_system();
      *a.done_ctr = 0;
      const unsigned tB = a.expect[1] + (unsigned)a.n;
      mm_signal(a.flag_mc + 1);   // barrier B: my shard has landed everywhere
      wait_geq(a.flag_uc + 1, tB);
      a.expect[0] = s_targetA;
      a.expect[1] = tB;
      __threadfence();
    }
  }
}
}  // namespace

cudaError_t launch_zsync_nvls(int mode, const NvlsArgs& a, int num_ctas, cudaStream_t s) {
  const int64_t want = (a.len4 + kNvlsThreads - 1) / kNvlsThreads;
  int grid = (int)(want < num_ctas ? want : num_ctas);
  if (grid < 1) grid = 1;
  if (mode == kPartialA)
    zsync_nvls_kernel<kPartialA><<<grid, kNvlsThreads, 0, s>>>(a);
  else
    zsync_nvls_kernel<kPartialB><<<grid, kNvlsThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sma
