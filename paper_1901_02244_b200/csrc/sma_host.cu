// sma_host.cu -- libsma host-side pieces with no device state: error messages,
// the NCCL binding, and the pure bookkeeping functions of the ABI
// (sma_plan_*, Alg. 2's sma_autotune_step).  These are independent of the
// oracle's implementation; tests compare the two bit for bit.
#include <dlfcn.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "sma_host.h"
#include "sma_internal.h"

using namespace sma;

// ------------------------------------------------------------------ errors
namespace {
thread_local std::string g_last_error;
}

sma_status sma::fail(sma_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

extern "C" const char* sma_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------ NCCL (dlopen'ed)
namespace sma {
NcclApi g_nccl;

bool nccl_load_once();
std::once_flag g_nccl_once;
bool nccl_load() {
  std::call_once(g_nccl_once, [] { nccl_load_once(); });
  return g_nccl.ok;
}

bool nccl_load_once() {
  g_nccl.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    g_nccl.why = dlerror() ? dlerror() : "libnccl.so.2 not found";
    return false;
  }
#define BIND(field, sym)                                                       \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, sym));      \
  if (!g_nccl.field) {                                                         \
    g_nccl.why = std::string("missing symbol ") + sym;                         \
    return false;                                                              \
  }
  BIND(GetUniqueId, "ncclGetUniqueId");
  BIND(CommInitRank, "ncclCommInitRank");
  BIND(CommDestroy, "ncclCommDestroy");
  BIND(CommAbort, "ncclCommAbort");
  BIND(ReduceScatter, "ncclReduceScatter");
  BIND(AllGather, "ncclAllGather");
  BIND(AllReduce, "ncclAllReduce");
  BIND(GetErrorString, "ncclGetErrorString");
#undef BIND
  g_nccl.MemAlloc = reinterpret_cast<decltype(g_nccl.MemAlloc)>(dlsym(h, "ncclMemAlloc"));
  g_nccl.MemFree = reinterpret_cast<decltype(g_nccl.MemFree)>(dlsym(h, "ncclMemFree"));
  g_nccl.CommRegister = reinterpret_cast<decltype(g_nccl.CommRegister)>(dlsym(h, "ncclCommRegister"));
  g_nccl.CommDeregister =
      reinterpret_cast<decltype(g_nccl.CommDeregister)>(dlsym(h, "ncclCommDeregister"));
  g_nccl.ok = true;
  return true;
}

}  // namespace sma

// --------------------------------------------------- host bookkeeping
// Independent of the oracle's implementation (tests compare the two bit-exactly).
namespace {
uint64_t host_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
}  // namespace

extern "C" int64_t sma_plan_d_pad(int64_t d, int32_t world) {
  if (d < 1 || world < 1) return -1;
  int64_t a = 512, b = 64LL * world;  // lcm(512, 64 n)
  int64_t x = a, y = b;
  while (y) { int64_t t = x % y; x = y; y = t; }
  const int64_t l = a / x * b;
  return (d + l - 1) / l * l;
}

extern "C" sma_status sma_plan_local_replicas(int32_t k, int32_t world, int32_t rank,
                                              int32_t* first, int32_t* count) {
  if (k < 1 || world < 1 || rank < 0 || rank >= world || !first || !count)
    return fail(SMA_ERR_INVALID_ARG, "sma_plan_local_replicas: bad arguments");
  const int64_t lo = (int64_t)rank * k / world, hi = (int64_t)(rank + 1) * k / world;
  *first = (int32_t)lo;
  *count = (int32_t)(hi - lo);
  return SMA_OK;
}

extern "C" sma_status sma_plan_replica_location(int32_t k, int32_t world, int32_t j,
                                                int32_t* rank, int32_t* slot) {
  if (k < 1 || world < 1 || j < 0 || j >= k || !rank || !slot)
    return fail(SMA_ERR_INVALID_ARG, "sma_plan_replica_location: j=%d outside [0,%d)", j, k);
  // floor(g k / n) <= j  <=>  g <= (j n + n - 1) / k ... take the largest such g
  int32_t g = (int32_t)(((int64_t)j * world + world - 1) / k);
  if (g >= world) g = world - 1;
  while (g > 0 && (int64_t)g * k / world > j) --g;
  while ((int64_t)(g + 1) * k / world <= j) ++g;
  *rank = g;
  *slot = (int32_t)(j - (int64_t)g * k / world);
  return SMA_OK;
}

extern "C" sma_status sma_plan_shard_range(int64_t d, int32_t world, int32_t rank,
                                           int64_t* offset, int64_t* length) {
  if (d < 1 || world < 1 || rank < 0 || rank >= world || !offset || !length)
    return fail(SMA_ERR_INVALID_ARG, "sma_plan_shard_range: bad arguments");
  const int64_t len = sma_plan_d_pad(d, world) / world;
  *offset = rank * len;
  *length = len;
  return SMA_OK;
}

// Fisher-Yates permutation of [0, N) for `epoch` (reading R10), int32 output.
void sma::plan_epoch_permutation(int64_t N, uint64_t seed, int64_t epoch, int32_t* perm) {
  for (int64_t t = 0; t < N; ++t) perm[t] = (int32_t)t;
  const uint64_t key = host_splitmix64(seed ^ (uint64_t)epoch);
  for (int64_t t = N - 1; t > 0; --t) {
    const uint64_t u = host_splitmix64(key + (uint64_t)t);
    const int64_t r = (int64_t)(((unsigned __int128)u * (uint64_t)(t + 1)) >> 64);
    const int32_t tmp = perm[t];
    perm[t] = perm[r];
    perm[r] = tmp;
  }
}

extern "C" sma_status sma_plan_batch_indices(int64_t n_samples, int32_t k, int32_t batch,
                                             uint64_t batch_seed, int64_t round, int32_t j,
                                             int64_t* out) {
  if (n_samples < 1 || n_samples > INT32_MAX || k < 1 || batch < 1 || round < 0 || j < 0 ||
      j >= k || !out)
    return fail(SMA_ERR_INVALID_ARG, "sma_plan_batch_indices: bad arguments");
  const int64_t E = n_samples / ((int64_t)k * batch);
  if (E < 1) return fail(SMA_ERR_INVALID_ARG, "n_samples < k*batch");
  std::vector<int32_t> perm((size_t)n_samples);
  plan_epoch_permutation(n_samples, batch_seed, round / E, perm.data());
  const int64_t base = ((round % E) * k + j) * (int64_t)batch;
  for (int32_t t = 0; t < batch; ++t) out[t] = perm[(size_t)(base + t)];
  return SMA_OK;
}

// ------------------------------------------------ auto-tuner (Alg. 2)
extern "C" sma_status sma_autotune_step(int32_t m, double tau, const double* t, int32_t* l, double* t_prev) {
  if (m < 1 || !t || !l || !t_prev) return fail(SMA_ERR_INVALID_ARG, "bad auto-tuner arguments");
  for (int32_t g = 0; g < m; ++g) {
    const double dt = t[g] - t_prev[g];
    if (dt > tau)
      ++l[g];                          // Alg. 2 line 7: significant increase -> add a learner
    else if (t[g] < t_prev[g] && l[g] > 0)
      --l[g];                          // line 8: decrease -> remove one
    t_prev[g] = t[g];                  // line 9
  }
  return SMA_OK;
}


// ------------------------------------------------ dynamic shared memory cache
namespace sma {
cudaError_t ensure_dyn_smem(const void* func, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> done;  // (func, dev) -> bytes
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& kv : done)
    if (kv.first.first == func && kv.first.second == dev) {
      if (kv.second >= bytes) return cudaSuccess;
      e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e == cudaSuccess) kv.second = bytes;
      return e;
    }
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.push_back({{func, dev}, bytes});
  return e;
}
}  // namespace sma
