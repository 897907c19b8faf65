// sma_internal.h -- declarations shared by libsma's runtime (sma_runtime.cu) and
// its kernels (sma_kernels.cu).  Not part of the ABI (include/sma.h is).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <string>

#include "../../include/sma.h"

namespace sma {

// Up to SMA_MAX_LOCAL_REPLICAS gradient pointers, passed BY VALUE as a kernel
// parameter (constant bank: broadcast to every thread, no extra global load,
// and baked into a captured CUDA graph together with the other arguments).
struct GradTable {
  const float* p[SMA_MAX_LOCAL_REPLICAS];
};

// SMA_FLAG_P2P_PUSH: where each rank's slot buffer of the current partial is
// mapped in this process (owner g's buffer holds [n][shard] slots, one per source).
struct PushTable {
  float* p[SMA_MAX_LOCAL_REPLICAS];
};

// What the replica kernel emits besides the updated replicas.
enum ReplicaMode : int {
  kFused = 0,    // n == 1: also z_next = z + sum c + mu (z - z_prev)   (Alg. 1 line 13)
  kPartialA = 1, // collective path, paper order: P = sum_{local j} c_j
  kPartialB = 2, // collective path, lookahead: Q = sum_{local j} (w_j' - z)
  kLocal = 3,    // local-only iteration (sync period tau > 1): w_j' = w_j - gamma g_j
  // Two-level rule of Section 3.3 (SMA_FLAG_HIERARCHICAL, reading R20), GPU g >= 1
  // with reference model u = U: d_j = alpha (w_j - u), D = sum d_j,
  // c = alpha_g (u - z), u' = (u + D) - c, and out = c (Mode A) ...
  kHierA = 4,
  // ... or out = alpha_g (u' - z) (Mode B lookahead).
  kHierB = 5,
  // GPU 0 under Mode B: as kPartialB, but out = alpha * sum_j (w_j' - z).
  kHierB0 = 6,
};

struct ReplicaArgs {
  float* W;            // [r][ld] replicas, updated in place
  int64_t ld;          // row stride in floats (= d_pad, multiple of 512)
  int r;               // local replica count
  GradTable g;         // raw gradients, d floats each (16-byte aligned)
  int64_t d;           // valid length (g is read only below d)
  int64_t n4;          // d_pad / 4  (float4 chunks)
  const float* z;      // current central model z^i            [d_pad]
  float* zprev_next;   // kFused: reads z^{i-1}, writes z^{i+1} in place [d_pad]
  float* out;          // kPartialA: P, kPartialB: Q          [d_pad]
  float* C;            // MATERIALIZE_C: c_j buffer [r][ld] (else nullptr)
  float alpha, gamma, mu;
  int* nonfinite;      // CHECK_FINITE flag or nullptr
  int64_t c0;          // first float4 chunk this launch covers (LDG tail after TMA)
  float* U;            // kHierA/B: this GPU's reference model u_g, updated in place [d_pad]
  float alpha_g;       // kHierA/B: inter-GPU correction weight
  // SMA_FLAG_P2P_PUSH (push_n > 0): the per-GPU partial is not written to `out`
  // but pushed, shard by shard, into slot `push_rank` of every owner's buffer
  // (the reduce-scatter's data movement inside the replica kernel's epilogue)
  PushTable push;
  int64_t push_shard;  // floats per shard
  int push_n, push_rank;
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) only when the size
// grows for this (kernel, device): the call costs microseconds of host time and
// the learner launchers would otherwise issue it on every round.  Thread-safe.
cudaError_t ensure_dyn_smem(const void* func, int bytes);

// Launchers (return the launch error, never synchronise).
cudaError_t launch_replica_step(int mode, bool tma, const ReplicaArgs& a, int num_sms,
                                cudaStream_t s);
// TMA variant internals (sma_kernels_tma.cu): full kTile tiles below d.
int64_t tma_full_tiles(int64_t d);
int64_t tma_tile_floats();
cudaError_t launch_replica_step_tma(int mode, const ReplicaArgs& a, int64_t ntiles, int num_sms,
                                    cudaStream_t s);
// MATERIALIZE_C second pass: reduce C over replicas (warp shuffle + block tree),
// then the fused z update (mode kFused) or the partial (kPartialA).
cudaError_t launch_reduce_corrections(int mode, const ReplicaArgs& a, int num_sms,
                                      cudaStream_t s);
// Shard update after the reduce-scatter (a7).  Mode A: z' = z + S + mu (z - zp);
// Mode B: z' = z + alpha S + (mu - alpha k)(z - zp).  zprev_next is in/out.
cudaError_t launch_zsync(int mode, const float* S, const float* z, float* zprev_next,
                         int64_t n4, float alpha, float mu, float coef_b, int* nonfinite,
                         int num_sms, cudaStream_t s);
// SMA_FLAG_P2P_PUSH: push a full local partial src [d_pad] into the owners' slots.
cudaError_t launch_push_partial(const float* src, const ReplicaArgs& a, int num_sms, cudaStream_t s);
// Mode B prologue: Q = scale * sum_j (w_j - zprev) over local replicas, or
// Q = scale * (U - zprev) when U != nullptr (hierarchical, GPU g >= 1).
cudaError_t launch_q_prologue(const float* W, int64_t ld, int r, const float* zprev, float* Q,
                              int64_t n4, const float* U, float scale, int num_sms,
                              cudaStream_t s);
// Synthetic raw gradients of round `round` for local replicas [j0, j0 + r).
cudaError_t launch_synth_grads(float* G, int64_t ld, int r, int j0, int k, int64_t d,
                               int64_t round, uint64_t seed, int num_sms, cudaStream_t s);
// Softmax-regression learner gradient for the r local replicas.
// E: fp32 scratch [r][b][classes] (softmax minus one-hot).
cudaError_t launch_softmax_grad(const float* X, const int32_t* y, const int32_t* perm,
                                int64_t pos0, int b, int in_dim, int classes, const float* W,
                                int64_t ld, int r, int j0, float* E, float* G, cudaStream_t s);
// Softmax learner + the fused n = 1 round in two kernels (logits, then
// gradient slice + replica update + central update); bitwise equal to
// launch_softmax_grad followed by replica_step_ldg<kFused>.
cudaError_t launch_softmax_round(const float* X, const int32_t* y, const int32_t* perm,
                                 int64_t pos0, int b, int in_dim, int classes, int j0, float* E,
                                 float* G, const ReplicaArgs& a, cudaStream_t s);
// MLP learner (kind 1) gradient for the r local replicas (sma_learner_mlp.cu).
// A1: double-float scratch [r][b][hidden]; DA: fp32 scratch [r][b][hidden].
// E: fp32 scratch [r][b][classes].
cudaError_t launch_mlp_grad(const float* X, const int32_t* y, const int32_t* perm, int64_t pos0,
                            int b, int in_dim, int hidden, int classes, const float* W, int64_t ld,
                            int r, int j0, float2* A1, float* E, float* DA, float* G,
                            cudaStream_t s);
// SMA_MLP_TC as parsed: -1 unset (per-r defaults), else bits 1 = layer 1, 2 = dW1.
int mlp_tc_policy();
// The MLP learner as ONE kernel (sma_learner_mlp_fused.cu): the gradient of all
// r local learners into G and, with update = true, the fused n = 1 round
// (a3-a7) over every parameter, for `count` consecutive rounds of one epoch
// (count > 1 only with update; batch rows of round i at perm[pos0 + i kb + ...]).
// PL: scratch of 2 x num_sms x (16 x 32 + 32) floats; bar: 3 x num_sms zeroed 128-byte
// flag lines; epoch: the first round's number, above every earlier launch's
// (the caller adds count).  Returns cudaErrorNotSupported (nothing launched)
// outside its shapes or when disabled (SMA_MLP_FUSED=0, or SMA_MLP_TC set: the
// five-kernel GEMM paths).
bool mlp_fused_enabled();
cudaError_t launch_mlp_round(const float* X, const int32_t* y, const int32_t* perm, int64_t pos0,
                             int64_t kb, int count, int b, int in_dim, int hidden, int classes,
                             int j0, float* PL, unsigned* bar, unsigned epoch, float* G,
                             const ReplicaArgs& a, bool update, int num_sms, cudaStream_t s);
// The softmax-regression learner (kind 0) AND the n = 1 round for `count`
// consecutive rounds of one epoch as ONE thread-block cluster of r CTAs
// (sma_learner_softmax_fused.cu): replicas, z and batch rows on chip, z
// exchanged through distributed shared memory; G receives the last round's
// gradients.  cudaErrorNotSupported (nothing launched) outside its shapes or
// when disabled (SMA_SOFTMAX_CLUSTER=0).
bool softmax_cluster_enabled();
cudaError_t launch_softmax_cluster_rounds(const float* X, const int32_t* y, const int32_t* perm,
                                          int64_t pos0, int64_t kb, int count, int b, int in_dim,
                                          int classes, int j0, float* G, const ReplicaArgs& a,
                                          cudaStream_t s);
// MLP layer 1 on tcgen05 (3xTF32 + |.| bound MMAs, cluster K-split); returns
// cudaErrorNotSupported without launching when the shape is outside its path.
cudaError_t launch_mlp_hidden_tc(const float* X, const int32_t* perm, int64_t pos0, int b,
                                 int in_dim, int hidden, const float* W, int64_t ld, int r, int j0,
                                 float2* A1, cudaStream_t s);
// MLP dW1 = da1^T X / b on tcgen05 (3xTF32, M128 x N112 tiles); same
// cudaErrorNotSupported contract.
cudaError_t launch_mlp_w1_tc(const float* X, const int32_t* perm, int64_t pos0, int b, int in_dim,
                             int hidden, int j0, int64_t ld, int r, const float* DA, float* G,
                             cudaStream_t s);
// Broadcast: dst rows [r][ld] := src [ld]   and   y := x   (restart / init).
cudaError_t launch_broadcast_rows(float* dst, int64_t ld, int r, const float* src, int64_t n4,
                                  int num_sms, cudaStream_t s);

// ---------------------------------------------------------------- NVLS z-sync
// One physical allocation per rank bound to an NVSwitch multicast object
// (sma_nvls.cu).  uc: this rank's unicast mapping; mcva: the multicast mapping.
struct NvlsRegion {
  unsigned long long mc = 0, phys = 0;  // CUmemGenericAllocationHandle
  unsigned long long uc = 0, mcva = 0;  // CUdeviceptr
  size_t size = 0;
  int dev = 0;
  bool have_mc = false, have_phys = false, uc_mapped = false, mc_mapped = false, bound = false;
};
struct NvlsArgs {
  const float* part_mc;  // multicast view of this round's per-GPU partial (P or Q[qi])
  float* znext_mc;       // multicast view of z[1-cur] (receives z^{i+1})
  const float* z;        // local z[cur]
  const float* zprev;    // local z[1-cur] (z_prev of this GPU's shard)
  int64_t off4, len4;    // this GPU's shard in float4 chunks
  float alpha, mu, coef_b;
  unsigned* flag_uc;     // [0] barrier A, [1] barrier B (local view)
  unsigned* flag_mc;     // same, multicast view
  unsigned* expect;      // [2] device-side barrier targets (local memory)
  unsigned* done_ctr;    // CTA arrival counter (local memory)
  int n;                 // number of GPUs
  int* nonfinite;
};
bool nvls_supported(int device, std::string* err);
bool nvls_setup(NvlsRegion* R, int device, int rank, int world, size_t bytes, const std::string& key,
                const std::function<bool(std::string*)>& barrier, std::string* err);
void nvls_teardown(NvlsRegion* R);
cudaError_t launch_zsync_nvls(int mode, const NvlsArgs& a, int num_ctas, cudaStream_t s);

// ----------------------------------------------------------------- P2P z-sync
// (sma_p2p.cu) One cudaMalloc region per rank [flags (4 KB) | partial(s) | z[2]],
// mapped into every rank's address space with CUDA IPC.  base[g] is rank g's
// region as seen from this process; all offsets are in bytes.
constexpr int kMaxP2PRanks = 64;
struct P2PArgs {
  char* base[kMaxP2PRanks];
  int64_t off_flags, off_part, off_z, off_zprev;
  int64_t off4, len4;    // this rank's shard in float4 chunks
  float alpha, mu, coef_b;
  int n, rank;
  unsigned* ctl;         // local: [0] barrier-A target, [1] barrier-B target, [2] CTA counter,
                         // [3] barrier A passed (device-scope flag set by CTA 0)
  int* nonfinite;
  int push;              // SMA_FLAG_P2P_PUSH: the partials are already in local slots
  int emu_n;             // SMA_P2P_EMULATE_N (measurement only, 1 rank): 0 = off, else see sma_p2p.cu
};
cudaError_t launch_zsync_p2p(int mode, const P2PArgs& a, int num_ctas, cudaStream_t s);

}  // namespace sma
