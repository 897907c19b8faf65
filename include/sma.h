/*
 * sma.h -- C ABI of libsma, the B200-native hot path of Synchronous Model
 * Averaging (SMA), Algorithm 1 of Koliousis et al., "Crossbow: Scaling Deep
 * Learning with Small Batch Sizes on Multi-GPU Servers", arXiv 1901.02244.
 * Citations "P:n" are lines of the paper text; "S:n" lines of
 * SPEC.md; "Rn" the readings listed in DESIGN.md.
 *
 * One round (sma_step) is one iteration of Alg. 1 over all k
 * learners:   c_j = alpha (w_j - z);   w_j <- w_j - gamma g_j - c_j;
 *             z <- z + sum_j c_j + mu (z - z_prev);   z_prev <- old z.
 *
 * Conventions for every entry point
 *   - Scalars are fp32, vectors fp32, contiguous, unit stride.  d is the model
 *     size (number of parameters).  Parameter p of replica j is
 *     element p of that replica's vector.
 *   - Ownership: the handle owns every device buffer, stream, event, graph and
 *     NCCL communicator it creates.  Inputs marked BORROWED must stay valid
 *     (and unmodified) as stated; everything else is copied.  Outputs go to
 *     caller-owned memory.
 *   - Errors: every call returns sma_status; no C++ exception crosses the ABI.
 *     Arguments are validated before anything is enqueued, so a call that
 *     returns SMA_ERR_INVALID_ARG / _NOT_LOCAL / _GRADS_MISSING / _STATE has
 *     changed nothing.  sma_last_error() returns a thread-local message for
 *     the most recent failure on the calling thread.
 *   - Threading: one issuing host thread per handle.  sma_create,
 *     sma_step and sma_destroy are COLLECTIVE when world > 1: every rank calls
 *     them in the same order with identical (d, k, alpha, gamma, mu, flags).
 *   - Streams: calls taking `cuda_stream` (a cudaStream_t, NULL = legacy
 *     default stream) enqueue their work after all prior work on that stream,
 *     and later work on that stream is ordered after them.  No call in the
 *     hot path synchronises the host.
 *   - There is no CPU fallback: every arithmetic step runs in this library's
 *     CUDA kernels (and NCCL for the inter-GPU exchange).  Without a usable
 *     sm_100 device, sma_create fails with SMA_ERR_CUDA.
 */
#ifndef SMA_H_
#define SMA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMA_ABI_VERSION 2
#define SMA_MAX_LOCAL_REPLICAS 64   /* r = replicas per GPU, P:1193-1194 ("m") */
#define SMA_NCCL_ID_BYTES 128
#define SMA_P2P_HANDLE_BYTES 64  /* cudaIpcMemHandle_t */

typedef struct sma_handle sma_handle;   /* opaque; owns all device state */

typedef enum {
    SMA_OK = 0,
    SMA_ERR_INVALID_ARG = 1,   /* bad size/index/pointer/alignment/hyper-parameter */
    SMA_ERR_NOT_LOCAL = 2,     /* replica j lives on another rank */
    SMA_ERR_GRADS_MISSING = 3, /* a local learner has no gradient registered */
    SMA_ERR_NONFINITE = 4,     /* a NaN/Inf appeared (only with SMA_FLAG_CHECK_FINITE) */
    SMA_ERR_CUDA = 5,          /* CUDA runtime error (message in sma_last_error) */
    SMA_ERR_NCCL = 6,          /* NCCL error or NCCL library not loadable */
    SMA_ERR_OOM = 7,           /* device allocation failed */
    SMA_ERR_STATE = 8          /* call not valid in the handle's current state */
} sma_status;

/* Flags (sma_config.flags). */
enum {
    /* Mode B (lookahead): the inter-GPU z-sync of round i
     * runs on a second stream concurrently with the replica kernel of round i,
     * using the identity z^{i+1} = z^i + alpha Q^i + (mu - alpha k)(z^i - z^{i-1}),
     * Q^i = sum_j (w_j^i - z^{i-1}).  Exact in exact arithmetic; implements the
     * paper's overlap of global synchronisation with the next learning tasks
     * (P:885-889).  Only meaningful on the collective path. */
    SMA_FLAG_OVERLAP = 1u,
    /* North_star-literal variant: the replica kernel writes every c_j to HBM
     * and a separate warp-shuffle/block-tree kernel reduces them.
     * Moves 4 d_pad (5r+4) bytes per round instead of 4 d_pad (3r+3) at n = 1
     * (5r+2 instead of 3r+2 on the collective path). */
    SMA_FLAG_MATERIALIZE_C = 2u,
    /* Record a device flag when any updated value is not finite; sma_step then
     * returns SMA_ERR_NONFINITE at the NEXT call that synchronises
     * (sma_get_central / sma_get_replica / sma_check_finite). */
    SMA_FLAG_CHECK_FINITE = 4u,
    /* Capture the round into a CUDA graph on first use and replay it; the
     * graph is re-instantiated when registered gradient pointers change. */
    SMA_FLAG_CUDA_GRAPH = 8u,
    /* Use the n>1 structure (replica partial -> NCCL reduce-scatter -> shard
     * update -> NCCL all-gather) even when world == 1 (a 1-rank NCCL
     * communicator).  Exercises the multi-GPU path on one GPU. */
    SMA_FLAG_FORCE_COLLECTIVE = 16u,
    /* Time every replica-kernel launch with CUDA events on its own stream
     * (sma_kernel_time). */
    SMA_FLAG_TIMING = 32u,
    /* Replica kernel variant: TMA bulk-copy (cp.async.bulk) shared-memory
     * staging with an mbarrier pipeline (replica_step_tma) ... */
    SMA_FLAG_KERNEL_TMA = 64u,
    /* ... or direct 128-bit loads (replica_step_ldg), the default: on B200 the
     * direct-load kernel on a full grid measured faster at every size
     * (DESIGN.md §4). */
    SMA_FLAG_KERNEL_LDG = 128u,
    /* NEXT-1: the inter-GPU z-sync (reduce-scatter + shard update + all-gather)
     * as ONE kernel on NVSwitch multicast memory (multimem.ld_reduce /
     * multimem.st), with device-side barriers, instead of NCCL RS/AG.  Needs a
     * device with CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED; sma_create fails with
     * SMA_ERR_CUDA otherwise.  Collective path only. */
    SMA_FLAG_NVLS_ZSYNC = 256u,
    /* The inter-GPU z-sync (reduce-scatter + shard update + all-gather) as ONE
     * kernel over peer memory: every rank maps the others' [partial | z]
     * buffers with CUDA IPC and, for its shard, loads the partials of all ranks,
     * updates, and stores the result into every rank's z.  No NCCL is used (no
     * nccl_id needed): after sma_create each rank exports sma_p2p_handle(), the
     * caller all-gathers the handles and every rank calls sma_p2p_connect()
     * before its first sma_step.  Several ranks may share one GPU.
     * Collective path only; exclusive with SMA_FLAG_NVLS_ZSYNC. */
    SMA_FLAG_P2P_ZSYNC = 512u,
    /* NEXT-3: "training multiple learners per GPU" with per-GPU reference
     * models (Section 3.3; reading R20 in DESIGN.md).  GPU g keeps
     * a reference model u_g; GPU 0's reference model is z.  Per
     * round, against round-start values:
     *   d_j = alpha (w_j - u_g);  w_j <- w_j - gamma g_j - d_j
     *   c_g = alpha_g (u_g - z);  u_g <- u_g + sum_{j on g} d_j - c_g  (g >= 1)
     *   z <- z + sum_{j on 0} d_j + sum_{g>=1} c_g + mu (z - z_prev)
     * sma_config.alpha is the intra-GPU alpha_l; alpha_g is set with
     * sma_set_alpha_global (default 1/(2(world-1))).  With one GPU this is
     * exactly the flat Alg. 1.  Every z-sync variant (NCCL, P2P, NVLS, Mode A/B)
     * carries it unchanged: only the per-GPU partial differs.  Not combined
     * with SMA_FLAG_MATERIALIZE_C or SMA_FLAG_KERNEL_TMA. */
    SMA_FLAG_HIERARCHICAL = 1024u,
    /* With SMA_FLAG_P2P_ZSYNC: fuse the reduce-scatter's data movement into the
     * replica kernel.  Its epilogue stores each float4 chunk of the per-GPU
     * partial straight into the owner's slot over peer memory (owner g's
     * partial buffer holds one [shard] slot per source rank), so the z-sync
     * kernel sums local slots in rank order instead of loading every peer's
     * partial.  Same results bit for bit as SMA_FLAG_P2P_ZSYNC alone.  Not
     * combined with SMA_FLAG_MATERIALIZE_C or SMA_FLAG_KERNEL_TMA. */
    SMA_FLAG_P2P_PUSH = 2048u
};

typedef struct {
    int64_t  d;          /* model size, >= 1 */
    int32_t  k;          /* total learners = replicas, >= 1     */
    float    alpha;      /* correction weight, finite; paper: ~1/k             (R5) */
    float    gamma;      /* learning rate, finite; multiplies RAW gradients    (R1) */
    float    mu;         /* central-model momentum, finite */
    int32_t  rank;       /* this process's rank in [0, world)                               */
    int32_t  world;      /* number of GPUs n, >= 1; replicas are block-split over ranks      */
    int32_t  device;     /* CUDA device ordinal used by this rank                           */
    const void* nccl_id; /* SMA_NCCL_ID_BYTES from sma_nccl_unique_id() on rank 0, the same
                            bytes on every rank; required iff world > 1 and not
                            SMA_FLAG_P2P_ZSYNC (copied)                                     */
    uint32_t flags;      /* SMA_FLAG_* */
} sma_config;

/* ---------------------------------------------------------------- lifecycle */

/* Create the state of Alg. 1 lines 1-2 on this rank:
 *   z <- w0;  z_prev <- w0 (R2: the paper's "empty" read as zero momentum in
 *   round 1);  w_j <- w0 for every local replica j (R3; "initialised with the
 *   latest value of the average model").
 * w0_host: d floats in host memory (copied; need not be pinned).
 * Device layout (one allocation per array): W [r][d_pad],
 * z [2][d_pad] (ping-pong: the current z and z_prev), plus P [d_pad],
 * S [d_pad/n] and, with SMA_FLAG_OVERLAP, Q [2][d_pad] on the collective
 * path.  d_pad = sma_plan_d_pad(d, world); the padding [d, d_pad) is 0 and
 * stays exactly 0.  COLLECTIVE when world > 1 (ncclCommInitRank).
 * Errors: INVALID_ARG (d < 1, k < 1, world < 1, rank out of range, more than
 * SMA_MAX_LOCAL_REPLICAS replicas on this rank, non-finite hyper-parameter,
 * missing nccl_id when world > 1, NULL pointers), CUDA, NCCL, OOM.
 * On failure *out is set to NULL and nothing is leaked. */
sma_status sma_create(const sma_config* cfg, const float* w0_host, sma_handle** out);

/* Free everything the handle owns (after finishing its enqueued work).
 * NULL is a no-op.  COLLECTIVE when world > 1. */
void sma_destroy(sma_handle* h);

/* --------------------------------------------------------- gradient intake */

/* Register the RAW gradient of learner j (grad l_{B_j}(w_j), Alg. 1 line 8,
 * P:577; gamma is applied by sma_step, R1) as a device pointer.
 * j: GLOBAL learner index in [0, k); must live on this rank.
 * g_dev: d floats on this rank's device, 16-byte aligned.  BORROWED: must stay
 * valid and unmodified until the next sma_step that reads it has completed on
 * the device; the registration persists across steps until replaced.
 * Errors: INVALID_ARG (j out of range, NULL or misaligned pointer), NOT_LOCAL. */
sma_status sma_set_learner_grads(sma_handle* h, int32_t j, const float* g_dev);

/* Copy a RAW gradient from host memory into the handle's own gradient buffer
 * for learner j and register it (replaces any device registration of j).
 * g_host: d floats (pinned memory makes the copy asynchronous; pageable
 * memory works but the copy is then staged by the driver).  The copy is
 * enqueued on cuda_stream; g_host must stay valid until it has completed.
 * Errors: INVALID_ARG, NOT_LOCAL, CUDA, OOM. */
sma_status sma_set_learner_grads_host(sma_handle* h, int32_t j, const float* g_host,
                                      void* cuda_stream);

/* Pipelined host intake (the end-to-end path of a training loop that streams
 * one batch of gradients per round from the host).  Copies the RAW gradients
 * of ALL r local learners -- g_host[i] is learner local_first + i, d floats,
 * pinned host memory for an asynchronous copy -- into the handle's internal
 * gradient set `set` (0 or 1; two sets so the copies for round s+1 overlap
 * round s) on the handle's own host-to-device stream, ordered after the last
 * round that read that set, and registers them (replacing any registration)
 * for the next sma_step / sma_step_local, which waits for the copies on its
 * stream.  Does not block the host; g_host must stay valid until the copies
 * have completed (sma_synchronize).  Errors: INVALID_ARG (set not 0/1, NULL
 * pointer), CUDA, OOM. */
sma_status sma_stage_grads_host(sma_handle* h, int32_t set, const float* const* g_host);

/* Fill the handle's gradient buffers of all LOCAL learners with the synthetic
 * raw gradients of round `round` (R9):
 *   g_j^i[p] = (U(seed, (i k + j) d + p) - 1/2) 2^-4,
 *   U(s, c) = (splitmix64(splitmix64(s) + c) >> 40) 2^-24,
 * and register them.  Enqueued on cuda_stream.  Errors: CUDA, OOM. */
sma_status sma_synth_grads(sma_handle* h, int64_t round, uint64_t seed, void* cuda_stream);

/* ------------------------------------------------------------------- round */

/* One iteration of Alg. 1 for all k learners:
 *   a3 c_j = alpha (w_j - z) against the same z for all j   (line 9)
 *   a4 w_j <- w_j - gamma g_j - c_j, in place               (line 10)
 *   a5 per-GPU partial of sum_j c_j
 *      (summation order, R7: any order is correct.  The full-grid kernel
 *      adds the local c_j in ascending j; the small-round split kernel (chosen by
 *      d_pad/4, r and the SMA_SPLIT_* knobs) adds them per lane group j mod G and
 *      combines the G groups with xor-shuffles.  So results are bitwise stable
 *      for a given (d, r, knobs) but may differ in the last bits across them.)
 *   a6 NCCL reduce-scatter of the partials (world > 1)
 *   a7 z <- z + sum c + mu (z - z_prev) on this GPU's shard (line 13)
 *   a8 NCCL all-gather of z (world > 1)
 *   z_prev <- old z is a buffer swap (line 14).
 * world == 1 without FORCE_COLLECTIVE: a3-a7 are ONE fused kernel.
 * Every local learner must have a registered gradient (else GRADS_MISSING).
 * COLLECTIVE when world > 1.  Errors: GRADS_MISSING, CUDA, NCCL. */
sma_status sma_step(sma_handle* h, void* cuda_stream);

/* Local-only iteration for a synchronisation period tau > 1 (
 * reading R17 = S:348): every local learner applies only its gradient,
 * w_j <- w_j - gamma g_j; no correction, z and z_prev unchanged.  Call it on
 * the tau - 1 non-synchronising iterations and sma_step on every tau-th.  Not
 * collective.  Errors: GRADS_MISSING, CUDA. */
sma_status sma_step_local(sma_handle* h, void* cuda_stream);

/* ---------------------------------------------------- auto-tuner (NEXT-4) */

/* Alg. 2, one pass of its loop body over m GPUs (host only):
 *   if t[g] - t_prev[g] > tau: l[g] += 1;  else if t[g] < t_prev[g] and l[g] > 0:
 *   l[g] -= 1;  t_prev[g] = t[g].   (Initialise l = 1, t_prev = 0, lines 1-2.)
 * t: observed learning throughput per GPU (e.g. learner batches/s).
 * Follows the paper literally, so l[g] may reach 0.  Before feeding l into
 * sma_set_local_replicas the caller must (a) clamp it to >= 1 for a single-GPU
 * handle (which rejects 0) and to the learner's n_samples / (world * batch), and
 * (b) agree on ONE count across ranks (the resize takes a uniform l, R19),
 * e.g. the minimum or rank 0's value broadcast over the process group. */
sma_status sma_autotune_step(int32_t m, double tau, const double* t, int32_t* l, double* t_prev);

/* Set the number of learners on EVERY GPU to l_new (the same count on all
 * ranks; k becomes l_new * world).  Rank g keeps its first
 * min(r, l_new) replicas (global index g*l_new + slot afterwards); each added
 * replica is initialised with the current z.  alpha is NOT changed
 * (use sma_set_hparams, e.g. alpha = 1/k).  Gradients registered for kept
 * learners stay registered; added learners need one.  Synchronises; COLLECTIVE
 * when world > 1 (every rank calls it with the same l_new).
 * Errors: INVALID_ARG (l_new outside [0, SMA_MAX_LOCAL_REPLICAS], 0 on a
 * single-GPU handle, or -- with a learner attached -- l_new * world * batch >
 * n_samples, which leaves no full round per epoch), CUDA, OOM. */
sma_status sma_set_local_replicas(sma_handle* h, int32_t l_new, void* cuda_stream);

/* ----------------------------------------------------------------- outputs */

/* Copy the central model z (Alg. 1 output) into z_out (d floats;
 * device memory of this rank's GPU if out_is_device, else host memory).
 * Synchronises the host with all work the handle has enqueued.  Every rank
 * holds the full z.  Errors: INVALID_ARG, CUDA, NONFINITE (CHECK_FINITE). */
sma_status sma_get_central(sma_handle* h, float* z_out, int out_is_device);

/* Asynchronous read-back of z for the end-to-end path: enqueue a copy of the
 * central model as of every round enqueued so far (d floats) into z_host
 * (pinned host memory) on the handle's device-to-host stream, after those
 * rounds.  Does not block the host.  The round that would overwrite that z
 * buffer (z and z_prev are ping-ponged, so the second sma_step from now) waits
 * for the copy on its stream, so the value read is exact.  Completion:
 * sma_synchronize.  Errors: INVALID_ARG, CUDA. */
sma_status sma_get_central_async(sma_handle* h, float* z_host);

/* Block the host until all work the handle has enqueued -- rounds, staged
 * host-to-device copies and asynchronous read-backs -- has completed.
 * Errors: CUDA, NONFINITE (CHECK_FINITE). */
sma_status sma_synchronize(sma_handle* h);

/* Same for z_prev (the central model at the beginning of the previous round,
 * P:630-631), needed to checkpoint/resume without losing momentum. */
sma_status sma_get_central_prev(sma_handle* h, float* out, int out_is_device);

/* Copy local replica j (global index) into out (d floats). Synchronises. */
sma_status sma_get_replica(sma_handle* h, int32_t j, float* out, int out_is_device);

/* Overwrite local replica j / the central model / z_prev with d floats
 * (checkpoint restore, distinct initial replicas for tests, R3).
 * Synchronises.  Errors: INVALID_ARG, NOT_LOCAL, CUDA. */
sma_status sma_set_replica(sma_handle* h, int32_t j, const float* w, int in_is_device);
sma_status sma_set_central(sma_handle* h, const float* z, const float* z_prev, int in_is_device);

/* Read-only device views (valid until the next sma_step / sma_destroy):
 * replica j's d_pad floats, and the current z (d_pad floats). */
sma_status sma_replica_device_ptr(sma_handle* h, int32_t j, const float** w_dev);
sma_status sma_central_device_ptr(sma_handle* h, const float** z_dev);

/* SMA restart: every local replica := z and
 * z_prev := z (zero momentum); with SMA_FLAG_HIERARCHICAL also u_g := z.
 * Enqueued on cuda_stream. */
sma_status sma_restart(sma_handle* h, void* cuda_stream);

/* Change alpha, gamma, mu between rounds (online adaptation).
 * Errors: INVALID_ARG (non-finite). */
sma_status sma_set_hparams(sma_handle* h, float alpha, float gamma, float mu);

/* SMA_FLAG_HIERARCHICAL: set the inter-GPU correction weight alpha_g between
 * rounds (every rank, same value).  Errors: STATE (not hierarchical),
 * INVALID_ARG (non-finite). */
sma_status sma_set_alpha_global(sma_handle* h, float alpha_g);

/* SMA_FLAG_HIERARCHICAL: copy this rank's reference model u_g (d floats; on
 * rank 0 -- and on a single-GPU handle -- that is z) into out / overwrite it
 * from u (ranks >= 1 only: rank 0's reference model is set with
 * sma_set_central).  Checkpoint/restore of the two-level state.  Synchronise.
 * Errors: STATE (not hierarchical; set on rank 0), INVALID_ARG, CUDA. */
sma_status sma_get_reference(sma_handle* h, float* out, int out_is_device);
sma_status sma_set_reference(sma_handle* h, const float* u, int in_is_device);

/* If SMA_FLAG_CHECK_FINITE: synchronise and report whether any non-finite
 * value has been produced so far (*flag = 1) ; clears the flag. */
sma_status sma_check_finite(sma_handle* h, int* flag);

/* --------------------------------------------------- built-in learner (a2') */

/* Attach the built-in learner: kind 0 = softmax regression,
 * params W [classes][in_dim] row-major then b [classes] (R12), d =
 * classes*in_dim + classes; kind 1 = MLP in_dim-hidden-classes with ReLU
 * (NEXT-2), params W1 [hidden][in_dim], b1 [hidden], W2 [classes]
 * [hidden], b2 [classes], d = hidden*in_dim + hidden + classes*hidden + classes
 * (the ReLU mask is decided at fp64-level accuracy, R18).  X_dev: n_samples x in_dim fp32
 * row-major, y_dev: n_samples int32 labels in [0, classes); both on this
 * rank's device and BORROWED for the handle's lifetime.  batch = b rows per
 * learner per round; batch_seed keys the per-epoch permutation (R10).
 * Errors: INVALID_ARG (kind, sizes, n_samples < k*batch). */
sma_status sma_learner_attach(sma_handle* h, int32_t kind, int32_t in_dim, int32_t hidden,
                              int32_t classes, int32_t batch, const float* X_dev,
                              const int32_t* y_dev, int64_t n_samples, uint64_t batch_seed);

/* For every local learner j: gather batch B(round, j) (R10), compute the
 * batch-mean gradient (Eq. 2) of the mean cross-entropy at the
 * current replica w_j (max-subtracted softmax, R16) in fp32 (FFMA; for the MLP
 * with >= 12 local learners, unless its SIMT grid fills a wave, its layer-1
 * 784x256 GEMM runs on the tensor cores as 3xTF32, SMA_MLP_TC; the ReLU
 * mask is certain at fp64-level accuracy either way: an a-priori error
 * bound, and a double-float recomputation near a kink),
 * into the handle's gradient buffer, and register it.  Enqueued on
 * cuda_stream.  Errors: STATE (no learner attached), CUDA. */
sma_status sma_learner_grads(sma_handle* h, int64_t round, void* cuda_stream);

/* One full round with the learner in the loop: sma_learner_grads then sma_step
 * (Alg. 1 lines 6-14).  Under Mode B the z-sync of the round is forked before
 * the learner kernels, so it overlaps them.  On a single-GPU handle
 * (no MATERIALIZE_C, no CUDA graph) the gradient and the update of every local
 * learner run as ONE kernel: the MLP round kernel, or the softmax learner's
 * thread-block cluster (feature slices of every replica and of z in shared
 * memory, r <= 8, b <= 16, classes <= 16; SMA_SOFTMAX_CLUSTER=0 disables it) --
 * the same arithmetic per element except the order of the logits' K sum, so
 * within the oracle bar of the two-call form, not bitwise.  With the
 * environment variable SMA_LEARNER_FUSE=1 the softmax learner instead runs the
 * logits kernel then the gradient slice, replica update and central update in
 * one kernel (bitwise sma_learner_grads + sma_step's ascending-j order).
 * Errors: as sma_learner_grads and sma_step. */
sma_status sma_learner_step(sma_handle* h, int64_t round, void* cuda_stream);

/* Rounds round0, round0 + 1, ..., round0 + count - 1 with the learner in the
 * loop: the same results as sma_learner_step called for each of them in turn
 * (bitwise).  On a single-GPU handle (n = 1, no MATERIALIZE_C, no CUDA graph)
 * the rounds of one epoch (R10) run in ONE launch of the fused
 * learner kernel: for the MLP, the CTA that owns a learner's block of hidden
 * units keeps that block's weights on chip across the rounds and prefetches
 * the next round's batch rows and z block, the rounds ordered by per-CTA flags
 * instead of kernel boundaries; for the softmax learner, one thread-block
 * cluster keeps every replica and z in shared memory for the whole launch and
 * exchanges partial logits and softmax rows through distributed shared memory.
 * A new epoch starts a new launch.  Every other configuration calls
 * sma_learner_step per round.
 * Enqueued on cuda_stream; no host synchronisation.  count = 0 is a no-op.
 * Errors: INVALID_ARG (round0 < 0, count < 0, n_samples < k * batch), STATE
 * (no learner attached), CUDA, and sma_step's. */
sma_status sma_learner_steps(sma_handle* h, int64_t round0, int32_t count, void* cuda_stream);

/* ------------------------------------------------ bookkeeping (host only) */
/* Pure functions of their arguments; no device, no handle (bit-exact with
 * the oracle's independent implementation). */

/* d_pad = roundup(d, lcm(512, 64 n)); every shard is d_pad/n floats. */
int64_t sma_plan_d_pad(int64_t d, int32_t world);
/* Replica j -> (rank, slot): rank g with floor(g k/n) <= j < floor((g+1) k/n). */
sma_status sma_plan_replica_location(int32_t k, int32_t world, int32_t j,
                                     int32_t* rank, int32_t* slot);
/* First global replica index and count r on `rank`. */
sma_status sma_plan_local_replicas(int32_t k, int32_t world, int32_t rank,
                                   int32_t* first, int32_t* count);
/* Shard of rank g: [offset, offset + length) of the padded vector. */
sma_status sma_plan_shard_range(int64_t d, int32_t world, int32_t rank,
                                int64_t* offset, int64_t* length);
/* Batch of learner j in round i (R10): b row indices into [0, N). */
sma_status sma_plan_batch_indices(int64_t n_samples, int32_t k, int32_t batch,
                                  uint64_t batch_seed, int64_t round, int32_t j,
                                  int64_t* out);

/* ------------------------------------------------------- P2P bootstrap */

/* SMA_FLAG_P2P_ZSYNC: write this rank's SMA_P2P_HANDLE_BYTES IPC handle of its
 * [flags | partial | z] region to out (host memory).  Errors: STATE (not a P2P
 * handle), CUDA. */
sma_status sma_p2p_handle(sma_handle* h, void* out);

/* SMA_FLAG_P2P_ZSYNC: map the other ranks' regions.  handles: world x
 * SMA_P2P_HANDLE_BYTES, in rank order (this rank's own entry is ignored).  Call
 * once on every rank before the first sma_step.  Errors: STATE (not a P2P
 * handle, or already connected), INVALID_ARG, CUDA. */
sma_status sma_p2p_connect(sma_handle* h, const void* handles);

/* ------------------------------------------------------------- utilities */

/* Write a fresh NCCL unique id (SMA_NCCL_ID_BYTES) to out (rank 0 only;
 * broadcast the bytes to the other ranks).  Errors: NCCL. */
sma_status sma_nccl_unique_id(void* out);

/* With SMA_FLAG_TIMING: total device milliseconds and number of timed
 * intervals of `phase` since its last reset (synchronises).  Each interval is
 * bracketed by CUDA events on the stream the phase runs on:
 *   SMA_PHASE_REPLICA        the replica kernel launch(es) of a round (a3-a5[,a7])
 *   SMA_PHASE_REDUCE_SCATTER ncclReduceScatter of the per-GPU partial (a6)
 *   SMA_PHASE_SHARD_UPDATE   the shard update kernel (a7, collective path)
 *   SMA_PHASE_ALL_GATHER     ncclAllGather of z (a8)
 *   SMA_PHASE_FUSED_ZSYNC    the fused z-sync kernel (a6-a8; SMA_FLAG_NVLS_ZSYNC or
 *                            SMA_FLAG_P2P_ZSYNC; also named SMA_PHASE_NVLS_ZSYNC)
 * Errors: INVALID_ARG (phase out of range). */
enum { SMA_PHASE_REPLICA = 0, SMA_PHASE_REDUCE_SCATTER = 1, SMA_PHASE_SHARD_UPDATE = 2,
       SMA_PHASE_ALL_GATHER = 3, SMA_PHASE_NVLS_ZSYNC = 4, SMA_PHASE_FUSED_ZSYNC = 4,
       SMA_NUM_PHASES = 5 };
sma_status sma_kernel_time(sma_handle* h, int32_t phase, double* total_ms, int64_t* launches,
                           int reset);

/* Turn the per-phase CUDA events of SMA_FLAG_TIMING on or off between calls
 * (the flag sets the initial state).  The events cost GPU time between the
 * kernels of a round (~2.5 us each on B200, a third of a small round), so a
 * benchmark times its rounds with them off and measures the per-phase
 * durations in a separate pass with them on.  While timing is on, rounds are
 * not run as CUDA graphs.  Errors: INVALID_ARG. */
sma_status sma_set_timing(sma_handle* h, int on);

/* Number of libsma CUDA kernels this handle has launched (NCCL collectives not counted). */
int64_t sma_launch_count(const sma_handle* h);

/* Shape of this rank's state. */
sma_status sma_info(const sma_handle* h, int64_t* d_pad, int32_t* local_first,
                    int32_t* local_count, int64_t* shard_offset, int64_t* shard_length);

const char* sma_last_error(void);
int sma_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SMA_H_ */
