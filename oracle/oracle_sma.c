/*
 * oracle_sma.c -- the independent CPU oracle for the SMA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (libsma.so) never links, calls or includes anything here, and
 * nothing here includes anything from the product (include/, csrc/).
 *
 * What it computes: Algorithm 1 "Synchronous model averaging (SMA)" of
 * Koliousis et al., "Crossbow: Scaling Deep Learning with Small Batch Sizes on
 * Multi-GPU Servers", arXiv 1901.02244 (prose PAPER.md:602-635),
 * written out step by step in fp64 with plain loops, single-threaded.
 * Readings of what the paper leaves open are the ones DESIGN.md lists
 * (R1..R16, = SURVEY.md §8c Q1..Q16); each function names the ones it takes.
 *
 * Pins (tests/test_oracle_pins.py): SPEC worked examples, alpha=0 -> SGD,
 * alpha=1/k & mu=0 -> mean of replicas, k=1 leapfrog, the conservation law,
 * g=0 contraction, quadratic fixed point, exact-rational brute force,
 * splitmix64 published vectors, softmax loss ln(10) / finite differences.
 * Every function below is pinned; none is "parity unpinned" except the
 * summation-order-dependent bitwise comparison noted in DESIGN.md.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared oracle_sma.c -lm
 * (-ffp-contract=off: no FMA contraction, each operation rounds once in fp64).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Input generator (reading R9).  Re-implemented   */
/* here on purpose: the oracle shares no code with the CUDA path.            */
/* ------------------------------------------------------------------------ */

uint64_t orc_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* U(seed, ctr) = (splitmix64(splitmix64(seed) + ctr) >> 40) * 2^-24 */
double orc_uniform24(uint64_t seed, uint64_t ctr) {
    uint64_t key = orc_splitmix64(seed);
    uint64_t h = orc_splitmix64(key + ctr);
    return (double)(h >> 40) * ldexp(1.0, -24);
}

/* w0[p] = (U(seed_w, p) - 1/2) * 2^-3 for p in idx (R9). */
void orc_w0(int64_t n_idx, const int64_t *idx, uint64_t seed, double *out) {
    for (int64_t t = 0; t < n_idx; t++)
        out[t] = (orc_uniform24(seed, (uint64_t)idx[t]) - 0.5) * 0.125;
}

/* Raw synthetic gradient g_j^i[p] = (U(seed_g, (i*k+j)*d + p) - 1/2) * 2^-4
 * (R9).  gamma is applied by the algorithm, not here (R1). */
void orc_synth_grad(int64_t d, int32_t k, int64_t round, int32_t j, uint64_t seed,
                    int64_t n_idx, const int64_t *idx, double *out) {
    uint64_t base = ((uint64_t)round * (uint64_t)k + (uint64_t)j) * (uint64_t)d;
    for (int64_t t = 0; t < n_idx; t++)
        out[t] = (orc_uniform24(seed, base + (uint64_t)idx[t]) - 0.5) * 0.0625;
}

/* ------------------------------------------------------------------------ */
/* Bookkeeping (SURVEY.md §8b "Bookkeeping"; must be bit-exact vs libsma).   */
/* ------------------------------------------------------------------------ */

/* Replica j lives on the unique rank g with floor(g*k/n) <= j < floor((g+1)*k/n),
 * at slot j - floor(g*k/n): a balanced block split of the k learners over the
 * n GPUs ("multiple learners per GPU"; k = m x #GPUs,
 * PAPER.md:1455-1456).  Plain linear search. Returns 0 on success, -1 if j is
 * out of range. */
int orc_replica_location(int32_t k, int32_t n, int32_t j, int32_t *rank, int32_t *slot) {
    if (k < 1 || n < 1 || j < 0 || j >= k) return -1;
    for (int32_t g = 0; g < n; g++) {
        int64_t lo = ((int64_t)g * k) / n;
        int64_t hi = ((int64_t)(g + 1) * k) / n;
        if (lo <= j && j < hi) { *rank = g; *slot = (int32_t)(j - lo); return 0; }
    }
    return -1;
}

static int64_t gcd64(int64_t a, int64_t b) { while (b) { int64_t t = a % b; a = b; b = t; } return a; }

/* d_pad = roundup(d, lcm(512, 64 n)): every shard d_pad/n is a whole number of
 * 256-byte rows (64 floats); for n | 8 this is roundup(d, 512). */
int64_t orc_d_pad(int64_t d, int32_t n) {
    int64_t q = 64LL * n;
    int64_t l = 512 / gcd64(512, q) * q;
    return ((d + l - 1) / l) * l;
}

/* Shard g of the central model is [g*d_pad/n, (g+1)*d_pad/n): each GPU owns
 * one equal partition of z ("all-reduce evenly distributes the computation
 * of the update for the average model among the GPUs"). */
void orc_shard_range(int64_t d, int32_t n, int32_t g, int64_t *off, int64_t *len) {
    int64_t dp = orc_d_pad(d, n);
    *len = dp / n;
    *off = (int64_t)g * (dp / n);
}

/* select(B) (Alg. 1 line 6) without replacement, reading R10:
 * epoch e uses the Fisher-Yates permutation pi_e of [0, N) keyed by
 * splitmix64(seed ^ e); step t (t = N-1 .. 1) draws u = splitmix64(key + t)
 * and swaps positions t and floor(u * (t+1) / 2^64). */
void orc_epoch_permutation(int64_t N, uint64_t seed, int64_t epoch, int64_t *perm) {
    for (int64_t t = 0; t < N; t++) perm[t] = t;
    uint64_t key = orc_splitmix64(seed ^ (uint64_t)epoch);
    for (int64_t t = N - 1; t >= 1; t--) {
        uint64_t u = orc_splitmix64(key + (uint64_t)t);
        int64_t r = (int64_t)(((unsigned __int128)u * (unsigned __int128)(uint64_t)(t + 1)) >> 64);
        int64_t tmp = perm[t]; perm[t] = perm[r]; perm[r] = tmp;
    }
}

/* Batch of learner j in round i (R10): E = floor(N / (k b)) rounds per epoch,
 * e = floor(i / E), rows pi_e[((i mod E) k + j) b + t] for t < b.
 * Returns -1 if E < 1. */
int orc_batch_indices(int64_t N, int32_t k, int32_t b, uint64_t seed, int64_t round,
                      int32_t j, int64_t *out) {
    int64_t E = N / ((int64_t)k * b);
    if (E < 1 || j < 0 || j >= k || round < 0) return -1;
    int64_t e = round / E;
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    if (!perm) return -1;
    orc_epoch_permutation(N, seed, e, perm);
    int64_t base = ((round % E) * k + j) * (int64_t)b;
    for (int32_t t = 0; t < b; t++) out[t] = perm[base + t];
    free(perm);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1, one iteration, over m parameters.         */
/* ------------------------------------------------------------------------ */

/* One iteration of Alg. 1 with the raw gradients given (R1: g_j = gamma*G_j,
 * Alg. 1 line 8).
 *   W     [k][m]  replicas w_1..w_k, updated in place
 *   z     [m]     central average model, updated in place
 *   zprev [m]     previous central model, updated in place
 *   G     [k][m]  raw gradients grad l_{B_j}(w_j) evaluated at the current w_j
 *   csum  [m]     scratch (sum of the corrections)
 * Line 4:  c_1..c_k <- empty
 * Line 5:  for j = 1..k (ascending):
 * Line 8:     g_j <- gamma * G_j
 * Line 9:     c_j <- alpha (w_j - z)          (all j against the same z)
 * Line 10:    w_j <- w_j - g_j - c_j
 * Line 11: z' <- z
 * Line 13: z  <- z + sum_j c_j + mu (z - z_prev)   (sum in ascending j, R7)
 * Line 14: z_prev <- z'
 */
void orc_sma_round(int64_t m, int32_t k, double alpha, double gamma, double mu,
                   double *W, double *z, double *zprev, const double *G, double *csum) {
    for (int64_t p = 0; p < m; p++) csum[p] = 0.0;
    for (int32_t j = 0; j < k; j++) {
        double *w = W + (int64_t)j * m;
        const double *Gj = G + (int64_t)j * m;
        for (int64_t p = 0; p < m; p++) {
            double g = gamma * Gj[p];            /* line 8  */
            double c = alpha * (w[p] - z[p]);    /* line 9  */
            w[p] = w[p] - g - c;                 /* line 10 */
            csum[p] = csum[p] + c;               /* the sum of line 13, j ascending */
        }
    }
    for (int64_t p = 0; p < m; p++) {
        double zold = z[p];                                   /* line 11 */
        z[p] = z[p] + csum[p] + mu * (z[p] - zprev[p]);       /* line 13 */
        zprev[p] = zold;                                      /* line 14 */
    }
}

/* R rounds of Alg. 1 on the synthetic inputs at the parameter indices idx
 * (SMA with given gradients is separable per parameter index, so a sample
 * of indices runs the identical computation).  Initialisation: z <- w0
 * (line 1), z_prev <- w0 (R2: the paper's "empty" read as zero momentum in
 * round 1), w_j <- w0 for every j (R3).
 * Outputs z, zprev [n_idx] and, if W_out != NULL, the replicas [k][n_idx].
 * Returns 0, or -1 on allocation failure. */
int orc_sma_run_synth(int64_t d, int32_t k, double alpha, double gamma, double mu,
                      int64_t R, uint64_t seed_w, uint64_t seed_g,
                      int64_t n_idx, const int64_t *idx,
                      double *z_out, double *zprev_out, double *W_out) {
    double *W = (double *)malloc(sizeof(double) * (size_t)k * (size_t)n_idx);
    double *G = (double *)malloc(sizeof(double) * (size_t)k * (size_t)n_idx);
    double *cs = (double *)malloc(sizeof(double) * (size_t)n_idx);
    if (!W || !G || !cs) { free(W); free(G); free(cs); return -1; }
    orc_w0(n_idx, idx, seed_w, z_out);                                /* line 1 */
    for (int64_t t = 0; t < n_idx; t++) zprev_out[t] = z_out[t];      /* line 2, R2 */
    for (int32_t j = 0; j < k; j++)                                   /* R3 */
        for (int64_t t = 0; t < n_idx; t++) W[(int64_t)j * n_idx + t] = z_out[t];
    for (int64_t i = 0; i < R; i++) {                                 /* line 3, R4 */
        for (int32_t j = 0; j < k; j++)                               /* lines 6-8 */
            orc_synth_grad(d, k, i, j, seed_g, n_idx, idx, G + (int64_t)j * n_idx);
        orc_sma_round(n_idx, k, alpha, gamma, mu, W, z_out, zprev_out, G, cs);
    }
    if (W_out) memcpy(W_out, W, sizeof(double) * (size_t)k * (size_t)n_idx);
    free(W); free(G); free(cs);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Built-in learner: softmax regression (back-propagation; */
/* batch-mean gradient, Eq. 2).           */
/* Parameter layout (R12): W [classes][in_dim] row-major, then b [classes].  */
/* ------------------------------------------------------------------------ */

/* Mean cross-entropy over the b rows X[rows[t]] and, if grad != NULL, its
 * gradient:  logits_c = sum_f W[c][f] x_f + b_c;  p = softmax(logits) with the
 * row maximum subtracted first (R16);  loss = -(1/b) sum_t log p_{t, y_t};
 * dW[c][f] = (1/b) sum_t (p_tc - [y_t = c]) x_tf;  db[c] = (1/b) sum_t (p_tc - [y_t = c]).
 * All in fp64.  Returns the loss. */
double orc_softmax_loss_grad(int32_t in_dim, int32_t classes, int32_t b,
                             const float *X, const int32_t *y, const int64_t *rows,
                             const double *params, double *grad) {
    const double *Wm = params;
    const double *bias = params + (int64_t)classes * in_dim;
    int64_t dparams = (int64_t)classes * in_dim + classes;
    double *logit = (double *)malloc(sizeof(double) * (size_t)classes);
    double loss = 0.0;
    if (grad) for (int64_t q = 0; q < dparams; q++) grad[q] = 0.0;
    for (int32_t t = 0; t < b; t++) {
        const float *x = X + rows[t] * (int64_t)in_dim;
        for (int32_t c = 0; c < classes; c++) {
            double s = bias[c];
            for (int32_t f = 0; f < in_dim; f++) s += Wm[(int64_t)c * in_dim + f] * (double)x[f];
            logit[c] = s;
        }
        double mx = logit[0];
        for (int32_t c = 1; c < classes; c++) if (logit[c] > mx) mx = logit[c];
        double den = 0.0;
        for (int32_t c = 0; c < classes; c++) den += exp(logit[c] - mx);
        loss += -((logit[y[rows[t]]] - mx) - log(den));
        if (grad) {
            for (int32_t c = 0; c < classes; c++) {
                double pc = exp(logit[c] - mx) / den;
                double e = pc - (c == y[rows[t]] ? 1.0 : 0.0);
                for (int32_t f = 0; f < in_dim; f++)
                    grad[(int64_t)c * in_dim + f] += e * (double)x[f];
                grad[(int64_t)classes * in_dim + c] += e;
            }
        }
    }
    if (grad) for (int64_t q = 0; q < dparams; q++) grad[q] = grad[q] / (double)b;
    free(logit);
    return loss / (double)b;
}

/* R rounds of Alg. 1 with the softmax learner in the loop (config C1):
 * learner j in round i takes batch B(i, j) (R10, orc_batch_indices), computes
 * G_j = grad l_{B_j}(w_j) at its current replica, then the round proceeds as
 * orc_sma_round.  w0 [d] is the initial model (line 1; R2; R3).
 * Outputs z, zprev [d] and W_out [k][d] (may be NULL).  Returns 0 / -1. */
int orc_sma_run_softmax(int32_t in_dim, int32_t classes, int32_t b,
                        const float *X, const int32_t *y, int64_t N, uint64_t batch_seed,
                        int32_t k, double alpha, double gamma, double mu, int64_t R,
                        const double *w0, double *z_out, double *zprev_out, double *W_out) {
    int64_t d = (int64_t)classes * in_dim + classes;
    double *W = (double *)malloc(sizeof(double) * (size_t)k * (size_t)d);
    double *G = (double *)malloc(sizeof(double) * (size_t)k * (size_t)d);
    double *cs = (double *)malloc(sizeof(double) * (size_t)d);
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)b);
    if (!W || !G || !cs || !rows) { free(W); free(G); free(cs); free(rows); return -1; }
    for (int64_t p = 0; p < d; p++) { z_out[p] = w0[p]; zprev_out[p] = w0[p]; }
    for (int32_t j = 0; j < k; j++) memcpy(W + (int64_t)j * d, w0, sizeof(double) * (size_t)d);
    int rc = 0;
    for (int64_t i = 0; i < R && rc == 0; i++) {
        for (int32_t j = 0; j < k; j++) {
            rc = orc_batch_indices(N, k, b, batch_seed, i, j, rows);
            if (rc) break;
            orc_softmax_loss_grad(in_dim, classes, b, X, y, rows, W + (int64_t)j * d,
                                  G + (int64_t)j * d);
        }
        if (rc == 0) orc_sma_round(d, k, alpha, gamma, mu, W, z_out, zprev_out, G, cs);
    }
    if (W_out) memcpy(W_out, W, sizeof(double) * (size_t)k * (size_t)d);
    free(W); free(G); free(cs); free(rows);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* NEXT-3 / NEXT-4                                           */
/* ------------------------------------------------------------------------ */

/* Local-only iteration for synchronisation period tau > 1 (PAPER.md:1462-1471,
 * reading R17 = SPEC S:348): on a non-synchronising iteration every learner
 * applies only its gradient, w_j <- w_j - gamma G_j (Eq. 1); no correction and
 * no update of z or z_prev. */
void orc_local_round(int64_t m, int32_t k, double gamma, double *W, const double *G) {
    for (int32_t j = 0; j < k; j++)
        for (int64_t p = 0; p < m; p++)
            W[(int64_t)j * m + p] = W[(int64_t)j * m + p] - gamma * G[(int64_t)j * m + p];
}

/* Alg. 2, "Selecting the number of learners per GPU", one
 * pass of its while-loop body over the m GPUs (lines 4-9):
 *   if t_g - t'_g > tau:            l_g <- l_g + 1     (line 7)
 *   else if t_g < t'_g and l_g > 0: l_g <- l_g - 1     (line 8)
 *   t'_g <- t_g                                         (line 9)
 * l [m] and t_prev [m] are updated in place; t [m] is the observed
 * throughput.  Initial values (line 1-2): l = 1, t' = 0. */
void orc_autotune_step(int32_t m, double tau, const double *t, int32_t *l, double *t_prev) {
    for (int32_t g = 0; g < m; g++) {
        if (t[g] - t_prev[g] > tau) l[g] = l[g] + 1;
        else if (t[g] < t_prev[g] && l[g] > 0) l[g] = l[g] - 1;
        t_prev[g] = t[g];
    }
}

/* Replica resize with the same number l of learners on each of n GPUs
 * (one GPU's throughput may set the count for all), from l
 * to l_new: GPU g keeps its first min(l, l_new) replicas in order; each added
 * replica is initialised with the current central model z ("initialised with
 * the latest value of the average model").  Global index of
 * replica s on GPU g is g*l + s before and g*l_new + s after.
 * W [n*l][m] -> W_new [n*l_new][m]. */
void orc_resize_replicas(int64_t m, int32_t n, int32_t l, int32_t l_new, const double *W,
                         const double *z, double *W_new) {
    for (int32_t g = 0; g < n; g++)
        for (int32_t s = 0; s < l_new; s++) {
            double *dst = W_new + ((int64_t)g * l_new + s) * m;
            const double *src = (s < l) ? W + ((int64_t)g * l + s) * m : z;
            for (int64_t p = 0; p < m; p++) dst[p] = src[p];
        }
}

/* ------------------------------------------------------------------------ */
/* Built-in learner, kind 1: MLP in_dim-hidden-classes with ReLU (SPEC.md    */
/* S:104 "MLP (784-256-10)"; back-propagation; batch-mean   */
/* gradient Eq. 2).  Parameter layout (R12): W1 [hidden]    */
/* [in_dim], b1 [hidden], W2 [classes][hidden], b2 [classes].  ReLU'(a) = 1  */
/* if a > 0 else 0 (R18).  All fp64.  Returns the mean cross-entropy; fills  */
/* grad (if not NULL) and, if min_abs_pre != NULL, the smallest |a1| seen   */
/* (distance of the batch from a ReLU kink).                                  */
/* ------------------------------------------------------------------------ */
double orc_mlp_loss_grad(int32_t in_dim, int32_t hidden, int32_t classes, int32_t b,
                         const float *X, const int32_t *y, const int64_t *rows,
                         const double *params, double *grad, double *min_abs_pre) {
    const double *W1 = params;
    const double *b1 = W1 + (int64_t)hidden * in_dim;
    const double *W2 = b1 + hidden;
    const double *b2 = W2 + (int64_t)classes * hidden;
    int64_t dparams = (int64_t)hidden * in_dim + hidden + (int64_t)classes * hidden + classes;
    double *a1 = (double *)malloc(sizeof(double) * (size_t)hidden);
    double *h = (double *)malloc(sizeof(double) * (size_t)hidden);
    double *logit = (double *)malloc(sizeof(double) * (size_t)classes);
    double *e = (double *)malloc(sizeof(double) * (size_t)classes);
    double loss = 0.0, mn = INFINITY;
    if (grad) for (int64_t q = 0; q < dparams; q++) grad[q] = 0.0;
    double *gW1 = grad, *gb1 = grad ? grad + (int64_t)hidden * in_dim : NULL;
    double *gW2 = grad ? gb1 + hidden : NULL, *gb2 = grad ? gW2 + (int64_t)classes * hidden : NULL;
    for (int32_t t = 0; t < b; t++) {
        const float *x = X + rows[t] * (int64_t)in_dim;
        const int32_t yt = y[rows[t]];
        for (int32_t k = 0; k < hidden; k++) {              /* forward, layer 1 */
            double s = b1[k];
            for (int32_t f = 0; f < in_dim; f++) s += W1[(int64_t)k * in_dim + f] * (double)x[f];
            a1[k] = s;
            h[k] = s > 0.0 ? s : 0.0;
            if (fabs(s) < mn) mn = fabs(s);
        }
        for (int32_t c = 0; c < classes; c++) {             /* forward, layer 2 */
            double s = b2[c];
            for (int32_t k = 0; k < hidden; k++) s += W2[(int64_t)c * hidden + k] * h[k];
            logit[c] = s;
        }
        double mx = logit[0];
        for (int32_t c = 1; c < classes; c++) if (logit[c] > mx) mx = logit[c];
        double den = 0.0;
        for (int32_t c = 0; c < classes; c++) den += exp(logit[c] - mx);
        loss += -((logit[yt] - mx) - log(den));
        if (!grad) continue;
        for (int32_t c = 0; c < classes; c++)               /* dL/dlogits */
            e[c] = exp(logit[c] - mx) / den - (c == yt ? 1.0 : 0.0);
        for (int32_t c = 0; c < classes; c++) {
            for (int32_t k = 0; k < hidden; k++) gW2[(int64_t)c * hidden + k] += e[c] * h[k];
            gb2[c] += e[c];
        }
        for (int32_t k = 0; k < hidden; k++) {              /* back through ReLU */
            double dh = 0.0;
            for (int32_t c = 0; c < classes; c++) dh += W2[(int64_t)c * hidden + k] * e[c];
            double da = a1[k] > 0.0 ? dh : 0.0;
            for (int32_t f = 0; f < in_dim; f++) gW1[(int64_t)k * in_dim + f] += da * (double)x[f];
            gb1[k] += da;
        }
    }
    if (grad) for (int64_t q = 0; q < dparams; q++) grad[q] = grad[q] / (double)b;
    if (min_abs_pre) *min_abs_pre = mn;
    free(a1); free(h); free(logit); free(e);
    return loss / (double)b;
}

/* ------------------------------------------------------------------------ */
/* NEXT-3: training multiple learners per GPU with per-GPU reference models  */
/* (Section 3.3, fig:multiple_learners PAPER.md:656-662;   */
/* formalised in SPEC.md S:327-335).  Reading R20:         */
/*   * GPU g (n GPUs, learners block-split as orc_replica_location) has a    */
/*     reference model u_g; GPU 0's reference model IS the central average   */
/*     model z ("It uses one of the local reference models as the central    */
/*     average model").  U[g] holds u_g for g >= 1; U[0]   */
/*     is not used.                                                          */
/*   * intra-GPU level ("each learner then computes the difference between   */
/*     its model replica and the local reference model. This difference is   */
/*     then applied to the respective replica"):    */
/*        d_j = alpha_l (w_j - u_g);  w_j <- w_j - gamma G_j - d_j;          */
/*        the reference model accumulates D_g = sum_{j on g} d_j.           */
/*   * inter-GPU level ("the SMA algorithm is executed ... all other         */
/*     reference models are the replicas"): Alg. 1 lines  */
/*     9-14 over the replicas u_1..u_{n-1} (no gradient of their own):      */
/*        c_g = alpha_g (u_g - z);  u_g <- u_g + D_g - c_g   (g >= 1)        */
/*        z   <- z + D_0 + sum_{g>=1} c_g + mu (z - z_prev);  z_prev <- old z */
/*   * every difference of a round is taken against the round-start values  */
/*     (the snapshot rule of Alg. 1 line 9, applied at both levels), and the */
/*     momentum term is Alg. 1's mu (z - z_prev) on round-start z / z_prev. */
/*     With n = 1 this is exactly Alg. 1 with alpha = alpha_l.       */
/* Sums in ascending local j, then ascending g.                              */
/*   W [k][m], U [n][m] (row 0 unused), z, zprev [m], G [k][m] raw gradients,*/
/*   part [n][m] scratch (part[g] = D_0 for g = 0, c_g for g >= 1).          */
/* ------------------------------------------------------------------------ */
void orc_hier_round(int64_t m, int32_t n, int32_t k, double alpha_l, double alpha_g,
                    double gamma, double mu, double *W, double *U, double *z, double *zprev,
                    const double *G, double *part) {
    for (int32_t g = 0; g < n; g++) {
        double *pg = part + (int64_t)g * m;
        const double *ref = (g == 0) ? z : U + (int64_t)g * m;  /* u_0 = z */
        for (int64_t p = 0; p < m; p++) pg[p] = 0.0;             /* D_g */
        for (int32_t j = 0; j < k; j++) {
            int32_t rank = -1, slot = -1;
            orc_replica_location(k, n, j, &rank, &slot);
            if (rank != g) continue;                             /* learners of GPU g */
            double *w = W + (int64_t)j * m;
            const double *Gj = G + (int64_t)j * m;
            for (int64_t p = 0; p < m; p++) {
                double gj = gamma * Gj[p];                       /* Alg. 1 line 8 */
                double dj = alpha_l * (w[p] - ref[p]);           /* difference to u_g */
                w[p] = w[p] - gj - dj;                           /* applied to the replica */
                pg[p] = pg[p] + dj;                              /* D_g, ascending j */
            }
        }
        if (g >= 1) {
            double *u = U + (int64_t)g * m;
            for (int64_t p = 0; p < m; p++) {
                double D = pg[p];
                double c = alpha_g * (u[p] - z[p]);              /* Alg. 1 line 9 over u_g */
                u[p] = u[p] + D - c;                             /* absorbs D_g; line 10, no gradient */
                pg[p] = c;
            }
        }
    }
    for (int64_t p = 0; p < m; p++) {
        double s = 0.0;
        for (int32_t g = 0; g < n; g++) s = s + part[(int64_t)g * m + p];  /* ascending g */
        double zold = z[p];                                               /* line 11 */
        z[p] = z[p] + s + mu * (z[p] - zprev[p]);                         /* line 13 */
        zprev[p] = zold;                                                  /* line 14 */
    }
}

/* R rounds of the two-level rule on the synthetic inputs at indices idx
 * (separable per index, as orc_sma_run_synth).  Init: z = z_prev = w0 (R2),
 * w_j = w0 (R3), u_g = w0 (every reference model starts as the initial
 * model, like the average model it stands for).
 * Outputs z, zprev [n_idx], and optionally W [k][n_idx], U [n][n_idx]. */
int orc_hier_run_synth(int64_t d, int32_t n, int32_t k, double alpha_l, double alpha_g,
                       double gamma, double mu, int64_t R, uint64_t seed_w, uint64_t seed_g,
                       int64_t n_idx, const int64_t *idx, double *z_out, double *zprev_out,
                       double *W_out, double *U_out) {
    double *W = (double *)malloc(sizeof(double) * (size_t)k * (size_t)n_idx);
    double *U = (double *)malloc(sizeof(double) * (size_t)n * (size_t)n_idx);
    double *G = (double *)malloc(sizeof(double) * (size_t)k * (size_t)n_idx);
    double *part = (double *)malloc(sizeof(double) * (size_t)n * (size_t)n_idx);
    if (!W || !U || !G || !part) { free(W); free(U); free(G); free(part); return -1; }
    orc_w0(n_idx, idx, seed_w, z_out);
    for (int64_t t = 0; t < n_idx; t++) zprev_out[t] = z_out[t];
    for (int32_t j = 0; j < k; j++) memcpy(W + (int64_t)j * n_idx, z_out, sizeof(double) * (size_t)n_idx);
    for (int32_t g = 0; g < n; g++) memcpy(U + (int64_t)g * n_idx, z_out, sizeof(double) * (size_t)n_idx);
    for (int64_t i = 0; i < R; i++) {
        for (int32_t j = 0; j < k; j++)
            orc_synth_grad(d, k, i, j, seed_g, n_idx, idx, G + (int64_t)j * n_idx);
        orc_hier_round(n_idx, n, k, alpha_l, alpha_g, gamma, mu, W, U, z_out, zprev_out, G, part);
    }
    if (W_out) memcpy(W_out, W, sizeof(double) * (size_t)k * (size_t)n_idx);
    if (U_out) {
        memcpy(U_out, U, sizeof(double) * (size_t)n * (size_t)n_idx);
        memcpy(U_out, z_out, sizeof(double) * (size_t)n_idx);   /* row 0: u_0 = z */
    }
    free(W); free(U); free(G); free(part);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Host-parallel timing variant (SURVEY.md §8d "Oracle timing (ii)").        */
/* Compiled only into liboracle_sma_omp.so (gcc -fopenmp): the sampled index */
/* set is cut into contiguous chunks and each chunk runs orc_sma_run_synth   */
/* unchanged on its own thread -- SMA with given gradients is separable per  */
/* parameter index, so the result equals the single-thread run bit for bit.  */
/* Returns the number of threads used, or -1 on allocation failure.          */
/* ------------------------------------------------------------------------ */
#ifdef _OPENMP
#include <omp.h>
int orc_sma_run_synth_omp(int64_t d, int32_t k, double alpha, double gamma, double mu,
                          int64_t R, uint64_t seed_w, uint64_t seed_g,
                          int64_t n_idx, const int64_t *idx, double *z_out, double *zprev_out) {
    int nt = omp_get_max_threads();
    int bad = 0;
    #pragma omp parallel for schedule(static) reduction(|:bad)
    for (int t = 0; t < nt; t++) {
        int64_t lo = n_idx * t / nt, hi = n_idx * (t + 1) / nt;
        if (hi > lo)
            bad |= orc_sma_run_synth(d, k, alpha, gamma, mu, R, seed_w, seed_g, hi - lo, idx + lo,
                                     z_out + lo, zprev_out + lo, NULL) != 0;
    }
    return bad ? -1 : nt;
}
#endif
