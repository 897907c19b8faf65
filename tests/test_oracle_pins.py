"""Pins of the oracle against what the paper and the mathematics fix.

Each test names the passage or identity it pins.  None of them re-types the
oracle's own formula: they check worked examples, special cases
that reduce to textbook algorithms (SGD, plain averaging), closed forms and
invariants derived from Alg. 1, an exact-rational
brute force, and published generator vectors.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import sma_inputs
from oracle import exact

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
F32 = lambda x: float(np.float32(x))  # noqa: E731  (R6: fp32 hyper-parameters)


# ------------------------------------------------------------------ generator
def test_splitmix64_published_vectors(orc):
    """Published splitmix64 outputs (tests/golden/splitmix64_vectors.json)."""
    g = json.load(open(os.path.join(GOLDEN, "splitmix64_vectors.json")))
    for n, want in enumerate(g["outputs"]):
        x = (g["seed"] + n * sma_inputs.GOLDEN) % 2**64
        assert orc.splitmix64(x) == int(want)
        assert sma_inputs.splitmix64_int(x) == int(want)


def test_generator_sides_agree_and_are_fp32_exact(orc):
    """The oracle's own generator equals the shared input module bit for bit,
    and every value is exactly representable in fp32 (R9)."""
    d, k = 1000, 3
    idx = np.arange(d)
    w_np = sma_inputs.w0(d)
    w_or = orc.w0(d, sma_inputs.SEED_W, idx)
    assert np.array_equal(w_np.astype(np.float64), w_or)
    assert np.all(np.abs(w_or) <= 1 / 16)
    for rnd, j in [(0, 0), (5, 2), (99, 1)]:
        g_np = sma_inputs.grad(rnd, j, k, d)
        g_or = orc.synth_grad(d, k, rnd, j, sma_inputs.SEED_G, idx)
        assert np.array_equal(g_np.astype(np.float64), g_or)
        assert np.array_equal(g_or.astype(np.float32).astype(np.float64), g_or)
        assert np.all(np.abs(g_or) <= 1 / 32)
    # the counters of different (round, learner) pairs do not overlap
    assert not np.array_equal(orc.synth_grad(d, k, 0, 1, 2244, idx),
                              orc.synth_grad(d, k, 1, 0, 2244, idx))
    # uniform24 mean and range (a plausible shift/scale mistake breaks this)
    u = np.array([orc.uniform24(9, c) for c in range(4000)])
    assert u.min() >= 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.02


# ------------------------------------------------------------ worked examples
def test_spec_scalar_examples(orc):
    """SPEC.md:265-300 worked examples (tests/golden/spec_scalar_examples.json)."""
    g = json.load(open(os.path.join(GOLDEN, "spec_scalar_examples.json")))
    for ex in g["examples"]:
        st = orc.State(ex["W"], ex["z"], ex["z_prev"])
        st.round(ex["G"], ex["alpha"], ex["gamma"], ex["mu"])
        np.testing.assert_allclose(st.W, ex["W_after"], rtol=0, atol=1e-15, err_msg=ex["cite"])
        if "z_after" in ex:
            np.testing.assert_allclose(st.z, ex["z_after"], rtol=0, atol=1e-15, err_msg=ex["cite"])
            np.testing.assert_allclose(st.z_prev, ex["z_prev_after"], rtol=0, atol=1e-15)


# ---------------------------------------------------------- special cases
def _rand_state(orc, k, m, seed, distinct=True):
    rng = np.random.default_rng(seed)
    w0 = rng.uniform(-1, 1, m)
    W = w0 + (rng.uniform(-0.5, 0.5, (k, m)) if distinct else 0)
    return orc.State.init(w0, k, W), rng


def test_alpha_zero_is_independent_sgd(orc):
    """alpha = 0: c_j = 0, so each replica runs mini-batch SGD (Eq. 1,
    PAPER.md:220-223) and z stays w0 for any mu."""
    k, m, R = 3, 17, 25
    gamma, mu = F32(0.1), F32(0.9)
    st, rng = _rand_state(orc, k, m, 1)
    W0, z0 = st.W.copy(), st.z.copy()
    Gs = rng.uniform(-1, 1, (R, k, m))
    for i in range(R):
        st.round(Gs[i], 0.0, gamma, mu)
    assert np.array_equal(st.z, z0) and np.array_equal(st.z_prev, z0)   # bitwise
    sgd = W0.copy()
    for i in range(R):                                                  # Eq. 1
        sgd = sgd - gamma * Gs[i]
    np.testing.assert_allclose(st.W, sgd, rtol=0, atol=1e-13)


def test_alpha_1_over_k_mu_zero_gives_mean_of_replicas(orc):
    """alpha = 1/k, mu = 0: z^{i+1} = z^i + (1/k) sum_j (w_j^i - z^i) = mean_j w_j^i,
    the pre-step replicas (Alg. 1 lines 9, 13 with all c_j against one z)."""
    k, m = 4, 33
    st, rng = _rand_state(orc, k, m, 2)
    for i in range(6):
        pre = st.W.copy()
        st.round(rng.uniform(-1, 1, (k, m)), 1.0 / k, F32(0.1), 0.0)
        np.testing.assert_allclose(st.z, pre.mean(axis=0), rtol=0, atol=1e-14)


def test_k1_alpha1_leapfrog(orc):
    """k = 1, alpha = 1, mu = 0 (SURVEY Q14 reading of the north_star's k=1
    claim): z^{i+1} = w^i and w^{i+1} = z^i - gamma g^i (to fp64 rounding)."""
    m = 9
    st, rng = _rand_state(orc, 1, m, 3)
    gamma = F32(0.1)
    for i in range(5):
        w_pre, z_pre = st.W[0].copy(), st.z.copy()
        g = rng.uniform(-1, 1, (1, m))
        st.round(g, 1.0, gamma, 0.0)
        np.testing.assert_allclose(st.z, w_pre, rtol=0, atol=1e-15)
        np.testing.assert_allclose(st.W[0], z_pre - gamma * g[0], rtol=0, atol=1e-15)


def test_conservation_law(orc):
    """I = sum_j w_j + z - mu z_prev obeys I^{i+1} = I^i - gamma sum_j g_j^i for
    any alpha, mu (sum lines 10 and 13 of Alg. 1: the corrections cancel)."""
    k, m = 5, 21
    alpha, gamma, mu = 0.3, 0.07, 0.85
    st, rng = _rand_state(orc, k, m, 4)
    for i in range(30):
        I0 = st.W.sum(0) + st.z - mu * st.z_prev
        G = rng.uniform(-1, 1, (k, m))
        st.round(G, alpha, gamma, mu)
        I1 = st.W.sum(0) + st.z - mu * st.z_prev
        np.testing.assert_allclose(I1, I0 - gamma * G.sum(0), rtol=0, atol=1e-12)


def test_zero_gradient_contraction(orc):
    """g = 0: (w_j - w_l) shrinks by (1 - alpha) per round; with mu = 0,
    D = sum_j (w_j - z) scales by (1 - alpha (k + 1))."""
    k, m, alpha = 4, 11, 0.2
    st, _ = _rand_state(orc, k, m, 5)
    Z = np.zeros((k, m))
    for i in range(10):
        spread = st.W[0] - st.W[2]
        D = (st.W - st.z).sum(0)
        st.round(Z, alpha, 0.3, 0.0)
        np.testing.assert_allclose(st.W[0] - st.W[2], (1 - alpha) * spread, rtol=0, atol=1e-14)
        np.testing.assert_allclose((st.W - st.z).sum(0), (1 - alpha * (k + 1)) * D,
                                   rtol=0, atol=1e-13)


def test_fixed_point_mu_zero_z_is_mean(orc):
    """mu = 0 fixed point (north_star): with g = 0 the iteration converges and at
    the limit z equals the mean of the replicas (and all replicas agree)."""
    k, m = 4, 7
    st, _ = _rand_state(orc, k, m, 6)
    for i in range(400):
        st.round(np.zeros((k, m)), 1.0 / k, 0.1, 0.0)
    np.testing.assert_allclose(st.z, st.W.mean(0), rtol=0, atol=1e-12)
    np.testing.assert_allclose(st.W, np.tile(st.z, (k, 1)), rtol=0, atol=1e-12)


def test_quadratic_converges_to_minimiser(orc):
    """SPEC.md:742 (AC3): on l = 1/2 ||A(w - w*)||^2 (diag A, cond <= 10), SMA with
    k=4, alpha=1/4, gamma=0.05, mu=0.9 drives ||z - w*||_inf below 1e-3; and
    w_j = z = z_prev = w* is an exact fixed point."""
    dim, k = 50, 4
    a, ws = sma_inputs.quadratic(dim)
    alpha, gamma, mu = F32(0.25), F32(0.05), F32(0.9)
    st = orc.State.init(np.zeros(dim), k)
    for i in range(3000):
        G = (a * a) * (st.W - ws)            # closed-form gradient of the quadratic
        st.round(G, alpha, gamma, mu)
        if np.max(np.abs(st.z - ws)) < 1e-3:
            break
    assert np.max(np.abs(st.z - ws)) < 1e-3, i
    fp = orc.State.init(ws, k)
    fp.round(np.zeros((k, dim)), alpha, gamma, mu)
    assert np.array_equal(fp.z, ws) and np.array_equal(fp.W, np.tile(ws, (k, 1)))


# ------------------------------------------------------ exact brute force
def _dyadic_case(k, d, R, seed):
    w0 = sma_inputs.dyadic(d, seed)
    G = sma_inputs.dyadic((R, k, d), seed + 1)
    return w0, G


def test_exact_trace_satisfies_identities_exactly():
    """The Fraction brute force (the north_star's hand-unrolled 2-replica,
    4-parameter trace) satisfies the closed forms with equality."""
    k, d, R = 2, 4, 12
    w0, G = _dyadic_case(k, d, R, 10)
    W_init = [[Fraction(v) + Fraction(j, 8) for v in w0] for j in range(k)]
    alpha, gamma, mu = Fraction(1, 2), Fraction(1, 4), Fraction(1, 2)
    tr = exact.sma_exact(list(w0), G.tolist(), alpha, gamma, mu, w_init=W_init)
    for i in range(R):
        z0, zp0, W0 = tr[i]
        z1, zp1, W1 = tr[i + 1]
        for p in range(d):
            I0 = sum(W0[j][p] for j in range(k)) + z0[p] - mu * zp0[p]
            I1 = sum(W1[j][p] for j in range(k)) + z1[p] - mu * zp1[p]
            assert I1 == I0 - gamma * sum(Fraction(G[i][j][p]) for j in range(k))
            assert zp1[p] == z0[p]
    # alpha = 1/k, mu = 0 -> z^{i+1} is exactly the mean of the pre-step replicas
    tr = exact.sma_exact(list(w0), G.tolist(), Fraction(1, 2), gamma, 0, w_init=W_init)
    for i in range(R):
        W0 = tr[i][2]
        assert tr[i + 1][0] == [(W0[0][p] + W0[1][p]) / 2 for p in range(d)]


@pytest.mark.parametrize("k,alpha,gamma,mu,rounds", [
    (2, Fraction(1, 2), Fraction(1, 4), Fraction(1, 2), 8),   # north_star 2x4 trace
    (4, Fraction(1, 4), Fraction(1, 8), Fraction(1, 2), 8),
])
def test_oracle_equals_exact_trace_bitwise(orc, k, alpha, gamma, mu, rounds):
    """On dyadic inputs the fp64 oracle is exact for the first rounds (SURVEY
    Appendix A6), so it must equal the exact-rational trace bit for bit."""
    d = 4
    w0, G = _dyadic_case(k, d, rounds, 20 + k)
    tr = exact.sma_exact(list(w0), G.tolist(), alpha, gamma, mu)
    st = orc.State.init(w0, k)
    for i in range(rounds):
        st.round(G[i], float(alpha), float(gamma), float(mu))
        z, zp, W = tr[i + 1]
        assert st.z.tolist() == [float(v) for v in z]
        assert st.z_prev.tolist() == [float(v) for v in zp]
        assert st.W.tolist() == [[float(v) for v in row] for row in W]


def test_sampled_indices_equal_full_vector(orc):
    """SMA with given gradients is separable per parameter index, so the
    sampled-index oracle used at C4/C5 size equals the full run bitwise."""
    d, k, R = 3001, 4, 7
    z, zp, W = orc.run_synth(d, k, F32(0.25), F32(0.1), F32(0.9), R, 1901, 2244)
    idx = np.array([0, 1, 17, 1500, 2999, 3000])
    zs, zps, Ws = orc.run_synth(d, k, F32(0.25), F32(0.1), F32(0.9), R, 1901, 2244, idx)
    assert np.array_equal(zs, z[idx]) and np.array_equal(zps, zp[idx])
    assert np.array_equal(Ws, W[:, idx])


def test_run_synth_composes_rounds(orc):
    """run_synth == init (lines 1-2, R2, R3) + R rounds with the synthetic
    gradients from the shared input module."""
    d, k, R = 257, 3, 5
    a, g, m = F32(1 / 3), F32(0.1), F32(0.9)
    z, zp, W = orc.run_synth(d, k, a, g, m, R, 1901, 2244)
    st = orc.State.init(sma_inputs.w0(d), k)
    for i in range(R):
        st.round(np.stack([sma_inputs.grad(i, j, k, d) for j in range(k)]), a, g, m)
    assert np.array_equal(st.z, z) and np.array_equal(st.W, W)


# ------------------------------------------------------------- softmax learner
def _blobs_small():
    return sma_inputs.blobs(200, dim=784, classes=10, seed=3)


def test_softmax_loss_at_zero_is_ln10(orc):
    """LOGREG with w = 0 has loss ln(10) (uniform softmax)."""
    X, y = _blobs_small()
    loss, g = orc.softmax_loss_grad(X, y, np.arange(16), np.zeros(7850))
    assert abs(loss - math.log(10)) < 1e-12
    # with w = 0, db_c = mean_t (1/10 - [y_t = c]) and the class sums vanish
    assert abs(g[7840:].sum()) < 1e-15
    cnt = np.bincount(y[:16], minlength=10)
    np.testing.assert_allclose(g[7840:], 0.1 - cnt / 16, atol=1e-15)


def test_softmax_gradient_finite_differences(orc):
    """analytic gradient vs central finite differences of the loss."""
    X, y = _blobs_small()
    rng = np.random.default_rng(0)
    w = rng.normal(0, 0.01, 7850)
    rows = np.arange(5, 21)
    _, g = orc.softmax_loss_grad(X, y, rows, w)
    h = 1e-5
    for q in list(rng.integers(0, 7850, 25)) + [7840, 7849, 0, 783]:
        wp, wm = w.copy(), w.copy()
        wp[q] += h
        wm[q] -= h
        fd = (orc.softmax_loss_grad(X, y, rows, wp, want_grad=False)[0]
              - orc.softmax_loss_grad(X, y, rows, wm, want_grad=False)[0]) / (2 * h)
        assert abs(fd - g[q]) < 1e-7, q


def test_softmax_gradient_is_batch_mean(orc):
    """Eq. 2 / SPEC.md:131-132: the batch gradient is the mean
    of the per-sample gradients, so duplicating the batch leaves it unchanged."""
    X, y = _blobs_small()
    w = np.random.default_rng(1).normal(0, 0.01, 7850)
    rows = np.array([3, 9, 40, 41])
    _, g = orc.softmax_loss_grad(X, y, rows, w)
    per = [orc.softmax_loss_grad(X, y, [r], w)[1] for r in rows]
    np.testing.assert_allclose(g, np.mean(per, axis=0), rtol=0, atol=1e-15)
    _, g2 = orc.softmax_loss_grad(X, y, np.concatenate([rows, rows]), w)
    np.testing.assert_allclose(g2, g, rtol=0, atol=1e-15)


def test_softmax_sma_learns_blobs(orc):
    """End-to-end: Alg. 1 with the softmax learner on separable blobs drives the
    central model's training accuracy to 1.0 (SPEC.md:646 property)."""
    X, y = sma_inputs.blobs(2000, seed=4)
    k = 4
    z, _, _ = orc.run_softmax(X, y, 16, 77, k, F32(1 / k), F32(0.1), F32(0.9), 30,
                              np.zeros(7850))
    logits = X.astype(np.float64) @ z[:7840].reshape(10, 784).T + z[7840:]
    assert np.mean(np.argmax(logits, 1) == y) > 0.99


def test_run_softmax_composes_pieces(orc):
    """run_softmax == batch_indices + softmax_loss_grad at the pre-step replica +
    one Alg. 1 round, for every round."""
    X, y = sma_inputs.blobs(640, seed=5)
    k, b, R = 2, 16, 4
    a, g, m = F32(0.5), F32(0.1), F32(0.9)
    w0 = np.random.default_rng(2).normal(0, 0.01, 7850)
    z, zp, W = orc.run_softmax(X, y, b, 9, k, a, g, m, R, w0)
    st = orc.State.init(w0, k)
    for i in range(R):
        G = np.stack([orc.softmax_loss_grad(X, y, orc.batch_indices(640, k, b, 9, i, j), st.W[j])[1]
                      for j in range(k)])
        st.round(G, a, g, m)
    assert np.array_equal(st.z, z) and np.array_equal(st.W, W)


# ------------------------------------------------------------- bookkeeping
@pytest.mark.parametrize("k,n", [(1, 1), (4, 1), (16, 8), (16, 3), (5, 4), (3, 8), (32, 8)])
def test_replica_map_is_balanced_block_split(orc, k, n):
    """Replica j -> (rank, slot): each j exactly once, ranks contiguous and
    ascending, per-rank counts within one of k/n (k = m x #GPUs)."""
    locs = [orc.replica_location(k, n, j) for j in range(k)]
    counts = np.bincount([r for r, _ in locs], minlength=n)
    assert counts.sum() == k and counts.max() - counts.min() <= 1
    assert [r for r, _ in locs] == sorted(r for r, _ in locs)
    for g in range(n):
        assert [s for r, s in locs if r == g] == list(range(counts[g]))
    with pytest.raises(ValueError):
        orc.replica_location(k, n, k)


@pytest.mark.parametrize("d,n", [(1, 1), (7, 4), (7850, 1), (464154, 8), (25557032, 8),
                                 (138357544, 8), (1000, 3), (513, 2)])
def test_shard_table_partitions_padded_vector(orc, d, n):
    """Shards partition [0, d_pad) into n equal, 256-byte-aligned pieces; the
    padding is minimal for the alignment (all-reduce partitions)."""
    dp = orc.d_pad(d, n)
    assert dp >= d and dp % 512 == 0 and dp % (64 * n) == 0 and dp - d < math.lcm(512, 64 * n)
    ends = 0
    for g in range(n):
        off, ln = orc.shard_range(d, n, g)
        assert off == ends and ln == dp // n and ln % 64 == 0
        ends = off + ln
    assert ends == dp
    if (d, n) == (25557032, 8):
        assert dp == 25557504
    if (d, n) == (138357544, 8):
        assert dp == 138357760


def test_epoch_permutation_is_uniform_fisher_yates(orc):
    """Fisher-Yates must produce every permutation of [0,3) with equal
    probability (a Sattolo-style off-by-one produces only the 2 cycles)."""
    counts = {}
    T = 6000
    for e in range(T):
        p = tuple(orc.epoch_permutation(3, 123, e))
        counts[p] = counts.get(p, 0) + 1
    assert len(counts) == 6
    chi2 = sum((c - T / 6) ** 2 / (T / 6) for c in counts.values())
    assert chi2 < 25.0        # 5 dof, p ~ 1e-4
    p = orc.epoch_permutation(1000, 5, 2)
    assert sorted(p.tolist()) == list(range(1000))
    assert np.array_equal(p, orc.epoch_permutation(1000, 5, 2))
    assert not np.array_equal(p, orc.epoch_permutation(1000, 5, 3))


def test_batches_within_an_epoch_are_disjoint(orc):
    """select(B) removes the batch (Alg. 1 lines 6-7): within
    one epoch no sample is used twice; rounds of the next epoch start over."""
    N, k, b = 200, 3, 8
    E = N // (k * b)
    seen = []
    for i in range(E):
        for j in range(k):
            seen.extend(orc.batch_indices(N, k, b, 42, i, j).tolist())
    assert len(set(seen)) == len(seen) == E * k * b and min(seen) >= 0 and max(seen) < N
    nxt = orc.batch_indices(N, k, b, 42, E, 0)
    assert np.array_equal(nxt, orc.epoch_permutation(N, 42, 1)[:b])


# ------------------------------------------------ NEXT-3 / NEXT-4 functions
def test_local_round_is_sgd_and_leaves_z(orc):
    """tau > 1 local iterations (R17): tau local rounds equal tau rounds
    of alpha = 0 SMA on the replicas (itself pinned to Eq. 1 above), and leave z,
    z_prev untouched; with tau = 1 the schedule is plain SMA."""
    k, m, tau = 3, 13, 4
    st, rng = _rand_state(orc, k, m, 30)
    ref = orc.State(st.W, st.z, st.z_prev)
    z0, zp0 = st.z.copy(), st.z_prev.copy()
    for i in range(tau):
        G = rng.uniform(-1, 1, (k, m))
        st.local_round(G, F32(0.1))
        ref.round(G, 0.0, F32(0.1), 0.0)
    np.testing.assert_allclose(st.W, ref.W, rtol=0, atol=1e-15)
    assert np.array_equal(st.z, z0) and np.array_equal(st.z_prev, zp0)


def test_alg2_worked_examples(orc):
    """Alg. 2 lines 7-9 on SPEC's examples (tests/golden/alg2_examples.json)."""
    g = json.load(open(os.path.join(GOLDEN, "alg2_examples.json")))
    for ex in g["examples"]:
        l, tp = orc.autotune_step(ex["tau"], [ex["t"]], [ex["l"]], [ex["t_prev"]])
        assert l[0] == ex["l_after"] and tp[0] == ex["t"]


def test_alg2_settles_at_throughput_peak(orc):
    """S:500 / S:745 (AC6): against a concave throughput curve peaking at l* = 3
    the tuner reaches l in {3, 4} within 6 rounds, oscillates by at most one
    afterwards and never reaches 0 (add on increase > tau, remove on
    decrease).  Two GPUs with different curves adapt independently."""
    f = [lambda l: 100.0 - 10.0 * (l - 3) ** 2, lambda l: 80.0 - 2.0 * (l - 5) ** 2]
    l, tp = np.array([1, 1]), np.array([0.0, 0.0])   # Alg. 2 lines 1-2
    hist = []
    for it in range(20):
        t = [f[g](l[g]) for g in range(2)]
        l, tp = orc.autotune_step(4.0, t, l, tp)
        hist.append(l.copy())
    assert all(h[0] >= 1 and h[1] >= 1 for h in hist)
    assert all(h[0] in (3, 4) for h in hist[5:])
    assert all(h[1] in (5, 6) for h in hist[10:])


def test_resize_keeps_replicas_and_seeds_from_z(orc):
    """an added replica starts from the current central model; the
    kept replicas of every GPU are unchanged (uniform count per GPU)."""
    n, l, m = 2, 3, 5
    st, _ = _rand_state(orc, n * l, m, 31)
    W0 = st.W.copy()
    st.resize(n, 5)
    assert st.W.shape == (n * 5, m)
    for g in range(n):
        assert np.array_equal(st.W[g * 5:g * 5 + 3], W0[g * 3:g * 3 + 3])
        assert np.array_equal(st.W[g * 5 + 3], st.z) and np.array_equal(st.W[g * 5 + 4], st.z)
    st.resize(n, 2)
    for g in range(n):
        assert np.array_equal(st.W[g * 2:g * 2 + 2], W0[g * 3:g * 3 + 2])


# ------------------------------------------------------------- MLP learner
def _mlp_point(seed, scale=0.05):
    rng = np.random.default_rng(seed)
    return rng.normal(0, scale, orc_mlp_d())


def orc_mlp_d():
    import oracle
    return oracle.mlp_dims()


def test_mlp_loss_at_zero_is_ln10(orc):
    """MLP with w = 0 has loss ln(10) (zero hidden activations
    still give a uniform softmax); only the output bias gets a gradient."""
    X, y = _blobs_small()
    loss, g, _ = orc.mlp_loss_grad(X, y, np.arange(16), np.zeros(orc.mlp_dims()))
    assert abs(loss - math.log(10)) < 1e-12
    nb2 = orc.mlp_dims() - 10
    assert np.all(g[:nb2] == 0)
    cnt = np.bincount(y[:16], minlength=10)
    np.testing.assert_allclose(g[nb2:], 0.1 - cnt / 16, atol=1e-15)


def test_mlp_gradient_finite_differences(orc):
    """SPEC.md:130 / S:148: analytic gradient vs central differences, on
    parameters of both layers and both biases (away from ReLU kinks)."""
    X, y = _blobs_small()
    w = _mlp_point(1)
    rows = np.arange(3, 11)
    _, g, mn = orc.mlp_loss_grad(X, y, rows, w)
    h = 1e-6
    assert mn > 10 * h * np.abs(X).max()      # no probe crosses a ReLU kink
    rng = np.random.default_rng(2)
    D = orc.mlp_dims()
    probes = list(rng.integers(0, 256 * 784, 12)) + list(range(200704, 200714)) + \
        list(rng.integers(200960, D, 12))
    for q in probes:
        wp, wm = w.copy(), w.copy()
        wp[q] += h
        wm[q] -= h
        fd = (orc.mlp_loss_grad(X, y, rows, wp, want_grad=False)[0]
              - orc.mlp_loss_grad(X, y, rows, wm, want_grad=False)[0]) / (2 * h)
        assert abs(fd - g[q]) < 1e-7, q


def test_mlp_gradient_is_batch_mean(orc):
    """Eq. 2: batch gradient = mean of per-sample gradients."""
    X, y = _blobs_small()
    w = _mlp_point(3)
    rows = np.array([0, 7, 19])
    _, g, _ = orc.mlp_loss_grad(X, y, rows, w)
    per = [orc.mlp_loss_grad(X, y, [r], w)[1] for r in rows]
    np.testing.assert_allclose(g, np.mean(per, axis=0), rtol=0, atol=1e-15)


def test_openmp_timing_variant_equals_serial_oracle(orc):
    """The host-parallel timing variant (bench cpu_baseline.all_cores) splits the
    index set over threads; separability makes it bitwise equal to the serial
    oracle."""
    idx = np.arange(3, 50_000, 11)
    z, zp, _ = orc.run_synth(50_000, 4, F32(0.25), F32(0.1), F32(0.9), 6, 1901, 2244, idx,
                             want_W=False)
    z2, zp2, nt = orc.run_synth_omp(50_000, 4, F32(0.25), F32(0.1), F32(0.9), 6, 1901, 2244, idx)
    assert nt >= 1 and np.array_equal(z, z2) and np.array_equal(zp, zp2)
