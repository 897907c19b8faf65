"""Pins of the two-level oracle (per-GPU reference models, Section 3.3,
PAPER.md:664-690; reading R20 in DESIGN.md) against what the paper and the
mathematics fix -- not against a re-typed copy of its formula:

* the hierarchy collapses to flat Alg. 1 on one GPU;
* with alpha_g = 0 the levels decouple into one flat Alg. 1 per GPU with the
  reference model as its central model, and with alpha_l = 0,
  gamma = 0 the global level is flat Alg. 1 over the reference models as its
  replicas with GPU 0's reference model as z -- both
  against the independently pinned flat oracle, bitwise;
* a hand-derived closed form (n = 2, one learner per GPU, alpha = 1, mu = 0);
* the conservation law sum_j w_j + sum_{g>=1} u_g + z - mu z_prev (derived
  from the update rules; corrections cancel level by level);
* zero-gradient contraction of same-GPU replica spreads by (1 - alpha_l);
* the exact-rational brute force equal to the fp64 oracle bit for bit on
  dyadic inputs, and the quadratic testbed fixed point.
"""
from fractions import Fraction

import numpy as np
import pytest

import sma_inputs
from oracle import exact

F32 = lambda x: float(np.float32(x))  # noqa: E731


def _gpu_of(k, n):
    return [next(g for g in range(n) if g * k // n <= j < (g + 1) * k // n) for j in range(k)]


def _rand(orc, n, k, m, seed):
    rng = np.random.default_rng(seed)
    w0 = rng.uniform(-1, 1, m)
    W = w0 + rng.uniform(-0.5, 0.5, (k, m))
    U = w0 + rng.uniform(-0.5, 0.5, (n, m))
    st = orc.HierState.init(w0, k, n, W, U)
    st.z_prev = st.z - rng.uniform(-0.1, 0.1, m)
    return st, rng


@pytest.mark.parametrize("k", [1, 2, 5])
def test_one_gpu_collapses_to_flat_sma_bitwise(orc, k):
    """one device, k learners == flat Alg. 1 (the reference
    model is z itself), bitwise, for any alpha_g."""
    m, R = 19, 12
    st, rng = _rand(orc, 1, k, m, 1 + k)
    flat = orc.State(st.W, st.z, st.z_prev)
    for i in range(R):
        G = rng.uniform(-1, 1, (k, m))
        st.round(G, F32(1 / max(k, 2)), 0.37, F32(0.1), F32(0.9))
        flat.round(G, F32(1 / max(k, 2)), F32(0.1), F32(0.9))
        assert np.array_equal(st.z, flat.z) and np.array_equal(st.z_prev, flat.z_prev)
        assert np.array_equal(st.W, flat.W)


@pytest.mark.parametrize("n,k", [(2, 4), (3, 7), (4, 4)])
def test_alpha_g_zero_decouples_into_flat_sma_per_gpu(orc, n, k):
    """alpha_g = 0: no inter-GPU correction, so GPU g's learners and its
    reference model run flat Alg. 1 among themselves --
    GPU 0 with z and the momentum, GPU g >= 1 with u_g as its central model
    and no momentum -- bitwise equal to the flat oracle on each sub-problem."""
    m, R, al = 13, 10, F32(0.25)
    st, rng = _rand(orc, n, k, m, 10 + n)
    gpu = _gpu_of(k, n)
    subs = []
    for g in range(n):
        js = [j for j in range(k) if gpu[j] == g]
        if g == 0:
            subs.append((js, orc.State(st.W[js], st.z, st.z_prev), F32(0.9)))
        else:
            subs.append((js, orc.State(st.W[js], st.U[g], st.U[g]), 0.0))
    for i in range(R):
        G = rng.uniform(-1, 1, (k, m))
        st.round(G, al, 0.0, F32(0.1), F32(0.9))
        for g, (js, sub, mu) in enumerate(subs):
            sub.round(G[js], al, F32(0.1), mu)
            assert np.array_equal(st.W[js], sub.W)
            assert np.array_equal(st.U[g], sub.z)
    assert np.array_equal(st.z_prev, subs[0][1].z_prev)


@pytest.mark.parametrize("n,k", [(2, 2), (3, 6), (5, 5)])
def test_global_level_is_flat_sma_over_reference_models(orc, n, k):
    """alpha_l = 0, gamma = 0: the learners are inert and the global level is
    exactly Alg. 1 with the reference models u_1..u_{n-1} as its replicas and
    GPU 0's reference model as z, bitwise."""
    m, R, ag, mu = 11, 15, F32(0.3), F32(0.9)
    st, rng = _rand(orc, n, k, m, 20 + n)
    W0 = st.W.copy()
    flat = orc.State(st.U[1:], st.z, st.z_prev)
    for i in range(R):
        st.round(rng.uniform(-1, 1, (k, m)), 0.0, ag, 0.0, mu)
        flat.round(np.zeros((n - 1, m)), ag, 0.0, mu)
        assert np.array_equal(st.U[1:], flat.W)
        assert np.array_equal(st.z, flat.z) and np.array_equal(st.z_prev, flat.z_prev)
    assert np.array_equal(st.W, W0)


def test_closed_form_two_gpus_one_learner_each(orc):
    """n = 2, one learner per GPU, alpha_l = alpha_g = 1, mu = 0, derived by hand:
    w_0' = z - gamma g_0,  w_1' = u_1 - gamma g_1,  u_1' = w_1 - u_1 + z,
    z' = w_0 + u_1 - z."""
    m, gamma = 8, 0.125
    st, rng = _rand(orc, 2, 2, m, 30)
    for i in range(4):
        w0, w1, u1, z = st.W[0].copy(), st.W[1].copy(), st.U[1].copy(), st.z.copy()
        G = rng.uniform(-1, 1, (2, m))
        st.round(G, 1.0, 1.0, gamma, 0.0)
        np.testing.assert_allclose(st.W[0], z - gamma * G[0], rtol=0, atol=1e-14)
        np.testing.assert_allclose(st.W[1], u1 - gamma * G[1], rtol=0, atol=1e-14)
        np.testing.assert_allclose(st.U[1], w1 - u1 + z, rtol=0, atol=1e-14)
        np.testing.assert_allclose(st.z, w0 + u1 - z, rtol=0, atol=1e-14)
        np.testing.assert_array_equal(st.z_prev, z)


@pytest.mark.parametrize("n,k", [(2, 4), (3, 5), (4, 8)])
def test_conservation_law(orc, n, k):
    """I = sum_j w_j + sum_{g>=1} u_g + z - mu z_prev obeys
    I^{i+1} = I^i - gamma sum_j g_j^i for any alpha_l, alpha_g, mu (each
    difference d_j leaves a replica and enters its reference model; each c_g
    leaves u_g and enters z; the momentum cancels against -mu z_prev)."""
    m = 17
    al, ag, gamma, mu = 0.3, 0.45, 0.07, 0.85
    st, rng = _rand(orc, n, k, m, 40 + n)
    inv = lambda s: s.W.sum(0) + s.U[1:].sum(0) + s.z - mu * s.z_prev  # noqa: E731
    for i in range(30):
        I0 = inv(st)
        G = rng.uniform(-1, 1, (k, m))
        st.round(G, al, ag, gamma, mu)
        np.testing.assert_allclose(inv(st), I0 - gamma * G.sum(0), rtol=0, atol=1e-12)


def test_zero_gradient_same_gpu_spread_contracts(orc):
    """g = 0: two learners on the same GPU see the same reference model, so
    their difference shrinks by exactly (1 - alpha_l) per round; learners on
    different GPUs do not obey this."""
    n, k, m, al = 2, 4, 9, 0.2
    st, _ = _rand(orc, n, k, m, 50)
    Z = np.zeros((k, m))
    for i in range(10):
        same, cross = st.W[0] - st.W[1], st.W[0] - st.W[2]
        st.round(Z, al, 0.25, 0.3, 0.5)
        np.testing.assert_allclose(st.W[0] - st.W[1], (1 - al) * same, rtol=0, atol=1e-14)
    assert not np.allclose(st.W[0] - st.W[2], (1 - al) * cross, rtol=0, atol=1e-6)


def test_zero_gradient_consensus_and_fixed_point(orc):
    """g = 0 with stable parameters: every vector converges to the conserved
    I / (k + n - mu) (all equal => I = (k + (n-1) + 1 - mu) v); a state with
    all vectors equal and z = z_prev is an exact fixed point."""
    n, k, m = 2, 4, 5
    al, ag, mu = 0.25, 0.25, 0.5   # spectral radius 0.886 without the conserved mode
    st, _ = _rand(orc, n, k, m, 60)
    I = st.W.sum(0) + st.U[1:].sum(0) + st.z - mu * st.z_prev
    for i in range(2000):
        st.round(np.zeros((k, m)), al, ag, 0.1, mu)
    v = I / (k + n - mu)
    np.testing.assert_allclose(st.z, v, rtol=0, atol=1e-12)
    np.testing.assert_allclose(st.W, np.tile(v, (k, 1)), rtol=0, atol=1e-12)
    np.testing.assert_allclose(st.U, np.tile(v, (n, 1)), rtol=0, atol=1e-12)
    c = np.linspace(-1, 1, m)
    fp = orc.HierState.init(c, k, n)
    fp.round(np.zeros((k, m)), al, ag, 0.1, mu)
    assert np.array_equal(fp.z, c) and np.array_equal(fp.W, np.tile(c, (k, 1)))
    assert np.array_equal(fp.U, np.tile(c, (n, 1)))


def test_exact_trace_conserves_exactly():
    """The Fraction brute force satisfies the conservation law with equality."""
    n, k, d, R = 2, 4, 3, 6
    w0 = sma_inputs.dyadic(d, 70)
    G = sma_inputs.dyadic((R, k, d), 71)
    W_init = [[Fraction(v) + Fraction(j, 8) for v in w0] for j in range(k)]
    U_init = [[Fraction(v) - Fraction(g, 4) for v in w0] for g in range(n)]
    al, ag, gamma, mu = Fraction(1, 2), Fraction(1, 4), Fraction(1, 4), Fraction(1, 2)
    tr = exact.hier_exact(list(w0), G.tolist(), n, al, ag, gamma, mu, W_init, U_init)
    for i in range(R):
        (z0, zp0, W0, U0), (z1, zp1, W1, U1) = tr[i], tr[i + 1]
        for p in range(d):
            I0 = sum(r[p] for r in W0) + sum(U0[g][p] for g in range(1, n)) + z0[p] - mu * zp0[p]
            I1 = sum(r[p] for r in W1) + sum(U1[g][p] for g in range(1, n)) + z1[p] - mu * zp1[p]
            assert I1 == I0 - gamma * sum(Fraction(G[i][j][p]) for j in range(k))
            assert zp1[p] == z0[p]


@pytest.mark.parametrize("n,k,al,ag,rounds", [
    (2, 4, Fraction(1, 2), Fraction(1, 2), 8),
    (3, 5, Fraction(1, 4), Fraction(1, 2), 6),
])
def test_oracle_equals_exact_trace_bitwise(orc, n, k, al, ag, rounds):
    """On dyadic inputs the fp64 two-level oracle is exact for the first
    rounds, so it equals the exact-rational trace bit for bit."""
    d = 4
    w0 = sma_inputs.dyadic(d, 80 + n)
    G = sma_inputs.dyadic((rounds, k, d), 81 + n)
    gamma, mu = Fraction(1, 8), Fraction(1, 2)
    tr = exact.hier_exact(list(w0), G.tolist(), n, al, ag, gamma, mu)
    st = orc.HierState.init(w0, k, n)
    for i in range(rounds):
        st.round(G[i], float(al), float(ag), float(gamma), float(mu))
        z, zp, W, U = tr[i + 1]
        assert st.z.tolist() == [float(v) for v in z]
        assert st.z_prev.tolist() == [float(v) for v in zp]
        assert st.W.tolist() == [[float(v) for v in row] for row in W]
        assert st.U.tolist() == [[float(v) for v in row] for row in U]


def test_quadratic_converges_to_minimiser(orc):
    """The quadratic testbed of SPEC.md:742 under the two-level rule (n = 2 GPUs
    x 2 learners, alpha_l = 1/(2r), alpha_g = 1/(2(n-1)): z's total pull
    alpha_l r + alpha_g (n-1) = 1, like alpha = 1/k in flat Alg. 1): z -> w*,
    and w* is an exact fixed point of every vector."""
    dim, n, k = 50, 2, 4
    a, ws = sma_inputs.quadratic(dim)
    al, ag, gamma, mu = F32(0.25), F32(0.5), F32(0.05), F32(0.9)
    st = orc.HierState.init(np.zeros(dim), k, n)
    for i in range(4000):
        st.round((a * a) * (st.W - ws), al, ag, gamma, mu)
        if np.max(np.abs(st.z - ws)) < 1e-3:
            break
    assert np.max(np.abs(st.z - ws)) < 1e-3, i
    fp = orc.HierState.init(ws, k, n)
    fp.round(np.zeros((k, dim)), al, ag, gamma, mu)
    assert np.array_equal(fp.z, ws) and np.array_equal(fp.W, np.tile(ws, (k, 1)))


def test_hier_run_synth_composes_rounds(orc):
    """hier_run_synth == init (z = z_prev = w_j = u_g = w0) + R rounds with the
    synthetic gradients of the shared input module; sampled indices equal the
    full run (separability)."""
    d, n, k, R = 301, 3, 7, 5
    al, ag, g, m = F32(0.5), F32(1 / 3), F32(0.1), F32(0.9)
    z, zp, W, U = orc.hier_run_synth(d, n, k, al, ag, g, m, R, 1901, 2244)
    st = orc.HierState.init(sma_inputs.w0(d), k, n)
    for i in range(R):
        st.round(np.stack([sma_inputs.grad(i, j, k, d) for j in range(k)]), al, ag, g, m)
    assert np.array_equal(st.z, z) and np.array_equal(st.W, W) and np.array_equal(st.U, U)
    idx = np.array([0, 5, 150, 300])
    zs, zps, Ws, Us = orc.hier_run_synth(d, n, k, al, ag, g, m, R, 1901, 2244, idx)
    assert np.array_equal(zs, z[idx]) and np.array_equal(Ws, W[:, idx])
    assert np.array_equal(Us, U[:, idx]) and np.array_equal(zps, zp[idx])
