"""Exact-rational brute force of Algorithm 1.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Pure-Python loops over
``fractions.Fraction``: no rounding anywhere, so every identity the algebra
implies holds with equality.  Used on tiny cases only (the north_star's
hand-unrolled 2-replica, 4-parameter trace and k = 4), where dyadic inputs
keep the fp32 and fp64 computations exact for the first rounds (SURVEY.md
Appendix A6) and therefore bit-equal to this trace.

Readings: R1 gamma multiplies the raw gradient; R2 z_prev = w0 at
start; R3 w_j = w0 unless given; R7 corrections summed in ascending j.
"""
from __future__ import annotations

from fractions import Fraction


def _frac(x) -> Fraction:
    return x if isinstance(x, Fraction) else Fraction(x)


def sma_exact(w0, grads, alpha, gamma, mu, w_init=None):
    """Run len(grads) iterations of Alg. 1 exactly.

    w0     : list of d numbers (initial model, line 1)
    grads  : grads[i][j][p] raw gradient of learner j in round i (line 8 / R1)
    w_init : optional list of k initial replicas (R3 default: all w0)
    Returns a list of per-round states (z, z_prev, W) AFTER each round, with
    the initial state at position 0.
    """
    alpha, gamma, mu = _frac(alpha), _frac(gamma), _frac(mu)
    d = len(w0)
    k = len(grads[0]) if grads else len(w_init)
    z = [_frac(v) for v in w0]                       # line 1
    z_prev = list(z)                                 # line 2 (R2)
    if w_init is None:
        W = [list(z) for _ in range(k)]              # R3
    else:
        W = [[_frac(v) for v in row] for row in w_init]
    trace = [(list(z), list(z_prev), [list(r) for r in W])]
    for g_round in grads:                            # line 3 (R4: fixed rounds)
        c = [None] * k                               # line 4
        for j in range(k):                           # line 5
            g = [gamma * _frac(v) for v in g_round[j]]            # line 8
            c[j] = [alpha * (W[j][p] - z[p]) for p in range(d)]   # line 9
            W[j] = [W[j][p] - g[p] - c[j][p] for p in range(d)]   # line 10
        z_old = list(z)                                           # line 11
        csum = [sum((c[j][p] for j in range(k)), Fraction(0)) for p in range(d)]
        z = [z[p] + csum[p] + mu * (z[p] - z_prev[p]) for p in range(d)]  # line 13
        z_prev = z_old                                            # line 14
        trace.append((list(z), list(z_prev), [list(r) for r in W]))
    return trace


def hier_exact(w0, grads, n, alpha_l, alpha_g, gamma, mu, w_init=None, u_init=None):
    """Exact two-level rule of Section 3.3 (reading R20):
    per GPU g, d_j = alpha_l (w_j - u_g), w_j <- w_j - gamma G_j - d_j,
    D_g = sum d_j; for g >= 1, c_g = alpha_g (u_g - z), u_g <- u_g + D_g - c_g;
    z <- z + D_0 + sum_{g>=1} c_g + mu (z - z_prev), with u_0 = z and every
    difference against the round-start values.  Learners are block-split over
    the n GPUs (GPU g holds j with floor(g k/n) <= j < floor((g+1) k/n)).
    Returns per-round (z, z_prev, W, U) with U[0] = z, initial state first."""
    alpha_l, alpha_g = _frac(alpha_l), _frac(alpha_g)
    gamma, mu = _frac(gamma), _frac(mu)
    d = len(w0)
    k = len(grads[0]) if grads else len(w_init)
    gpu = [next(g for g in range(n) if g * k // n <= j < (g + 1) * k // n) for j in range(k)]
    z = [_frac(v) for v in w0]
    z_prev = list(z)
    W = [list(z) for _ in range(k)] if w_init is None else [[_frac(v) for v in r] for r in w_init]
    U = [list(z) for _ in range(n)] if u_init is None else [[_frac(v) for v in r] for r in u_init]
    U[0] = list(z)
    trace = [(list(z), list(z_prev), [list(r) for r in W], [list(r) for r in U])]
    for g_round in grads:
        ref = [list(z)] + [list(U[g]) for g in range(1, n)]     # round-start snapshots
        D = [[Fraction(0)] * d for _ in range(n)]
        for j in range(k):
            g = gpu[j]
            dj = [alpha_l * (W[j][p] - ref[g][p]) for p in range(d)]
            W[j] = [W[j][p] - gamma * _frac(g_round[j][p]) - dj[p] for p in range(d)]
            D[g] = [D[g][p] + dj[p] for p in range(d)]
        c = [None] + [[alpha_g * (ref[g][p] - z[p]) for p in range(d)] for g in range(1, n)]
        for g in range(1, n):
            U[g] = [U[g][p] + D[g][p] - c[g][p] for p in range(d)]
        z_old = list(z)
        z = [z[p] + D[0][p] + sum((c[g][p] for g in range(1, n)), Fraction(0))
             + mu * (z[p] - z_prev[p]) for p in range(d)]
        z_prev = z_old
        U[0] = list(z)
        trace.append((list(z), list(z_prev), [list(r) for r in W], [list(r) for r in U]))
    return trace
