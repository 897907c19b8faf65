"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the SMA method (arXiv 1901.02244, Alg. 1,
PAPER.md:544-599).  It only produces the inputs both sides consume: the initial
model w0, the synthetic per-learner gradients g_j^i, an MNIST-shaped labelled
dataset for the built-in softmax learner, and a quadratic test objective.

Counter-based generator.  Every
side that needs these numbers at full size (the CUDA ``synth_fill`` kernel and
the C oracle) re-implements the same four lines independently:

    splitmix64(x) = mix(x + 0x9E3779B97F4A7C15)
        mix(z): z = (z ^ z>>30) * 0xBF58476D1CE4E5B9
                z = (z ^ z>>27) * 0x94D049BB133111EB
                return z ^ z>>31                        (all mod 2^64)
    key(seed)     = splitmix64(seed)
    U(seed, ctr)  = (splitmix64(key(seed) + ctr) >> 40) * 2^-24        in [0, 1)
    w0[p]         = (U(SEED_W, p) - 1/2) * 2^-3                         in [-1/16, 1/16)
    g_j^i[p]      = (U(SEED_G, (i*k + j)*d + p) - 1/2) * 2^-4           in [-1/32, 1/32)

Both values are exact in fp32 (24 significant bits), so the GPU and the fp64
oracle see bit-identical inputs.
"""
from __future__ import annotations

import numpy as np

SEED_W = 1901
SEED_G = 2244
GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1

# The paper's model sizes as BASELINE.json fixes them.
CONFIGS = {
    "C1": dict(name="softmax", d=7_850, k=4, n=1, batch=16),
    "C2": dict(name="lenet", d=431_080, k=8, n=1, batch=4),
    "C3": dict(name="resnet32", d=464_154, k=16, n=8, batch=64),
    "C4": dict(name="resnet50", d=25_557_032, k=16, n=8, batch=16),
    "C5": dict(name="vgg16", d=138_357_544, k=32, n=8, batch=16),
    # NEXT-2: the MLP learner in the loop, MNIST-shaped
    "MLP": dict(name="mlp784-256-10", d=256 * 784 + 256 + 10 * 256 + 10, k=4, n=1, batch=16),
}


def splitmix64_int(x: int) -> int:
    """Scalar splitmix64 on Python ints (reference for the vector form)."""
    z = (x + GOLDEN) & _MASK
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 over a uint64 array (wrapping arithmetic)."""
    z = np.asarray(x, dtype=np.uint64) + np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def uniform24(seed: int, ctr: np.ndarray) -> np.ndarray:
    """U(seed, ctr) as float64 in [0, 1) with 24 random bits."""
    key = np.uint64(splitmix64_int(seed))
    h = splitmix64(np.asarray(ctr, dtype=np.uint64) + key)
    return (h >> np.uint64(40)).astype(np.float64) * 2.0 ** -24


def w0(d: int, seed: int = SEED_W, idx: np.ndarray | None = None) -> np.ndarray:
    """Initial model w0 (fp32, exact).  ``idx`` selects parameter indices."""
    p = np.arange(d, dtype=np.uint64) if idx is None else np.asarray(idx, dtype=np.uint64)
    return ((uniform24(seed, p) - 0.5) * 0.125).astype(np.float32)


def grad(rnd: int, j: int, k: int, d: int, seed: int = SEED_G,
         idx: np.ndarray | None = None) -> np.ndarray:
    """Synthetic raw gradient g_j^i (fp32, exact); gamma is NOT applied."""
    p = np.arange(d, dtype=np.uint64) if idx is None else np.asarray(idx, dtype=np.uint64)
    base = np.uint64((rnd * k + j) * d)
    return ((uniform24(seed, p + base) - 0.5) * 0.0625).astype(np.float32)


def dyadic(shape, seed: int, lo: int = -8, hi: int = 8) -> np.ndarray:
    """Values on the 1/8 grid of [-1, 1] (exact in every float format)."""
    rng = np.random.default_rng(seed)
    return (rng.integers(lo, hi + 1, size=shape) / 8.0).astype(np.float64)


def blobs(n: int, dim: int = 784, classes: int = 10, sigma: float = 0.25,
          seed: int = 7) -> tuple[np.ndarray, np.ndarray]:
    """MNIST-shaped separable blobs (SPEC.md:641-649 recipe, synthetic).

    Class centres are uniform in [0,1]^dim (pairwise distance ~ sqrt(dim/6)
    = 11.4 for dim 784, i.e. > 40 sigma), samples are centre + N(0, sigma^2).
    Returns X [n, dim] fp32 row-major and y [n] int32, balanced classes.
    """
    rng = np.random.default_rng(seed)
    centres = rng.random((classes, dim), dtype=np.float32)
    y = (np.arange(n) % classes).astype(np.int32)
    rng.shuffle(y)
    X = centres[y] + sigma * rng.standard_normal((n, dim), dtype=np.float32)
    return X.astype(np.float32), y


def quadratic(dim: int, seed: int = 11, cond: float = 10.0):
    """l(w) = 1/2 ||A (w - w*)||^2 with diagonal A, condition number <= cond
    (SPEC.md:632-640).  Returns (a_diag, w_star) as float64."""
    rng = np.random.default_rng(seed)
    a = np.sqrt(rng.uniform(1.0, cond, size=dim))
    a[0], a[-1] = 1.0, np.sqrt(cond)
    w_star = rng.uniform(-1.0, 1.0, size=dim)
    return a, w_star


def sample_indices(d: int, d_pad: int, n: int, shard_bounds: list[int],
                   n_random: int = 65_536, seed: int = 5) -> np.ndarray:
    """Sampled index set for full-size parity (SURVEY.md §8c "Scaling the
    oracle"): first/last 64, every shard boundary +-2 and seeded random
    indices.  Sorted, unique, in [0, d).  (The padding region [d, d_pad) is
    a layout detail of the CUDA path; tests check it is exactly zero.)"""
    rng = np.random.default_rng(seed)
    parts = [np.arange(min(64, d)), np.arange(max(0, d - 64), d),
             rng.integers(0, d, size=n_random)]
    for b in shard_bounds:
        parts.append(np.arange(max(0, b - 2), min(d_pad, b + 2)))
    idx = np.unique(np.concatenate(parts).astype(np.int64))
    return idx[(idx >= 0) & (idx < d)]
