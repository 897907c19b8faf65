"""The SMA oracle: a plain, slow, obviously correct CPU implementation of
Algorithm 1 of arXiv 1901.02244 in fp64.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_1901_02244_b200``) and
neither imports the other; the only common dependency is ``sma_inputs`` (the
seeded input generator, which holds none of the method's arithmetic).

``liboracle_sma.so`` is built from ``oracle_sma.c`` with gcc (``build()``);
``exact.py`` is the exact-rational brute force used on tiny cases.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_sma.c")
_LIB = os.path.join(_HERE, "liboracle_sma.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, -O2, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fPIC",
                               "-shared", _SRC, "-o", _LIB, "-lm"])
    return _LIB


_LIB_OMP = os.path.join(_HERE, "liboracle_sma_omp.so")
_lib_omp = None


def build_omp(force: bool = False) -> str:
    """The same source with -fopenmp: adds orc_sma_run_synth_omp (bench timing only)."""
    if force or not os.path.exists(_LIB_OMP) or os.path.getmtime(_LIB_OMP) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fPIC", "-fopenmp",
                               "-shared", _SRC, "-o", _LIB_OMP, "-lm"])
    return _LIB_OMP


def run_synth_omp(d, k, alpha, gamma, mu, R, seed_w, seed_g, idx):
    """run_synth (z, z_prev only) with the index set split over OpenMP threads;
    bitwise equal to run_synth (separable per index).  Returns (z, z_prev, threads)."""
    global _lib_omp
    if _lib_omp is None:
        build_omp()
        L = C.CDLL(_LIB_OMP)
        i32, i64, u64, f64, P = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
        L.orc_sma_run_synth_omp.argtypes = [i64, i32, f64, f64, f64, i64, u64, u64, i64, P, P, P]
        L.orc_sma_run_synth_omp.restype = C.c_int
        _lib_omp = L
    idx = _i64(idx)
    z, zp = np.empty(idx.size), np.empty(idx.size)
    nt = _lib_omp.orc_sma_run_synth_omp(d, k, alpha, gamma, mu, R, seed_w, seed_g, idx.size,
                                        _p(idx), _p(z), _p(zp))
    if nt < 0:
        raise MemoryError("oracle allocation failed")
    return z, zp, nt


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
        P = C.c_void_p
        L.orc_splitmix64.argtypes, L.orc_splitmix64.restype = [u64], u64
        L.orc_uniform24.argtypes, L.orc_uniform24.restype = [u64, u64], f64
        L.orc_w0.argtypes, L.orc_w0.restype = [i64, P, u64, P], None
        L.orc_synth_grad.argtypes = [i64, i32, i64, i32, u64, i64, P, P]
        L.orc_synth_grad.restype = None
        L.orc_replica_location.argtypes = [i32, i32, i32, P, P]
        L.orc_replica_location.restype = C.c_int
        L.orc_d_pad.argtypes, L.orc_d_pad.restype = [i64, i32], i64
        L.orc_shard_range.argtypes, L.orc_shard_range.restype = [i64, i32, i32, P, P], None
        L.orc_epoch_permutation.argtypes = [i64, u64, i64, P]
        L.orc_epoch_permutation.restype = None
        L.orc_batch_indices.argtypes = [i64, i32, i32, u64, i64, i32, P]
        L.orc_batch_indices.restype = C.c_int
        L.orc_sma_round.argtypes = [i64, i32, f64, f64, f64, P, P, P, P, P]
        L.orc_sma_round.restype = None
        L.orc_sma_run_synth.argtypes = [i64, i32, f64, f64, f64, i64, u64, u64, i64, P, P, P, P]
        L.orc_sma_run_synth.restype = C.c_int
        L.orc_softmax_loss_grad.argtypes = [i32, i32, i32, P, P, P, P, P]
        L.orc_softmax_loss_grad.restype = f64
        L.orc_sma_run_softmax.argtypes = [i32, i32, i32, P, P, i64, u64, i32, f64, f64, f64,
                                          i64, P, P, P, P]
        L.orc_sma_run_softmax.restype = C.c_int
        L.orc_local_round.argtypes, L.orc_local_round.restype = [i64, i32, f64, P, P], None
        L.orc_autotune_step.argtypes = [i32, f64, P, P, P]
        L.orc_autotune_step.restype = None
        L.orc_resize_replicas.argtypes = [i64, i32, i32, i32, P, P, P]
        L.orc_resize_replicas.restype = None
        L.orc_mlp_loss_grad.argtypes = [i32, i32, i32, i32, P, P, P, P, P, P]
        L.orc_mlp_loss_grad.restype = f64
        L.orc_hier_round.argtypes = [i64, i32, i32, f64, f64, f64, f64, P, P, P, P, P, P]
        L.orc_hier_round.restype = None
        L.orc_hier_run_synth.argtypes = [i64, i32, i32, f64, f64, f64, f64, i64, u64, u64, i64,
                                         P, P, P, P, P]
        L.orc_hier_run_synth.restype = C.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def as_param(x) -> float:
    """R6: hyper-parameters are fp32 values promoted exactly to fp64."""
    return float(np.float32(x))


# ---------------------------------------------------------------- generator
def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(C.c_uint64(x & (2**64 - 1))))


def uniform24(seed: int, ctr: int) -> float:
    return float(lib().orc_uniform24(seed, ctr))


def w0(d: int, seed: int, idx=None) -> np.ndarray:
    idx = _i64(np.arange(d) if idx is None else idx)
    out = np.empty(idx.size, np.float64)
    lib().orc_w0(idx.size, _p(idx), seed, _p(out))
    return out


def synth_grad(d: int, k: int, rnd: int, j: int, seed: int, idx=None) -> np.ndarray:
    idx = _i64(np.arange(d) if idx is None else idx)
    out = np.empty(idx.size, np.float64)
    lib().orc_synth_grad(d, k, rnd, j, seed, idx.size, _p(idx), _p(out))
    return out


# -------------------------------------------------------------- bookkeeping
def replica_location(k: int, n: int, j: int) -> tuple[int, int]:
    r, s = C.c_int32(), C.c_int32()
    if lib().orc_replica_location(k, n, j, C.byref(r), C.byref(s)) != 0:
        raise ValueError("replica index out of range")
    return r.value, s.value


def d_pad(d: int, n: int) -> int:
    return int(lib().orc_d_pad(d, n))


def shard_range(d: int, n: int, g: int) -> tuple[int, int]:
    off, ln = C.c_int64(), C.c_int64()
    lib().orc_shard_range(d, n, g, C.byref(off), C.byref(ln))
    return off.value, ln.value


def epoch_permutation(N: int, seed: int, epoch: int) -> np.ndarray:
    out = np.empty(N, np.int64)
    lib().orc_epoch_permutation(N, seed, epoch, _p(out))
    return out


def batch_indices(N: int, k: int, b: int, seed: int, rnd: int, j: int) -> np.ndarray:
    out = np.empty(b, np.int64)
    if lib().orc_batch_indices(N, k, b, seed, rnd, j, _p(out)) != 0:
        raise ValueError("invalid batch-index request")
    return out


# ---------------------------------------------------------------- Alg. 1
class State:
    """fp64 state of Alg. 1: replicas W [k][m], z [m], z_prev [m]."""

    def __init__(self, W, z, z_prev):
        self.W = _f64(W).copy()
        self.z = _f64(z).copy()
        self.z_prev = _f64(z_prev).copy()

    @classmethod
    def init(cls, w0_vec, k: int, w_init=None):
        """Alg. 1 lines 1-2 with R2 (z_prev = w0) and R3 (w_j = w0)."""
        w0_vec = _f64(w0_vec)
        W = np.tile(w0_vec, (k, 1)) if w_init is None else _f64(w_init)
        return cls(W, w0_vec, w0_vec)

    def local_round(self, G, gamma):
        """Local-only iteration (sync period tau > 1, R17): w_j -= gamma G_j."""
        k, m = self.W.shape
        G = _f64(G).reshape(k, m)
        lib().orc_local_round(m, k, gamma, _p(self.W), _p(G))
        return self

    def resize(self, n: int, l_new: int):
        """Uniform per-GPU learner count l -> l_new (NEXT-4); new replicas := z."""
        k, m = self.W.shape
        assert k % n == 0
        Wn = np.empty((n * l_new, m))
        lib().orc_resize_replicas(m, n, k // n, l_new, _p(self.W), _p(self.z), _p(Wn))
        self.W = Wn
        return self

    def round(self, G, alpha, gamma, mu):
        """One iteration (Alg. 1 lines 4-14) with raw gradients G [k][m]."""
        k, m = self.W.shape
        G = _f64(G).reshape(k, m)
        cs = np.empty(m, np.float64)
        lib().orc_sma_round(m, k, alpha, gamma, mu, _p(self.W), _p(self.z), _p(self.z_prev),
                            _p(G), _p(cs))
        return self


def run_synth(d, k, alpha, gamma, mu, R, seed_w, seed_g, idx=None, want_W=True):
    """R rounds on the synthetic inputs at parameter indices idx (default all).
    Returns (z, z_prev, W or None) as fp64 arrays over idx."""
    idx = _i64(np.arange(d) if idx is None else idx)
    m = idx.size
    z, zp = np.empty(m), np.empty(m)
    W = np.empty((k, m)) if want_W else None
    rc = lib().orc_sma_run_synth(d, k, alpha, gamma, mu, R, seed_w, seed_g, m, _p(idx),
                                 _p(z), _p(zp), _p(W) if want_W else None)
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return z, zp, W


def softmax_loss_grad(X, y, rows, params, in_dim=784, classes=10, want_grad=True):
    X = np.ascontiguousarray(X, np.float32)
    y = np.ascontiguousarray(y, np.int32)
    rows = _i64(rows)
    params = _f64(params)
    g = np.empty_like(params) if want_grad else None
    loss = lib().orc_softmax_loss_grad(in_dim, classes, rows.size, _p(X), _p(y), _p(rows),
                                       _p(params), _p(g) if want_grad else None)
    return float(loss), g


def run_softmax(X, y, b, batch_seed, k, alpha, gamma, mu, R, w0_vec, in_dim=784, classes=10):
    """R rounds of Alg. 1 with the softmax learner in the loop (config C1)."""
    X = np.ascontiguousarray(X, np.float32)
    y = np.ascontiguousarray(y, np.int32)
    w0_vec = _f64(w0_vec)
    d = w0_vec.size
    z, zp, W = np.empty(d), np.empty(d), np.empty((k, d))
    rc = lib().orc_sma_run_softmax(in_dim, classes, b, _p(X), _p(y), X.shape[0], batch_seed, k,
                                   alpha, gamma, mu, R, _p(w0_vec), _p(z), _p(zp), _p(W))
    if rc != 0:
        raise ValueError("oracle softmax run failed")
    return z, zp, W


def autotune_step(tau: float, t, l, t_prev):
    """Alg. 2 lines 4-9 over all GPUs; returns new (l, t_prev)."""
    t = _f64(t)
    l = np.ascontiguousarray(l, dtype=np.int32).copy()
    tp = _f64(t_prev).copy()
    lib().orc_autotune_step(t.size, tau, _p(t), _p(l), _p(tp))
    return l, tp


def mlp_loss_grad(X, y, rows, params, in_dim=784, hidden=256, classes=10, want_grad=True):
    """MLP learner (kind 1): (loss, grad or None, min |pre-activation|)."""
    X = np.ascontiguousarray(X, np.float32)
    y = np.ascontiguousarray(y, np.int32)
    rows = _i64(rows)
    params = _f64(params)
    g = np.empty_like(params) if want_grad else None
    mn = C.c_double()
    loss = lib().orc_mlp_loss_grad(in_dim, hidden, classes, rows.size, _p(X), _p(y), _p(rows),
                                   _p(params), _p(g) if want_grad else None, C.byref(mn))
    return float(loss), g, mn.value


def mlp_dims(in_dim=784, hidden=256, classes=10) -> int:
    return hidden * in_dim + hidden + classes * hidden + classes


# ------------------------------------------- NEXT-3: per-GPU reference models
class HierState:
    """fp64 state of the two-level rule of Section 3.3 (R20): replicas W [k][m],
    reference models U [n][m] (row 0 mirrors z: GPU 0's reference model is the
    central average model), z, z_prev."""

    def __init__(self, W, U, z, z_prev):
        self.W = _f64(W).copy()
        self.U = _f64(U).copy()
        self.z = _f64(z).copy()
        self.z_prev = _f64(z_prev).copy()
        self.U[0] = self.z

    @classmethod
    def init(cls, w0_vec, k: int, n: int, w_init=None, u_init=None):
        w0_vec = _f64(w0_vec)
        W = np.tile(w0_vec, (k, 1)) if w_init is None else _f64(w_init)
        U = np.tile(w0_vec, (n, 1)) if u_init is None else _f64(u_init)
        return cls(W, U, w0_vec, w0_vec)

    def round(self, G, alpha_l, alpha_g, gamma, mu):
        k, m = self.W.shape
        n = self.U.shape[0]
        G = _f64(G).reshape(k, m)
        part = np.empty((n, m))
        lib().orc_hier_round(m, n, k, alpha_l, alpha_g, gamma, mu, _p(self.W), _p(self.U),
                             _p(self.z), _p(self.z_prev), _p(G), _p(part))
        self.U[0] = self.z
        return self


def hier_run_synth(d, n, k, alpha_l, alpha_g, gamma, mu, R, seed_w, seed_g, idx=None):
    """R rounds of the two-level rule (R20) on the synthetic inputs at indices
    idx.  Returns (z, z_prev, W [k][m], U [n][m]; U[0] = z)."""
    idx = _i64(np.arange(d) if idx is None else idx)
    m = idx.size
    z, zp, W, U = np.empty(m), np.empty(m), np.empty((k, m)), np.empty((n, m))
    rc = lib().orc_hier_run_synth(d, n, k, alpha_l, alpha_g, gamma, mu, R, seed_w, seed_g, m,
                                  _p(idx), _p(z), _p(zp), _p(W), _p(U))
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return z, zp, W, U
