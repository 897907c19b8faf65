"""Thin ctypes binding of libsma (include/sma.h).  Argument marshalling only:
every step of the SMA round runs in libsma's CUDA kernels (and NCCL).  There
is no CPU fallback: if libsma.so is missing or a call fails, this raises.

The module-level functions carry the C names (``sma_create``, ``sma_step``,
...) and take plain integers for pointers/streams; :class:`Sma` is a small
convenience wrapper that accepts torch tensors / numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsma.so")

FLAG_OVERLAP = 1
FLAG_MATERIALIZE_C = 2
FLAG_CHECK_FINITE = 4
FLAG_CUDA_GRAPH = 8
FLAG_FORCE_COLLECTIVE = 16
FLAG_TIMING = 32
FLAG_KERNEL_TMA = 64
FLAG_KERNEL_LDG = 128
FLAG_NVLS_ZSYNC = 256
FLAG_P2P_ZSYNC = 512
FLAG_HIERARCHICAL = 1024
FLAG_P2P_PUSH = 2048
P2P_HANDLE_BYTES = 64
MAX_LOCAL_REPLICAS = 64
NCCL_ID_BYTES = 128

STATUS = {0: "SMA_OK", 1: "SMA_ERR_INVALID_ARG", 2: "SMA_ERR_NOT_LOCAL",
          3: "SMA_ERR_GRADS_MISSING", 4: "SMA_ERR_NONFINITE", 5: "SMA_ERR_CUDA",
          6: "SMA_ERR_NCCL", 7: "SMA_ERR_OOM", 8: "SMA_ERR_STATE"}

# Every symbol include/sma.h declares (tests check the library exports them).
EXPORTS = ["sma_create", "sma_destroy", "sma_set_learner_grads", "sma_set_learner_grads_host",
           "sma_synth_grads", "sma_step", "sma_get_central", "sma_get_central_prev",
           "sma_get_replica", "sma_set_replica", "sma_set_central", "sma_replica_device_ptr",
           "sma_central_device_ptr", "sma_restart", "sma_set_hparams", "sma_check_finite",
           "sma_learner_attach", "sma_learner_grads", "sma_plan_d_pad",
           "sma_plan_replica_location", "sma_plan_local_replicas", "sma_plan_shard_range",
           "sma_plan_batch_indices", "sma_nccl_unique_id", "sma_kernel_time",
           "sma_launch_count", "sma_info", "sma_last_error", "sma_abi_version",
           "sma_step_local", "sma_autotune_step", "sma_set_local_replicas", "sma_learner_step",
           "sma_p2p_handle", "sma_p2p_connect", "sma_set_alpha_global", "sma_get_reference",
           "sma_set_reference", "sma_set_timing", "sma_stage_grads_host",
           "sma_get_central_async", "sma_synchronize", "sma_learner_steps"]


class SmaError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")


class sma_config(C.Structure):
    _fields_ = [("d", C.c_int64), ("k", C.c_int32), ("alpha", C.c_float), ("gamma", C.c_float),
                ("mu", C.c_float), ("rank", C.c_int32), ("world", C.c_int32),
                ("device", C.c_int32), ("nccl_id", C.c_void_p), ("flags", C.c_uint32)]


_lib = None


def load():
    """Load libsma.so (raise if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                          "(python -m paper_1901_02244_b200._build)")
    L = C.CDLL(LIB_PATH)
    i32, i64, u64, P, st = C.c_int32, C.c_int64, C.c_uint64, C.c_void_p, C.c_int
    sig = {
        "sma_create": ([C.POINTER(sma_config), P, C.POINTER(P)], st),
        "sma_destroy": ([P], None),
        "sma_set_learner_grads": ([P, i32, P], st),
        "sma_set_learner_grads_host": ([P, i32, P, P], st),
        "sma_synth_grads": ([P, i64, u64, P], st),
        "sma_step": ([P, P], st),
        "sma_get_central": ([P, P, C.c_int], st),
        "sma_get_central_prev": ([P, P, C.c_int], st),
        "sma_get_replica": ([P, i32, P, C.c_int], st),
        "sma_set_replica": ([P, i32, P, C.c_int], st),
        "sma_set_central": ([P, P, P, C.c_int], st),
        "sma_replica_device_ptr": ([P, i32, C.POINTER(P)], st),
        "sma_central_device_ptr": ([P, C.POINTER(P)], st),
        "sma_restart": ([P, P], st),
        "sma_set_hparams": ([P, C.c_float, C.c_float, C.c_float], st),
        "sma_check_finite": ([P, C.POINTER(C.c_int)], st),
        "sma_learner_attach": ([P, i32, i32, i32, i32, i32, P, P, i64, u64], st),
        "sma_learner_grads": ([P, i64, P], st),
        "sma_plan_d_pad": ([i64, i32], i64),
        "sma_plan_replica_location": ([i32, i32, i32, C.POINTER(i32), C.POINTER(i32)], st),
        "sma_plan_local_replicas": ([i32, i32, i32, C.POINTER(i32), C.POINTER(i32)], st),
        "sma_plan_shard_range": ([i64, i32, i32, C.POINTER(i64), C.POINTER(i64)], st),
        "sma_plan_batch_indices": ([i64, i32, i32, u64, i64, i32, P], st),
        "sma_nccl_unique_id": ([P], st),
        "sma_kernel_time": ([P, i32, C.POINTER(C.c_double), C.POINTER(i64), C.c_int], st),
        "sma_launch_count": ([P], i64),
        "sma_info": ([P, C.POINTER(i64), C.POINTER(i32), C.POINTER(i32), C.POINTER(i64),
                      C.POINTER(i64)], st),
        "sma_last_error": ([], C.c_char_p),
        "sma_abi_version": ([], C.c_int),
        "sma_step_local": ([P, P], st),
        "sma_autotune_step": ([i32, C.c_double, P, P, P], st),
        "sma_set_local_replicas": ([P, i32, P], st),
        "sma_learner_step": ([P, i64, P], st),
        "sma_learner_steps": ([P, i64, i32, P], st),
        "sma_p2p_handle": ([P, P], st),
        "sma_p2p_connect": ([P, P], st),
        "sma_set_alpha_global": ([P, C.c_float], st),
        "sma_get_reference": ([P, P, C.c_int], st),
        "sma_set_reference": ([P, P, C.c_int], st),
        "sma_set_timing": ([P, C.c_int], st),
        "sma_stage_grads_host": ([P, i32, P], st),
        "sma_get_central_async": ([P, P], st),
        "sma_synchronize": ([P], st),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes, fn.restype = args, res
    _lib = L
    return L


def _check(status: int, where: str):
    if status != 0:
        raise SmaError(status, where, load().sma_last_error().decode(errors="replace"))


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)}")


def _stream(s) -> int:
    if s is None:
        return 0
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ------------------------------------------------------- C-named functions
def sma_create(cfg: sma_config, w0_host) -> int:
    h = C.c_void_p()
    _check(load().sma_create(C.byref(cfg), _ptr(w0_host), C.byref(h)), "sma_create")
    return h.value


def sma_destroy(h: int) -> None:
    load().sma_destroy(h)


def sma_set_learner_grads(h: int, j: int, g_dev) -> None:
    _check(load().sma_set_learner_grads(h, j, _ptr(g_dev)), "sma_set_learner_grads")


def sma_set_learner_grads_host(h: int, j: int, g_host, stream=None) -> None:
    _check(load().sma_set_learner_grads_host(h, j, _ptr(g_host), _stream(stream)),
           "sma_set_learner_grads_host")


def sma_stage_grads_host(h: int, gset: int, g_hosts) -> None:
    """g_hosts: one host buffer (pinned tensor / numpy array / address) per local learner."""
    arr = (C.c_void_p * max(1, len(g_hosts)))(*[_ptr(g) for g in g_hosts])
    _check(load().sma_stage_grads_host(h, gset, arr), "sma_stage_grads_host")


def sma_get_central_async(h: int, z_host) -> None:
    _check(load().sma_get_central_async(h, _ptr(z_host)), "sma_get_central_async")


def sma_synchronize(h: int) -> None:
    _check(load().sma_synchronize(h), "sma_synchronize")


def sma_synth_grads(h: int, rnd: int, seed: int, stream=None) -> None:
    _check(load().sma_synth_grads(h, rnd, seed, _stream(stream)), "sma_synth_grads")


def sma_step(h: int, stream=None) -> None:
    _check(load().sma_step(h, _stream(stream)), "sma_step")


def sma_step_local(h: int, stream=None) -> None:
    _check(load().sma_step_local(h, _stream(stream)), "sma_step_local")


def sma_autotune_step(tau: float, t, l, t_prev):
    """Alg. 2 loop body over all GPUs; returns the new (l, t_prev) arrays."""
    t = np.ascontiguousarray(t, np.float64)
    l = np.ascontiguousarray(l, np.int32).copy()
    tp = np.ascontiguousarray(t_prev, np.float64).copy()
    _check(load().sma_autotune_step(t.size, tau, t.ctypes.data, l.ctypes.data, tp.ctypes.data),
           "sma_autotune_step")
    return l, tp


def sma_set_local_replicas(h: int, l_new: int, stream=None) -> None:
    _check(load().sma_set_local_replicas(h, l_new, _stream(stream)), "sma_set_local_replicas")


def sma_get_central(h: int, out, out_is_device: bool) -> None:
    _check(load().sma_get_central(h, _ptr(out), int(out_is_device)), "sma_get_central")


def sma_get_central_prev(h: int, out, out_is_device: bool) -> None:
    _check(load().sma_get_central_prev(h, _ptr(out), int(out_is_device)), "sma_get_central_prev")


def sma_get_replica(h: int, j: int, out, out_is_device: bool) -> None:
    _check(load().sma_get_replica(h, j, _ptr(out), int(out_is_device)), "sma_get_replica")


def sma_set_replica(h: int, j: int, w, in_is_device: bool) -> None:
    _check(load().sma_set_replica(h, j, _ptr(w), int(in_is_device)), "sma_set_replica")


def sma_set_central(h: int, z, z_prev, in_is_device: bool) -> None:
    _check(load().sma_set_central(h, _ptr(z), _ptr(z_prev), int(in_is_device)), "sma_set_central")


def sma_replica_device_ptr(h: int, j: int) -> int:
    p = C.c_void_p()
    _check(load().sma_replica_device_ptr(h, j, C.byref(p)), "sma_replica_device_ptr")
    return p.value


def sma_central_device_ptr(h: int) -> int:
    p = C.c_void_p()
    _check(load().sma_central_device_ptr(h, C.byref(p)), "sma_central_device_ptr")
    return p.value


def sma_restart(h: int, stream=None) -> None:
    _check(load().sma_restart(h, _stream(stream)), "sma_restart")


def sma_set_hparams(h: int, alpha: float, gamma: float, mu: float) -> None:
    _check(load().sma_set_hparams(h, alpha, gamma, mu), "sma_set_hparams")


def sma_set_alpha_global(h: int, alpha_g: float) -> None:
    _check(load().sma_set_alpha_global(h, alpha_g), "sma_set_alpha_global")


def sma_get_reference(h: int, out, out_is_device: bool) -> None:
    _check(load().sma_get_reference(h, _ptr(out), int(out_is_device)), "sma_get_reference")


def sma_set_reference(h: int, u, in_is_device: bool) -> None:
    _check(load().sma_set_reference(h, _ptr(u), int(in_is_device)), "sma_set_reference")


def sma_check_finite(h: int) -> bool:
    f = C.c_int()
    _check(load().sma_check_finite(h, C.byref(f)), "sma_check_finite")
    return bool(f.value)


def sma_learner_attach(h: int, kind: int, in_dim: int, hidden: int, classes: int, batch: int,
                       X_dev, y_dev, n_samples: int, batch_seed: int) -> None:
    _check(load().sma_learner_attach(h, kind, in_dim, hidden, classes, batch, _ptr(X_dev),
                                     _ptr(y_dev), n_samples, batch_seed), "sma_learner_attach")


def sma_learner_grads(h: int, rnd: int, stream=None) -> None:
    _check(load().sma_learner_grads(h, rnd, _stream(stream)), "sma_learner_grads")


def sma_learner_step(h: int, rnd: int, stream=None) -> None:
    _check(load().sma_learner_step(h, rnd, _stream(stream)), "sma_learner_step")


def sma_learner_steps(h: int, rnd0: int, count: int, stream=None) -> None:
    _check(load().sma_learner_steps(h, rnd0, count, _stream(stream)), "sma_learner_steps")


def sma_p2p_handle(h: int) -> bytes:
    buf = (C.c_char * P2P_HANDLE_BYTES)()
    _check(load().sma_p2p_handle(h, buf), "sma_p2p_handle")
    return bytes(buf)


def sma_p2p_connect(h: int, handles: list) -> None:
    blob = b"".join(bytes(x) for x in handles)
    buf = C.create_string_buffer(blob, len(blob))
    _check(load().sma_p2p_connect(h, buf), "sma_p2p_connect")


def sma_plan_d_pad(d: int, world: int) -> int:
    return int(load().sma_plan_d_pad(d, world))


def sma_plan_replica_location(k: int, world: int, j: int) -> tuple[int, int]:
    r, s = C.c_int32(), C.c_int32()
    _check(load().sma_plan_replica_location(k, world, j, C.byref(r), C.byref(s)),
           "sma_plan_replica_location")
    return r.value, s.value


def sma_plan_local_replicas(k: int, world: int, rank: int) -> tuple[int, int]:
    f, c = C.c_int32(), C.c_int32()
    _check(load().sma_plan_local_replicas(k, world, rank, C.byref(f), C.byref(c)),
           "sma_plan_local_replicas")
    return f.value, c.value


def sma_plan_shard_range(d: int, world: int, rank: int) -> tuple[int, int]:
    o, n = C.c_int64(), C.c_int64()
    _check(load().sma_plan_shard_range(d, world, rank, C.byref(o), C.byref(n)),
           "sma_plan_shard_range")
    return o.value, n.value


def sma_plan_batch_indices(n_samples: int, k: int, batch: int, seed: int, rnd: int,
                           j: int) -> np.ndarray:
    out = np.empty(batch, np.int64)
    _check(load().sma_plan_batch_indices(n_samples, k, batch, seed, rnd, j, out.ctypes.data),
           "sma_plan_batch_indices")
    return out


def sma_nccl_unique_id() -> bytes:
    buf = (C.c_char * NCCL_ID_BYTES)()
    _check(load().sma_nccl_unique_id(buf), "sma_nccl_unique_id")
    return bytes(buf)


PHASE_REPLICA, PHASE_REDUCE_SCATTER, PHASE_SHARD_UPDATE, PHASE_ALL_GATHER, PHASE_NVLS_ZSYNC = \
    0, 1, 2, 3, 4


def sma_kernel_time(h: int, phase: int = PHASE_REPLICA, reset: bool = False) -> tuple[float, int]:
    ms, n = C.c_double(), C.c_int64()
    _check(load().sma_kernel_time(h, phase, C.byref(ms), C.byref(n), int(reset)),
           "sma_kernel_time")
    return ms.value, n.value


def sma_set_timing(h: int, on: bool) -> None:
    _check(load().sma_set_timing(h, int(on)), "sma_set_timing")


def sma_launch_count(h: int) -> int:
    return int(load().sma_launch_count(h))


def sma_info(h: int) -> dict:
    dp, f, c, o, n = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
    _check(load().sma_info(h, C.byref(dp), C.byref(f), C.byref(c), C.byref(o), C.byref(n)),
           "sma_info")
    return dict(d_pad=dp.value, local_first=f.value, local_count=c.value,
                shard_offset=o.value, shard_length=n.value)


def sma_abi_version() -> int:
    return int(load().sma_abi_version())


# ---------------------------------------------------------- convenience
class Sma:
    """Owning wrapper of one sma_handle on one rank.

    d, k, alpha, gamma, mu: the paper's parameters.  w0: d floats
    (host array, torch CPU tensor or numpy).  rank/world/nccl_id for the
    multi-GPU path (nccl_id: bytes from sma_nccl_unique_id() on rank 0).
    """

    def __init__(self, d, k, alpha, gamma, mu, w0, *, rank=0, world=1, device=0,
                 nccl_id: bytes | None = None, flags=0):
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = C.create_string_buffer(bytes(nccl_id), NCCL_ID_BYTES)
        cfg = sma_config(d=d, k=k, alpha=alpha, gamma=gamma, mu=mu, rank=rank, world=world,
                         device=device,
                         nccl_id=C.cast(self._id_buf, C.c_void_p) if self._id_buf else None,
                         flags=flags)
        w0 = np.ascontiguousarray(np.asarray(w0, dtype=np.float32)) if not hasattr(w0, "data_ptr") \
            else w0.contiguous()
        self.d, self.k, self.world, self.rank, self.device = d, k, world, rank, device
        self._w0_keepalive = w0
        self.h = sma_create(cfg, w0)
        info = sma_info(self.h)
        self.d_pad = info["d_pad"]
        self.local_first, self.local_count = info["local_first"], info["local_count"]
        self.shard = (info["shard_offset"], info["shard_length"])

    def close(self):
        if getattr(self, "h", None):
            sma_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def local_replicas(self):
        return range(self.local_first, self.local_first + self.local_count)

    def set_grads(self, j, g_dev):
        sma_set_learner_grads(self.h, j, g_dev)

    def set_grads_host(self, j, g_host, stream=None):
        sma_set_learner_grads_host(self.h, j, g_host, stream)

    def synth_grads(self, rnd, seed, stream=None):
        sma_synth_grads(self.h, rnd, seed, stream)

    def step(self, stream=None):
        sma_step(self.h, stream)

    def step_local(self, stream=None):
        sma_step_local(self.h, stream)

    def set_local_replicas(self, l_new, stream=None):
        sma_set_local_replicas(self.h, l_new, stream)
        info = sma_info(self.h)
        self.local_first, self.local_count = info["local_first"], info["local_count"]
        self.k = self.local_count * self.world

    def central(self) -> np.ndarray:
        out = np.empty(self.d, np.float32)
        sma_get_central(self.h, out, False)
        return out

    def central_prev(self) -> np.ndarray:
        out = np.empty(self.d, np.float32)
        sma_get_central_prev(self.h, out, False)
        return out

    def replica(self, j) -> np.ndarray:
        out = np.empty(self.d, np.float32)
        sma_get_replica(self.h, j, out, False)
        return out

    def set_replica(self, j, w):
        w = np.ascontiguousarray(w, np.float32)
        sma_set_replica(self.h, j, w, False)

    def set_central(self, z, z_prev):
        z = np.ascontiguousarray(z, np.float32)
        zp = np.ascontiguousarray(z_prev, np.float32)
        sma_set_central(self.h, z, zp, False)

    def restart(self, stream=None):
        sma_restart(self.h, stream)

    def set_hparams(self, alpha, gamma, mu):
        sma_set_hparams(self.h, alpha, gamma, mu)

    def set_alpha_global(self, alpha_g):
        sma_set_alpha_global(self.h, alpha_g)

    def reference(self) -> np.ndarray:
        out = np.empty(self.d, np.float32)
        sma_get_reference(self.h, out, False)
        return out

    def set_reference(self, u):
        u = np.ascontiguousarray(u, np.float32)
        sma_set_reference(self.h, u, False)

    def kernel_time(self, reset=False, phase=PHASE_REPLICA):
        return sma_kernel_time(self.h, phase, reset)

    def set_timing(self, on):
        sma_set_timing(self.h, on)

    def launch_count(self):
        return sma_launch_count(self.h)
