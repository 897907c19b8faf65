"""GPU parity of the collective-path replica kernels at the size where they run
the full-grid direct-load kernel (`replica_step_ldg<MODE, ...>`), i.e. the
per-GPU kernel `bench.py` times at N > 1 (VERDICT r01 "next" #1).

`launch_replica_step` (sma_kernels.cu) takes the small-round split kernel
below n4 = d_pad/4 < 37,888 float4 columns (or < 151,552 with r >= 8); at
d = 1,000,003 (n4 = 250,112) every r in {2, 4, 8} and every mode runs
`replica_step_ldg` over the whole vector, with its scalar tail chunk at d.

* One process (FORCE_COLLECTIVE, a 1-rank communicator or 1-rank P2P z-sync):
  kPartialA (Mode A), kPartialB (Mode B), the P2P pull / push epilogue, and
  the Section 3.3 rank-0 partial kHierB0 -- 100 rounds (Alg. 1)
  vs the fp64 oracle on >= 65k sampled indices, plus every shard/tile edge,
  padding [d, d_pad) checked exactly 0.
* Two processes on the one GPU over the P2P z-sync (r = 2 per rank, the
  per-GPU replica count of C4 at N = 8): Modes A / B, push, and the two-level
  rule, which runs kHierA / kHierB on rank 1 and kHierB0 on rank 0
  (R20), 100 rounds.
"""
import os

import numpy as np
import pytest

import sma_inputs

pytestmark = pytest.mark.gpu

TOL = 1e-5
D = 1_000_003
R = 100
F32 = lambda x: float(np.float32(x))  # noqa: E731

# flags: FORCE_COLLECTIVE 16, OVERLAP 1, CUDA_GRAPH 8, P2P_ZSYNC 512, P2P_PUSH 2048,
# HIERARCHICAL 1024
VARIANTS = {
    "collA": 16,                      # replica_step_ldg<kPartialA> + NCCL RS / zsync / AG
    "collB": 16 | 1,                  # replica_step_ldg<kPartialB>, z-sync on the 2nd stream
    "collB_graph": 16 | 1 | 8,
    "p2pA": 16 | 512,                 # kPartialA + fused P2P z-sync
    "p2pB": 16 | 1 | 512,
    "pushA": 16 | 512 | 2048,         # kPartialA with the push epilogue (store_partial)
    "pushB": 16 | 1 | 512 | 2048,
    "hierB": 16 | 1 | 1024,           # rank 0 of the two-level rule: kHierB0
    "hierB_push": 16 | 1 | 512 | 2048 | 1024,
}


def relerr(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref) / (1.0 + np.abs(ref))))


def _dev_read(ptr, n):
    import ctypes
    import torch
    torch.cuda.synchronize()
    rt = ctypes.CDLL("libcudart.so.12")
    out = np.empty(n, np.float32)
    assert rt.cudaMemcpy(ctypes.c_void_p(out.ctypes.data), ctypes.c_void_p(ptr),
                         ctypes.c_size_t(4 * n), ctypes.c_int(2)) == 0
    return out


def _sample(d_pad, world=1):
    """>= 65,536 random indices, the first/last 64, every shard boundary +- 2,
    and every 1024-column boundary of one CTA of the LDG kernel (256 threads
    x float4) in the first 64 CTAs."""
    bounds = [g * (d_pad // world) for g in range(world + 1)]
    base = sma_inputs.sample_indices(D, d_pad, world, bounds, n_random=70_000)
    cta = np.concatenate([np.arange(c * 1024 - 2, c * 1024 + 2) for c in range(1, 65)])
    idx = np.unique(np.concatenate([base, cta]))
    idx = idx[(idx >= 0) & (idx < D)]
    assert idx.size >= 65_536
    return idx


_ORACLE = {}


def _oracle(orc, k, idx):
    key = (k, idx.size)
    if key not in _ORACLE:
        a, g, m = F32(1 / k), F32(0.1), F32(0.9)
        _ORACLE[key] = orc.run_synth(D, k, a, g, m, R, sma_inputs.SEED_W, sma_inputs.SEED_G, idx)
    return _ORACLE[key]


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no fallback)"
    torch.cuda.set_device(0)
    from paper_1901_02244_b200 import sma
    sma.load()
    return sma


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("r", [2, 4, 8])
def test_ldg_collective_kernel_at_size(S, orc, variant, r):
    """100 rounds at d = 1,000,003 with r local replicas through the collective
    path: the replica kernel is replica_step_ldg<MODE> on a full grid."""
    import torch
    k = r
    a, g, m = F32(1 / k), F32(0.1), F32(0.9)
    h = S.Sma(D, k, a, g, m, sma_inputs.w0(D), flags=VARIANTS[variant])
    assert h.d_pad // 4 >= 151_552, "this size must take the full-grid LDG kernel"
    s = torch.cuda.Stream()
    for i in range(R):
        h.synth_grads(i, sma_inputs.SEED_G, s)
        h.step(s)
    idx = _sample(h.d_pad)
    zr, zpr, Wr = _oracle(orc, k, idx)
    ctx = dict(variant=variant, r=r)
    assert relerr(h.central()[idx], zr) <= TOL, ctx
    assert relerr(h.central_prev()[idx], zpr) <= TOL, ctx
    for j in range(k):
        assert relerr(h.replica(j)[idx], Wr[j]) <= TOL, (ctx, j)
    for j in range(k):   # padding [d, d_pad) stays exactly 0
        assert np.all(_dev_read(S.sma_replica_device_ptr(h.h, j), h.d_pad)[D:] == 0), (ctx, j)
    assert np.all(_dev_read(S.sma_central_device_ptr(h.h), h.d_pad)[D:] == 0), ctx
    h.close()


# ------------------------------------------------ two ranks (processes), one GPU
def _mp_worker(rank, world, port, flags, k, hier, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_1901_02244_b200 import sma
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = k // world
    a = F32(1 / (2 * r)) if hier else F32(1 / k)
    f = flags | sma.FLAG_P2P_ZSYNC | (sma.FLAG_HIERARCHICAL if hier else 0)
    h = sma.Sma(D, k, a, F32(0.1), F32(0.9), sma_inputs.w0(D), rank=rank, world=world,
                device=0, flags=f)
    handles = [None] * world
    dist.all_gather_object(handles, sma.sma_p2p_handle(h.h))
    sma.sma_p2p_connect(h.h, handles)
    dist.barrier()
    s = torch.cuda.Stream()
    for i in range(R):
        h.synth_grads(i, sma_inputs.SEED_G, s)
        h.step(s)
    s.synchronize()
    np.save(os.path.join(out, f"z{rank}.npy"), h.central())
    np.save(os.path.join(out, f"zp{rank}.npy"), h.central_prev())
    if hier:
        np.save(os.path.join(out, f"u{rank}.npy"), h.reference())
    for j in h.local_replicas():
        np.save(os.path.join(out, f"w{j}.npy"), h.replica(j))
        np.save(os.path.join(out, f"pad{j}.npy"),
                _dev_read(sma.sma_replica_device_ptr(h.h, j), h.d_pad)[D:])
    dist.barrier()
    h.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["A", "B", "pushB", "hierA", "hierB"])
def test_p2p_two_ranks_at_size(orc, tmp_path, mode):
    """world = 2, k = 4 (r = 2 per rank), d = 1,000,003, 100 rounds: every rank
    runs replica_step_ldg over the full vector (kPartialA/B; kHierA/kHierB on
    rank 1 and kHierB0 on rank 0 for the two-level rule) and the fused P2P
    z-sync on its half; z is bitwise equal on both ranks and matches the
    oracle (flat, or the two-level oracle of R20) on sampled indices."""
    import socket

    import torch.multiprocessing as mp
    world, k = 2, 4
    flags = {"A": 0, "B": 1, "pushB": 1 | 2048, "hierA": 0, "hierB": 1}[mode]
    hier = mode.startswith("hier")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    mp.spawn(_mp_worker, args=(world, port, flags, k, hier, str(tmp_path)), nprocs=world)
    from paper_1901_02244_b200 import sma
    d_pad = sma.sma_plan_d_pad(D, world)
    idx = _sample(d_pad, world)
    g, m = F32(0.1), F32(0.9)
    if hier:
        al, ag = F32(1 / 4), F32(1 / 2)
        zr, zpr, Wr, Ur = orc.hier_run_synth(D, world, k, al, ag, g, m, R, sma_inputs.SEED_W,
                                             sma_inputs.SEED_G, idx)
    else:
        zr, zpr, Wr = _oracle(orc, k, idx)
    zs = [np.load(tmp_path / f"z{q}.npy") for q in range(world)]
    assert np.array_equal(zs[0], zs[1])
    assert relerr(zs[0][idx], zr) <= TOL
    assert relerr(np.load(tmp_path / "zp0.npy")[idx], zpr) <= TOL
    for j in range(k):
        assert relerr(np.load(tmp_path / f"w{j}.npy")[idx], Wr[j]) <= TOL, j
        assert np.all(np.load(tmp_path / f"pad{j}.npy") == 0), j
    if hier:
        assert np.array_equal(np.load(tmp_path / "u0.npy"), zs[0])
        assert relerr(np.load(tmp_path / "u1.npy")[idx], Ur[1]) <= TOL
