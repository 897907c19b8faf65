"""World-size-2 CPU test of the multi-GPU decomposition (gloo backend).

Each rank takes its replicas and its shard of z from libsma's host
bookkeeping (sma_plan_*), advances its replicas, forms the per-GPU partial,
and runs the same collective sequence libsma issues over NCCL:
reduce-scatter(partial) -> shard update -> all-gather(z).  Both Mode A (paper
order) and Mode B (lookahead, double-buffered Q) are checked against the flat
fp64 oracle, and all ranks must hold bitwise-identical z.  The per-rank
arithmetic here is fp64 numpy (this exercises the decomposition and the
host logic; the kernels themselves are checked on the GPU).
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, d, k, R, out_dir):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import sma_inputs
    from paper_1901_02244_b200 import sma

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    alpha, gamma, mu = float(np.float32(1 / k)), float(np.float32(0.1)), float(np.float32(0.9))
    dp = sma.sma_plan_d_pad(d, world)
    j0, r = sma.sma_plan_local_replicas(k, world, rank)
    off, ln = sma.sma_plan_shard_range(d, world, rank)
    w0 = np.zeros(dp)
    w0[:d] = sma_inputs.w0(d)
    z, zp = w0.copy(), w0.copy()
    W = np.tile(w0, (r, 1))
    Q = [np.zeros(dp), np.zeros(dp)]
    qi = 0
    if mode == "B":  # prologue: Q^0 = sum_j (w_j^0 - z^{-1})
        Q[qi] = (W - zp).sum(0)
    for i in range(R):
        G = np.zeros((r, dp))
        for s in range(r):
            G[s, :d] = sma_inputs.grad(i, j0 + s, k, d)
        if mode == "A":
            C = alpha * (W - z)
            W = W - gamma * G - C
            P = C.sum(0)
            S = torch.empty(ln, dtype=torch.float64)
            dist.reduce_scatter_tensor(S, torch.from_numpy(P))
            zn_shard = z[off:off + ln] + S.numpy() + mu * (z[off:off + ln] - zp[off:off + ln])
        else:
            S = torch.empty(ln, dtype=torch.float64)
            dist.reduce_scatter_tensor(S, torch.from_numpy(Q[qi]))
            coef = mu - alpha * k
            zn_shard = (z[off:off + ln] + alpha * S.numpy()
                        + coef * (z[off:off + ln] - zp[off:off + ln]))
            Wn = W - gamma * G - alpha * (W - z)
            Q[1 - qi] = (Wn - z).sum(0)
            W = Wn
            qi = 1 - qi
        full = torch.empty(dp, dtype=torch.float64)
        dist.all_gather_into_tensor(full, torch.from_numpy(np.ascontiguousarray(zn_shard)))
        zp, z = z, full.numpy().copy()
    np.save(os.path.join(out_dir, f"z{rank}.npy"), z)
    np.save(os.path.join(out_dir, f"W{rank}.npy"), W)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["A", "B"])
@pytest.mark.parametrize("d,k", [(1001, 4), (777, 3)])
def test_two_rank_decomposition_matches_oracle(orc, tmp_path, mode, d, k):
    import torch.multiprocessing as mp

    from paper_1901_02244_b200 import _build
    _build.build()
    world, R = 2, 12
    mp.spawn(_worker, args=(world, _free_port(), mode, d, k, R, str(tmp_path)), nprocs=world)
    import sma_inputs
    from paper_1901_02244_b200 import sma
    z_ref, _, W_ref = orc.run_synth(d, k, float(np.float32(1 / k)), float(np.float32(0.1)),
                                    float(np.float32(0.9)), R, sma_inputs.SEED_W,
                                    sma_inputs.SEED_G)
    zs = [np.load(tmp_path / f"z{g}.npy") for g in range(world)]
    assert np.array_equal(zs[0], zs[1])                       # every rank holds the same z
    assert np.all(zs[0][d:] == 0)                            # padding stays exactly 0
    np.testing.assert_allclose(zs[0][:d], z_ref, rtol=0, atol=1e-12)
    for g in range(world):
        j0, r = sma.sma_plan_local_replicas(k, world, g)
        Wg = np.load(tmp_path / f"W{g}.npy")
        np.testing.assert_allclose(Wg[:, :d], W_ref[j0:j0 + r], rtol=0, atol=1e-12)


def _hier_worker(rank, world, port, mode, d, k, R, al, ag, out_dir):
    """The two-level rule of Section 3.3 (R20) decomposed as libsma issues it:
    rank 0's reference model is z, ranks >= 1 keep u_g; the per-GPU partial is
    D_0 (rank 0) or c_g = alpha_g (u_g - z) (ranks >= 1), then the same
    reduce-scatter -> shard update -> all-gather as flat Alg. 1.  Mode B emits
    the pre-scaled lookahead partials alpha_l sum_j (w_j' - z) / alpha_g (u_g' - z)
    and updates z' = z + S + (mu - alpha_l r_0 - alpha_g (n-1)) (z - z_prev)."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import sma_inputs
    from paper_1901_02244_b200 import sma

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gamma, mu = float(np.float32(0.1)), float(np.float32(0.9))
    dp = sma.sma_plan_d_pad(d, world)
    j0, r = sma.sma_plan_local_replicas(k, world, rank)
    _, r0 = sma.sma_plan_local_replicas(k, world, 0)
    off, ln = sma.sma_plan_shard_range(d, world, rank)
    w0 = np.zeros(dp)
    w0[:d] = sma_inputs.w0(d)
    z, zp = w0.copy(), w0.copy()
    W = np.tile(w0, (r, 1))
    U = w0.copy() if rank > 0 else None
    E = [np.zeros(dp), np.zeros(dp)]
    qi = 0
    if mode == "B":  # prologue
        E[qi] = al * (W - zp).sum(0) if rank == 0 else ag * (U - zp)
    for i in range(R):
        G = np.zeros((r, dp))
        for s in range(r):
            G[s, :d] = sma_inputs.grad(i, j0 + s, k, d)
        ref = z if rank == 0 else U
        Dj = al * (W - ref)
        Wn = W - gamma * G - Dj
        if rank > 0:
            c = ag * (U - z)
            Un = U + Dj.sum(0) - c
        S = torch.empty(ln, dtype=torch.float64)
        if mode == "A":
            P = Dj.sum(0) if rank == 0 else c
            dist.reduce_scatter_tensor(S, torch.from_numpy(np.ascontiguousarray(P)))
            zn_shard = z[off:off + ln] + S.numpy() + mu * (z[off:off + ln] - zp[off:off + ln])
        else:
            dist.reduce_scatter_tensor(S, torch.from_numpy(E[qi]))
            coef = mu - al * r0 - ag * (world - 1)
            zn_shard = z[off:off + ln] + S.numpy() + coef * (z[off:off + ln] - zp[off:off + ln])
            E[1 - qi] = al * (Wn - z).sum(0) if rank == 0 else ag * (Un - z)
            qi = 1 - qi
        W = Wn
        if rank > 0:
            U = Un
        full = torch.empty(dp, dtype=torch.float64)
        dist.all_gather_into_tensor(full, torch.from_numpy(np.ascontiguousarray(zn_shard)))
        zp, z = z, full.numpy().copy()
    np.save(os.path.join(out_dir, f"z{rank}.npy"), z)
    np.save(os.path.join(out_dir, f"W{rank}.npy"), W)
    np.save(os.path.join(out_dir, f"U{rank}.npy"), z if rank == 0 else U)
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["A", "B"])
@pytest.mark.parametrize("d,k", [(1001, 4), (777, 5)])
def test_two_rank_hierarchical_decomposition_matches_oracle(orc, tmp_path, mode, d, k):
    import torch.multiprocessing as mp

    from paper_1901_02244_b200 import _build
    _build.build()
    world, R = 2, 12
    al, ag = float(np.float32(0.25)), float(np.float32(0.5))
    mp.spawn(_hier_worker, args=(world, _free_port(), mode, d, k, R, al, ag, str(tmp_path)),
             nprocs=world)
    import sma_inputs
    from paper_1901_02244_b200 import sma
    z_ref, _, W_ref, U_ref = orc.hier_run_synth(d, world, k, al, ag, float(np.float32(0.1)),
                                                float(np.float32(0.9)), R, sma_inputs.SEED_W,
                                                sma_inputs.SEED_G)
    zs = [np.load(tmp_path / f"z{g}.npy") for g in range(world)]
    assert np.array_equal(zs[0], zs[1])
    assert np.all(zs[0][d:] == 0)
    np.testing.assert_allclose(zs[0][:d], z_ref, rtol=0, atol=1e-12)
    for g in range(world):
        j0, r = sma.sma_plan_local_replicas(k, world, g)
        np.testing.assert_allclose(np.load(tmp_path / f"W{g}.npy")[:, :d], W_ref[j0:j0 + r],
                                   rtol=0, atol=1e-12)
        np.testing.assert_allclose(np.load(tmp_path / f"U{g}.npy")[:d], U_ref[g], rtol=0,
                                   atol=1e-12)
