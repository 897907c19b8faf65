"""Multi-rank SMA on ONE GPU: several processes, one rank each, all on cuda:0,
with the P2P z-sync (SMA_FLAG_P2P_ZSYNC: CUDA IPC mappings of every rank's
buffers, no NCCL).  This exercises the real multi-rank path -- replica block
split, shards, the fused reduce-scatter / shard update / all-gather kernel over
another process's memory, its cross-process barriers, Mode A and Mode B, CUDA
graphs -- against the flat fp64 oracle, and checks that every rank ends with a
bitwise-identical z.  (Kernels of different processes time-slice on the GPU, so
this is a correctness test, not a performance one.)"""
import os
import socket
import sys

import numpy as np
import pytest

from oracle import exact

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, flags, d, k, R, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import sma_inputs
    from paper_1901_02244_b200 import sma
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, g, m = (float(np.float32(x)) for x in (1 / k, 0.1, 0.9))
    h = sma.Sma(d, k, a, g, m, sma_inputs.w0(d), rank=rank, world=world, device=0,
                flags=flags | sma.FLAG_P2P_ZSYNC)
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
    for j in h.local_replicas():
        np.save(os.path.join(out, f"w{j}.npy"), h.replica(j))
    dist.barrier()          # nobody unmaps while a peer may still read its buffers
    h.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 4), (2, 3), (4, 8), (3, 7)])
@pytest.mark.parametrize("mode", ["A", "B", "B_graph"])
def test_p2p_ranks_on_one_gpu_match_oracle(orc, tmp_path, world, k, mode):
    import torch
    import torch.multiprocessing as mp

    import sma_inputs
    assert torch.cuda.is_available()
    flags = {"A": 0, "B": 1, "B_graph": 1 | 8}[mode]
    d, R = 100_003, 12
    mp.spawn(_worker, args=(world, _port(), flags, d, k, R, str(tmp_path)), nprocs=world)
    zr, zpr, Wr = orc.run_synth(d, k, float(np.float32(1 / k)), float(np.float32(0.1)),
                                float(np.float32(0.9)), R, sma_inputs.SEED_W, sma_inputs.SEED_G)
    zs = [np.load(tmp_path / f"z{g}.npy") for g in range(world)]
    for z in zs[1:]:
        assert np.array_equal(z, zs[0])                 # every rank holds the same z, bitwise
    rel = lambda x, y: np.max(np.abs(x - y) / (1 + np.abs(y)))  # noqa: E731
    assert rel(zs[0], zr) <= 1e-5
    assert rel(np.load(tmp_path / "zp0.npy"), zpr) <= 1e-5
    for j in range(k):
        assert rel(np.load(tmp_path / f"w{j}.npy"), Wr[j]) <= 1e-5


# --------------------------------------- Section 3.3 two-level rule (R20)
def _hier_worker(rank, world, port, flags, d, k, R, al, ag, dyadic, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import sma_inputs
    from paper_1901_02244_b200 import sma
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, m = (0.125, 0.5) if dyadic else (float(np.float32(0.1)), float(np.float32(0.9)))
    w0 = sma_inputs.dyadic(d, 300).astype(np.float32) if dyadic else sma_inputs.w0(d)
    h = sma.Sma(d, k, al, g, m, w0, rank=rank, world=world, device=0,
                flags=flags | sma.FLAG_P2P_ZSYNC | sma.FLAG_HIERARCHICAL)
    if ag is not None:
        h.set_alpha_global(ag)
    handles = [None] * world
    dist.all_gather_object(handles, sma.sma_p2p_handle(h.h))
    sma.sma_p2p_connect(h.h, handles)
    dist.barrier()
    s = torch.cuda.Stream()
    if dyadic:
        G = torch.tensor(sma_inputs.dyadic((R, k, d), 301), dtype=torch.float32, device="cuda")
    for i in range(R):
        if dyadic:
            for j in h.local_replicas():
                h.set_grads(j, G[i, j])
        else:
            h.synth_grads(i, sma_inputs.SEED_G, s)
        h.step(s)
    s.synchronize()
    np.save(os.path.join(out, f"z{rank}.npy"), h.central())
    np.save(os.path.join(out, f"zp{rank}.npy"), h.central_prev())
    np.save(os.path.join(out, f"u{rank}.npy"), h.reference())
    for j in h.local_replicas():
        np.save(os.path.join(out, f"w{j}.npy"), h.replica(j))
    dist.barrier()
    h.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k,ag", [(2, 4, None), (3, 7, 0.25), (4, 8, None)])
@pytest.mark.parametrize("mode", ["A", "B", "B_graph"])
def test_p2p_hierarchical_ranks_match_oracle(orc, tmp_path, world, k, ag, mode):
    """SMA_FLAG_HIERARCHICAL with 2-4 ranks (processes) on one GPU over the P2P
    z-sync: z, z_prev, every replica and every GPU's reference model u_g match
    the two-level fp64 oracle (R20) after 12 rounds; z is bitwise equal on
    every rank; rank 0's reference model is z."""
    import torch.multiprocessing as mp

    import sma_inputs
    flags = {"A": 0, "B": 1, "B_graph": 1 | 8}[mode]
    d, R = 100_003, 12
    al = float(np.float32(0.25))
    ag_eff = float(np.float32(ag if ag is not None else 1 / (2 * (world - 1))))
    mp.spawn(_hier_worker, args=(world, _port(), flags, d, k, R, al, ag, False, str(tmp_path)),
             nprocs=world)
    zr, zpr, Wr, Ur = orc.hier_run_synth(d, world, k, al, ag_eff, float(np.float32(0.1)),
                                         float(np.float32(0.9)), R, sma_inputs.SEED_W,
                                         sma_inputs.SEED_G)
    zs = [np.load(tmp_path / f"z{g}.npy") for g in range(world)]
    for z in zs[1:]:
        assert np.array_equal(z, zs[0])
    assert np.array_equal(np.load(tmp_path / "u0.npy"), zs[0])
    rel = lambda x, y: np.max(np.abs(x - y) / (1 + np.abs(y)))  # noqa: E731
    assert rel(zs[0], zr) <= 1e-5
    assert rel(np.load(tmp_path / "zp0.npy"), zpr) <= 1e-5
    for g in range(1, world):
        assert rel(np.load(tmp_path / f"u{g}.npy"), Ur[g]) <= 1e-5, g
    for j in range(k):
        assert rel(np.load(tmp_path / f"w{j}.npy"), Wr[j]) <= 1e-5, j
    # the two levels matter: the result is not flat Alg. 1
    zf, _, _ = orc.run_synth(d, k, al, float(np.float32(0.1)), float(np.float32(0.9)), R,
                             sma_inputs.SEED_W, sma_inputs.SEED_G)
    assert rel(zs[0], zf) > 1e-4


@pytest.mark.parametrize("world,k", [(2, 4), (3, 5)])
@pytest.mark.parametrize("mode", ["A", "B"])
def test_p2p_hierarchical_dyadic_bitwise(tmp_path, world, k, mode):
    """Dyadic inputs keep fp32 exact for the first rounds: the multi-rank GPU
    two-level rule equals the exact-rational brute force (oracle/exact.py)
    bit for bit -- replicas, reference models, z and z_prev."""
    import torch.multiprocessing as mp

    import sma_inputs
    d, R = 4, 6
    al, ag = 0.25, 0.5
    mp.spawn(_hier_worker, args=(world, _port(), {"A": 0, "B": 1}[mode], d, k, R, al, ag, True,
                                 str(tmp_path)), nprocs=world)
    w0 = sma_inputs.dyadic(d, 300)
    G = sma_inputs.dyadic((R, k, d), 301)
    z, zp, W, U = exact.hier_exact(list(w0), G.tolist(), world, al, ag, 0.125, 0.5)[R]
    assert np.load(tmp_path / "z0.npy").tolist() == [float(v) for v in z]
    assert np.load(tmp_path / "zp0.npy").tolist() == [float(v) for v in zp]
    for g in range(world):
        assert np.load(tmp_path / f"u{g}.npy").tolist() == [float(v) for v in U[g]], g
    for j in range(k):
        assert np.load(tmp_path / f"w{j}.npy").tolist() == [float(v) for v in W[j]], j


def _hier_ckpt_worker(rank, world, port, flags, d, k, out):
    """Two-level rule over 3 phases: 5 rounds; checkpoint every vector
    (replicas, u_g, z, z_prev), 2 more rounds, restore the checkpoint (so those
    2 rounds are undone) and change alpha_g; 2 local-only iterations (tau);
    restart (replicas, u_g, z_prev := z); 3 more rounds."""
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import sma_inputs
    from paper_1901_02244_b200 import sma
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    al, g, m = (float(np.float32(x)) for x in (0.25, 0.1, 0.9))
    h = sma.Sma(d, k, al, g, m, sma_inputs.w0(d), rank=rank, world=world, device=0,
                flags=flags | sma.FLAG_P2P_ZSYNC | sma.FLAG_HIERARCHICAL)
    handles = [None] * world
    dist.all_gather_object(handles, sma.sma_p2p_handle(h.h))
    sma.sma_p2p_connect(h.h, handles)
    dist.barrier()
    s = torch.cuda.Stream()

    def rnd(i, local=False):
        h.synth_grads(i, sma_inputs.SEED_G, s)
        (h.step_local if local else h.step)(s)

    for i in range(5):
        rnd(i)
    s.synchronize()
    ck = (h.central(), h.central_prev(), [h.replica(j) for j in h.local_replicas()],
          h.reference() if rank else None)
    for i in range(5, 7):
        rnd(i)
    s.synchronize()
    dist.barrier()
    h.set_central(ck[0], ck[1])
    for j, w in zip(h.local_replicas(), ck[2]):
        h.set_replica(j, w)
    if rank:
        h.set_reference(ck[3])
    h.set_alpha_global(float(np.float32(0.125)))
    dist.barrier()
    for i in range(7, 9):
        rnd(i, local=True)
    h.restart(s)
    for i in range(9, 12):
        rnd(i)
    s.synchronize()
    np.save(os.path.join(out, f"z{rank}.npy"), h.central())
    np.save(os.path.join(out, f"u{rank}.npy"), h.reference())
    for j in h.local_replicas():
        np.save(os.path.join(out, f"w{j}.npy"), h.replica(j))
    dist.barrier()
    h.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["A", "B"])
def test_p2p_hierarchical_checkpoint_tau_restart(orc, tmp_path, mode):
    """Checkpoint / restore of the complete two-level state (sma_get/set_reference
    with the central model and the replicas), alpha_g changed between rounds,
    tau-periodic local iterations (R17) and restart, 3 ranks / 7 learners, vs the
    two-level oracle driven through the same sequence."""
    import torch.multiprocessing as mp

    import sma_inputs
    world, k, d = 3, 7, 20_011
    mp.spawn(_hier_ckpt_worker, args=(world, _port(), {"A": 0, "B": 1}[mode], d, k,
                                      str(tmp_path)), nprocs=world)
    f = lambda x: float(np.float32(x))  # noqa: E731
    al, g, m = f(0.25), f(0.1), f(0.9)
    G = lambda i: np.stack([sma_inputs.grad(i, j, k, d) for j in range(k)])  # noqa: E731
    st = orc.HierState.init(sma_inputs.w0(d), k, world)
    for i in range(5):
        st.round(G(i), al, f(1 / (2 * (world - 1))), g, m)
    ag = f(0.125)
    for i in range(7, 9):  # local-only iterations: w_j -= gamma g_j
        st.W = st.W - g * G(i)
    st.W[:] = st.z                         # restart: replicas, u_g, z_prev := z
    st.U[:] = st.z
    st.z_prev = st.z.copy()
    for i in range(9, 12):
        st.round(G(i), al, ag, g, m)
    rel = lambda x, y: np.max(np.abs(x - y) / (1 + np.abs(y)))  # noqa: E731
    assert rel(np.load(tmp_path / "z0.npy"), st.z) <= 1e-5
    for r in range(world):
        assert rel(np.load(tmp_path / f"u{r}.npy"), st.U[r]) <= 1e-5
    for j in range(k):
        assert rel(np.load(tmp_path / f"w{j}.npy"), st.W[j]) <= 1e-5


@pytest.mark.parametrize("world,k", [(2, 4), (3, 7), (4, 8)])
@pytest.mark.parametrize("mode", ["A", "B", "B_graph"])
def test_p2p_push_equals_pull_bitwise(orc, tmp_path, world, k, mode):
    """SMA_FLAG_P2P_PUSH (the replica kernel's epilogue stores each partial chunk
    into its owner's slot over peer memory; the z-sync sums local slots) gives
    the same bits as the pull z-sync (peer loads of every partial), and both
    match the oracle; 2-4 ranks as processes on one GPU, uneven splits."""
    import torch.multiprocessing as mp

    import sma_inputs
    from paper_1901_02244_b200 import sma
    flags = {"A": 0, "B": 1, "B_graph": 1 | 8}[mode]
    d, R = 100_003, 12
    res = {}
    for push in (0, sma.FLAG_P2P_PUSH):
        out = tmp_path / f"p{push}"
        out.mkdir()
        mp.spawn(_worker, args=(world, _port(), flags | push, d, k, R, str(out)), nprocs=world)
        res[push] = out
    for g in range(world):
        assert np.array_equal(np.load(res[0] / f"z{g}.npy"), np.load(res[sma.FLAG_P2P_PUSH] / f"z{g}.npy"))
    for j in range(k):
        assert np.array_equal(np.load(res[0] / f"w{j}.npy"), np.load(res[sma.FLAG_P2P_PUSH] / f"w{j}.npy"))
    zr, _, _ = orc.run_synth(d, k, float(np.float32(1 / k)), float(np.float32(0.1)),
                             float(np.float32(0.9)), R, sma_inputs.SEED_W, sma_inputs.SEED_G,
                             want_W=False)
    z = np.load(res[sma.FLAG_P2P_PUSH] / "z0.npy")
    assert np.max(np.abs(z - zr) / (1 + np.abs(zr))) <= 1e-5


@pytest.mark.parametrize("mode", ["A", "B"])
def test_p2p_push_hierarchical_matches_oracle(orc, tmp_path, mode):
    """The push epilogue also carries the two-level rule's partials (kHierA/B/B0)."""
    import torch.multiprocessing as mp

    import sma_inputs
    from paper_1901_02244_b200 import sma
    world, k, d, R = 3, 7, 100_003, 12
    al = float(np.float32(0.25))
    mp.spawn(_hier_worker, args=(world, _port(), {"A": 0, "B": 1}[mode] | sma.FLAG_P2P_PUSH, d, k, R,
                                 al, None, False, str(tmp_path)), nprocs=world)
    f = lambda x: float(np.float32(x))  # noqa: E731
    zr, _, Wr, Ur = orc.hier_run_synth(d, world, k, al, f(1 / (2 * (world - 1))), f(0.1), f(0.9), R,
                                       sma_inputs.SEED_W, sma_inputs.SEED_G)
    rel = lambda x, y: np.max(np.abs(x - y) / (1 + np.abs(y)))  # noqa: E731
    assert rel(np.load(tmp_path / "z0.npy"), zr) <= 1e-5
    for g in range(1, world):
        assert rel(np.load(tmp_path / f"u{g}.npy"), Ur[g]) <= 1e-5
    for j in range(k):
        assert rel(np.load(tmp_path / f"w{j}.npy"), Wr[j]) <= 1e-5
