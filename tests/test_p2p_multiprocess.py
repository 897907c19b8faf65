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
