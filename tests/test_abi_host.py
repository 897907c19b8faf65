"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and its host bookkeeping is bit-exact with the oracle's
independent implementation (SURVEY.md §8b "Bookkeeping")."""
import os
import re

import numpy as np
import pytest

from paper_1901_02244_b200 import sma

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1901_02244_b200 import _build
    _build.build()
    return sma.load()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "sma.h")).read()
    declared = set(re.findall(r"^\s*(?:sma_status|void|int64_t|int|const char\*)\s+(sma_\w+)\s*\(",
                              hdr, flags=re.M))
    assert declared, "header parse failed"
    assert declared == set(sma.EXPORTS), declared ^ set(sma.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert sma.sma_abi_version() == 2


def test_library_has_sm100a_code_and_no_torch_link():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", sma.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    ldd = subprocess.run(["ldd", sma.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in ldd and "nccl" not in ldd


@pytest.mark.parametrize("k,n", [(1, 1), (4, 1), (16, 2), (16, 4), (16, 8), (16, 3), (5, 4),
                                 (3, 8), (32, 8), (7, 5), (64, 1)])
def test_replica_map_matches_oracle(lib, orc, k, n):
    for j in range(k):
        assert sma.sma_plan_replica_location(k, n, j) == orc.replica_location(k, n, j)
    firsts = [sma.sma_plan_local_replicas(k, n, g) for g in range(n)]
    for g, (f, c) in enumerate(firsts):
        owned = [j for j in range(k) if orc.replica_location(k, n, j)[0] == g]
        assert list(range(f, f + c)) == owned


@pytest.mark.parametrize("d,n", [(1, 1), (7, 4), (7850, 1), (431080, 1), (464154, 8),
                                 (25557032, 8), (138357544, 8), (1000, 3), (4099, 6)])
def test_shards_match_oracle(lib, orc, d, n):
    assert sma.sma_plan_d_pad(d, n) == orc.d_pad(d, n)
    for g in range(n):
        assert sma.sma_plan_shard_range(d, n, g) == orc.shard_range(d, n, g)


@pytest.mark.parametrize("N,k,b,seed", [(200, 3, 8, 42), (60000, 4, 16, 7), (1000, 16, 4, 1)])
def test_batch_indices_match_oracle(lib, orc, N, k, b, seed):
    E = N // (k * b)
    for rnd in [0, 1, E - 1, E, 2 * E + 3]:
        for j in {0, k - 1, k // 2}:
            assert np.array_equal(sma.sma_plan_batch_indices(N, k, b, seed, rnd, j),
                                  orc.batch_indices(N, k, b, seed, rnd, j))


def test_invalid_arguments_rejected_before_any_device_work(lib):
    w0 = np.zeros(8, np.float32)
    for kw, what in [(dict(d=0, k=2), "d must be"), (dict(d=8, k=0), "k must be"),
                     (dict(d=8, k=2, rank=2, world=2), "rank/world"),
                     (dict(d=8, k=2, world=2), "nccl_id"),
                     (dict(d=8, k=2, alpha=float("nan")), "non-finite")]:
        args = dict(d=8, k=2, alpha=0.5, gamma=0.1, mu=0.9, rank=0, world=1, device=0,
                    nccl_id=None, flags=0)
        args.update(kw)
        with pytest.raises(sma.SmaError) as e:
            sma.sma_create(sma.sma_config(**args), w0)
        assert e.value.status == 1 and what in str(e.value)
    with pytest.raises(sma.SmaError):
        sma.sma_plan_replica_location(4, 2, 4)
    with pytest.raises(sma.SmaError):
        sma.sma_plan_batch_indices(10, 4, 4, 0, 0, 0)   # N < k*b


def test_no_cpu_fallback_without_gpu(lib):
    """On a machine without a usable GPU the product path fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sma.SmaError) as e:
        sma.Sma(16, 2, 0.5, 0.1, 0.9, np.zeros(16, np.float32))
    assert e.value.status == 5


def test_binding_refuses_missing_library(monkeypatch, tmp_path):
    monkeypatch.setattr(sma, "_lib", None)
    monkeypatch.setattr(sma, "LIB_PATH", str(tmp_path / "libsma.so"))
    with pytest.raises(ImportError):
        sma.load()


def test_autotune_matches_oracle(lib, orc):
    """libsma's Alg. 2 (independent implementation) == the oracle's, on random
    throughput traces, including the l > 0 guard."""
    rng = np.random.default_rng(4)
    for trial in range(50):
        m = int(rng.integers(1, 9))
        l = rng.integers(0, 4, m)
        tp = rng.uniform(0, 100, m)
        t = tp + rng.uniform(-20, 20, m)
        tau = float(rng.uniform(0, 10))
        a = sma.sma_autotune_step(tau, t, l, tp)
        b = orc.autotune_step(tau, t, l, tp)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
