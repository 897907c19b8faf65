#!/usr/bin/env python
"""Benchmark of the SMA hot path (arXiv 1901.02244, Alg. 1) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl sma|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1)

Workload (BASELINE.json metric, config C4): one SMA round at ResNet-50 size,
d = 25,557,032 parameters, k = 16 replicas in total (strong scaling: r = 16/N
per GPU), alpha = 1/16, gamma = 0.1, mu = 0.9, fp32, synthetic gradients
 resident in HBM.  A "step" is one full round
(a3-a9: replica kernel, per-GPU partial, [NCCL RS, shard update, NCCL AG]).
The per-round working set (>= 3.4 GB per GPU at N = 1, 0.85 GB at N = 8) is
far larger than the 126 MB L2, so no L2 flush is needed between steps.

Prints ONE JSON line on rank 0 (the driver's contract), with `roofline`
(dominant kernel: the replica kernel, algorithmic bytes / CUDA-event time vs
MEASURED_PEAKS.json), `cpu_baseline` (the fp64 oracle on the host, bounded
sample), `e2e` (through the C ABI with host buffers) and `clocks`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import sma_inputs  # noqa: E402

METRIC = ("SMA rounds/sec and HBM/NVLink GB/s vs peak at ResNet-50 size, k replicas, "
          "1/2/4/8 B200")
UNIT = "rounds/s"
HBM_FALLBACK_GBS = 6650.0
NVLINK_PEAK_GBS = 770.0   # measured per-direction peer bandwidth (B200_PROFILING.md)
# L2-resident rounds (C1-C3, the learners): the L2 slice (LTS) throughput cap of
# /opt/skills/guides/B300_MICROARCH.md ("~6300 B/cyc full-chip", measured on B300)
# x the B200's 1,965 MHz max SM clock.  torch's own L2-resident copy / add kernels
# reach 8.2 / 9.2 TB/s on this B200 (profiles/r02_l2_bw.json), below our replica
# kernel at C3, so the guide's cap is the denominator.
L2_PEAK_GBS = 6300 * 1.965
L2_BYTES = 126 * (1 << 20)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["sma", "reference"], default="sma")
    ap.add_argument("--config", default="C4", choices=["C1", "MLP", "C2", "C3", "C4", "C5"],
                    help="C4 is the metric's workload; C1/MLP run the built-in learner in the loop")
    ap.add_argument("--k", type=int, default=None, help="override total replicas")
    ap.add_argument("--mode", choices=["auto", "A", "B"], default="auto",
                    help="collective path mode when N > 1 (auto = B, the overlapped round)")
    ap.add_argument("--tma", action="store_true", help="force the TMA-staged replica kernel")
    ap.add_argument("--ldg", action="store_true", help="force the direct-load replica kernel")
    ap.add_argument("--matc", action="store_true", help="north_star-literal c_j materialisation")
    ap.add_argument("--force-collective", action="store_true")
    ap.add_argument("--zsync", choices=["auto", "nccl", "nvls", "p2p"], default="auto",
                    help="inter-GPU z-sync: one fused kernel over IPC-mapped peer memory (p2p), "
                         "NCCL RS/AG (nccl), or one fused kernel over NVSwitch multicast (nvls); "
                         "auto = p2p, falling back to nccl if the peer mapping cannot be set up")
    ap.add_argument("--tau", type=int, default=1,
                    help="synchronise every tau iterations (sma_step_local on the others; "
                         "0 = never: the paper's 'no synchronisation' point, fig:overhead)")
    ap.add_argument("--push", action="store_true",
                    help="with the P2P z-sync: the replica kernel pushes each partial chunk into "
                         "its owner's slot over peer memory (SMA_FLAG_P2P_PUSH)")
    ap.add_argument("--hier", action="store_true",
                    help="Section 3.3 two-level rule (per-GPU reference models, R20): "
                         "alpha_l = 1/(2r), alpha_g = 1/(2(N-1)); identical to flat SMA at N = 1")
    ap.add_argument("--rounds-per-call", type=int, default=1,
                    help="learner configs: rounds per sma_learner_steps call (the MLP learner "
                         "then runs the rounds of one epoch in one launch of its fused kernel); "
                         "1 = one sma_learner_step per round")
    ap.add_argument("--emulate-n", type=int, default=0,
                    help="measurement only, 1 GPU with --force-collective --zsync p2p: the 1-rank "
                         "z-sync moves the HBM traffic ONE GPU of an N-rank job sees (whole partial "
                         "read, whole z written, z/z_prev read on 1/N) while the replica kernel of "
                         "r = k/N replicas runs -- the per-GPU load of N GPUs (SMA_P2P_EMULATE_N); "
                         "the z it computes is wrong, so the line is not a bench value")
    ap.add_argument("--emulate-ctas", type=int, default=0,
                    help="with --emulate-n: cap the z-sync grid (SMA_P2P_CTAS) to pace its traffic "
                         "like the NVLink-bound real one")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            j = json.load(open(p))
            return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def host_info():
    """The host the oracle ran on: online cores and the CPU model (/proc/cpuinfo)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def cpu_baseline(d, k, alpha, gamma, mu, rounds=3):
    """The oracle as it stands (fp64, single thread) timed on the host for
    `rounds` FULL SMA rounds of the same workload (all k replicas, all d
    parameter indices, synthetic gradients generated inside, initialisation
    included; SURVEY §8d "3 full-vector oracle rounds"), and the same rounds
    with the index set split over every host core (OpenMP build of the same
    source, bitwise the same result).  Measured, not
    extrapolated: value = rounds / seconds."""
    import oracle
    oracle.build()
    t = time.perf_counter()
    oracle.run_synth(d, k, alpha, gamma, mu, rounds, sma_inputs.SEED_W, sma_inputs.SEED_G,
                     want_W=False)
    dt = time.perf_counter() - t
    omp = None
    try:
        t = time.perf_counter()
        _, _, nt = oracle.run_synth_omp(d, k, alpha, gamma, mu, rounds, sma_inputs.SEED_W,
                                        sma_inputs.SEED_G, np.arange(d, dtype=np.int64))
        dto = time.perf_counter() - t
        omp = {"value": rounds / dto, "unit": UNIT, "cores": nt, "kind": "oracle",
               "sample": f"the same {rounds} full rounds, index set split over {nt} OpenMP "
                         f"threads, {dto:.1f} s"}
    except Exception as e:  # noqa: BLE001 -- a missing OpenMP runtime only drops this field
        omp = {"unavailable": str(e)[:200]}
    return {"value": rounds / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "host": host_info(), "all_cores": omp,
            "sample": f"{rounds} full SMA rounds (k={k}, all d={d} parameter indices, synthetic "
                      f"gradients generated inside, init included), fp64 single-thread C oracle, "
                      f"{dt:.1f} s measured"}


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only).
    Each step is one FULL SMA round of the workload (all d indices, all k
    replicas, the step's synthetic gradients generated inside it) when the
    whole --steps/--warmup run fits in ~3 minutes at ~4 s per round; beyond
    that each step is a seeded sample of parameter indices (SMA with given
    gradients is separable per index) and the line says so."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = sma_inputs.CONFIGS[args.config]
    d = cfg["d"]
    k = args.k or 16
    alpha, gamma, mu = float(np.float32(1 / k)), float(np.float32(0.1)), float(np.float32(0.9))
    import oracle
    oracle.build()
    full_round_s = 4.5 * d * k / (25_557_032 * 16)     # measured order of one full C4 round
    n_steps = args.steps + args.warmup
    if n_steps * full_round_s <= 180:
        n_idx = d
    else:
        n_idx = max(1 << 14, int(d * 180 / (n_steps * full_round_s)))
    rng = np.random.default_rng(1)
    idx = np.sort(rng.choice(d, n_idx, replace=False)) if n_idx < d else np.arange(d)
    state = oracle.State.init(sma_inputs.w0(d, idx=idx).astype(np.float64), k)
    G = np.empty((k, n_idx))
    step_times = []
    for s in range(n_steps):
        t = time.perf_counter()
        for j in range(k):
            G[j] = oracle.synth_grad(d, k, s, j, sma_inputs.SEED_G, idx)
        state.round(G, alpha, gamma, mu)
        dt = time.perf_counter() - t
        if s >= args.warmup:
            step_times.append(dt)
    tot = sum(step_times)
    sample_s = tot / args.steps
    value = args.steps * (n_idx / d) / tot
    if n_idx == d:
        sample = (f"each step: one full SMA round (k={k}, all d={d} parameter indices, the "
                  f"step's synthetic gradients generated inside it); fp64 single-thread C "
                  f"oracle; {sample_s:.2f} s per step measured")
    else:
        sample = (f"each step: one SMA round (k={k}, synthetic gradients generated in the step) "
                  f"over {n_idx} of d={d} parameter indices ({sample_s:.3f} s per step "
                  f"measured), scaled by d/{n_idx} to rounds/s of the full vector; fp64 "
                  f"single-thread C oracle")
    d_pad = oracle.d_pad(d, args.gpus)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * sample_s, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(args, args.gpus, d, d_pad, k, alpha, gamma, mu),
            "full_vector_steps": n_idx == d,
            "measured_s_per_step": sample_s, "indices_per_step": n_idx,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "host": host_info(), "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def arm_config(args, world, d, d_pad, k, alpha, gamma, mu, zsync=None, push=False):
    """The `config` object of the JSON line (the same for both arms)."""
    collective = world > 1 or args.force_collective
    mode = "fused" if not collective else ("A" if args.mode == "A" else "B")
    if zsync is None:
        zsync = args.zsync if args.zsync != "auto" else ("p2p" if collective else "none")
    r = k // world if k % world == 0 else -(-k // world)
    alg_bytes = 4 * d_pad * (3 * r + (3 if mode == "fused" else 2))
    return {"workload": workload_name(args.config, d, k), "d": d, "d_pad": d_pad,
            "k": k, "replicas_per_gpu": r, "alpha": alpha, "gamma": gamma, "mu": mu,
            "mode": mode, "kernel": "tma" if args.tma else "ldg",
            "materialize_c": bool(args.matc), "hierarchical": bool(args.hier),
            "parallelism": f"sma-dp{world}" + ("" if not collective else f"+{zsync}-zsync") +
                           ("-push" if push else ""),
            "l2": l2_note(d_pad, r)}


def working_set(d_pad, r):
    """Bytes a round touches per GPU: r replicas + r gradients + z and z_prev."""
    return 4 * d_pad * (2 * r + 2)


def l2_note(d_pad, r):
    ws = working_set(d_pad, r)
    if ws > L2_BYTES:
        return f"no flush: per-round working set {ws / 1e9:.2f} GB/GPU >> 126 MB L2"
    return (f"L2-resident: per-round working set {ws / 1e6:.1f} MB/GPU < 126 MB L2, not flushed "
            "(the rounds of a training loop reuse it); roofline against the L2 throughput cap")


def nvlink_counters(device):
    """Cumulative NVLink data counters of one GPU (KiB transmitted / received,
    summed over its links) from `nvidia-smi nvlink -gt d`; None where the GPU
    has no NVLink or the query is unsupported."""
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(device)],
                             capture_output=True, text=True, timeout=10).stdout
    except Exception:  # noqa: BLE001
        return None
    tx = rx = 0
    seen = False
    for line in out.splitlines():
        low = line.lower()
        if "kib" not in low:
            continue
        try:
            val = int(line.split(":")[-1].strip().split()[0])
        except (ValueError, IndexError):
            continue
        if "tx" in low:
            tx += val
            seen = True
        elif "rx" in low:
            rx += val
            seen = True
    return (tx * 1024, rx * 1024) if seen else None


def nvlink_block(zsync, mode, world, d_pad, phase_avg, serial, link_counters, rank_info):
    """NVLink side of the metric for the collective path.  Link bytes are
    counted PER DIRECTION per GPU and compared with the 770 GB/s per-direction
    peer bandwidth, so frac <= 1 holds by construction:
      NCCL ring RS, AG:        4 d_pad (n-1)/n each (nccl-tests busBW convention),
                               run one after the other;
      fused P2P z-sync (pull): ingress = the n-1 peers' partial shards and egress =
                               this GPU's z shard to n-1 peers, 4 d_pad (n-1)/n each way,
                               concurrently in one kernel (push: the same bytes, the
                               partial leg during the replica kernel);
      NVLS z-sync:             ~4 d_pad per direction (multimem ld_reduce / st)."""
    one = 4 * d_pad * (world - 1) / world
    rs_ms, up_ms, ag_ms, fz_ms = phase_avg[1], phase_avg[2], phase_avg[3], phase_avg[4]
    gbs = lambda b, ms_: (b / (ms_ * 1e-3) / 1e9) if ms_ > 0 else None  # noqa: E731
    per_dir = one if zsync in ("p2p", "nccl") else 4 * d_pad
    if fz_ms > 0:
        bus = gbs(per_dir, fz_ms)
        how = "fused z-sync kernel: per-direction link bytes / its event time"
    else:
        bus = gbs(2 * one, rs_ms + ag_ms)   # RS then AG, each 4 d_pad (n-1)/n per direction
        how = "NCCL RS + AG (sequential): per-direction link bytes of both / their summed time"
    blk = {
        "zsync": zsync, "link_bytes_per_direction_per_gpu_per_round": per_dir if fz_ms > 0
        else 2 * one,
        "reduce_scatter_ms": rs_ms, "shard_update_ms": up_ms, "all_gather_ms": ag_ms,
        "fused_zsync_ms": fz_ms, "rs_bus_gbs": gbs(one, rs_ms), "ag_bus_gbs": gbs(one, ag_ms),
        "bus_gbs_per_direction": bus, "peak_gbs_per_direction": NVLINK_PEAK_GBS,
        "frac": (bus / NVLINK_PEAK_GBS) if bus else None, "how": how,
        "note": "times from CUDA events around each phase on its stream, max over ranks" +
                ("; in Mode B the z-sync runs concurrently with the replica kernel"
                 if mode == "B" else ""),
        "ranks": rank_info}
    if serial is not None:
        s_rs, s_ag, s_fz = serial[2], serial[4], serial[5]
        s_bus = gbs(per_dir, s_fz) if s_fz > 0 else gbs(2 * one, s_rs + s_ag)
        blk["serial_mode_a"] = {
            "ms_per_round": serial[0], "replica_ms": serial[1], "reduce_scatter_ms": s_rs,
            "shard_update_ms": serial[3], "all_gather_ms": s_ag, "fused_zsync_ms": s_fz,
            "bus_gbs_per_direction": s_bus,
            "frac": (s_bus / NVLINK_PEAK_GBS) if s_bus else None,
            "note": "separate Mode-A handle, same workload, z-sync not overlapped"}
    if link_counters is not None:
        blk["measured_link_bytes"] = link_counters
    return blk


def workload_name(cfg, d, k):
    names = {"C2": "LeNet-sized", "C3": "ResNet-32-sized", "C4": "ResNet-50-sized",
             "C5": "VGG-16-sized", "C1": "softmax-regression learner in the loop,",
             "MLP": "MLP 784-256-10 learner in the loop,"}
    return f"{cfg}: SMA round, {names[cfg]} vector d={d}, k={k} replicas, fp32"


def main():
    args = parse()
    if args.emulate_n:
        os.environ["SMA_P2P_EMULATE_N"] = str(args.emulate_n)
        if args.emulate_ctas:
            os.environ["SMA_P2P_CTAS"] = str(args.emulate_ctas)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1901_02244_b200 import sma

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # SMA_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0, gloo for the
    # host-side plumbing and the P2P z-sync (NCCL cannot put two ranks on one
    # GPU), so the N > 1 code path of this script runs on a 1-GPU box
    shared = os.environ.get("SMA_BENCH_SHARED_GPU") == "1" and world > 1
    if shared:
        local = 0
        args.zsync = "p2p"
    torch.cuda.set_device(local)
    red_dev = "cpu" if shared else "cuda"   # device of the small reduction tensors
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg = sma_inputs.CONFIGS[args.config]
    d = cfg["d"]
    k = args.k or (16 if args.config == "C4" else cfg["k"])
    alpha, gamma, mu = float(np.float32(1 / k)), float(np.float32(0.1)), float(np.float32(0.9))
    learner = args.config in ("C1", "MLP")

    collective = world > 1 or args.force_collective
    mode = "fused" if not collective else ("A" if args.mode == "A" else "B")
    # Per-phase CUDA events (SMA_FLAG_TIMING) are OFF in the timed region: each
    # costs ~2.5 us of GPU time between kernels (C2: 13.7 vs 8.2 us per round).
    # A round that is one kernel (the fused n = 1 path) gets its kernel's average
    # launch duration from the timed window itself; otherwise a separate pass
    # with the events on (sma_set_timing) measures the phases.
    flags = sma.FLAG_CUDA_GRAPH if os.environ.get("SMA_BENCH_GRAPH") == "1" else 0
    if collective:
        flags |= sma.FLAG_FORCE_COLLECTIVE
        if mode == "B":
            flags |= sma.FLAG_OVERLAP
    if args.tma:
        flags |= sma.FLAG_KERNEL_TMA
    if args.ldg:
        flags |= sma.FLAG_KERNEL_LDG
    use_tma = args.tma      # libsma's default is the direct-load kernel
    if args.matc:
        flags |= sma.FLAG_MATERIALIZE_C
    if args.zsync == "nvls" and collective:
        flags |= sma.FLAG_NVLS_ZSYNC
    if args.zsync in ("p2p", "auto") and collective:
        flags |= sma.FLAG_P2P_ZSYNC
    if args.push and (flags & sma.FLAG_P2P_ZSYNC):
        flags |= sma.FLAG_P2P_PUSH
    if args.hier:   # alpha is the intra-GPU alpha_l = 1/(2r); alpha_g keeps libsma's default
        flags |= sma.FLAG_HIERARCHICAL
        alpha = float(np.float32(1 / (2 * max(1, k // world))))

    nccl_id = nccl_id_a = None
    if world > 1:   # one NCCL id per libsma communicator (the bench may create two)
        obj = [(sma.sma_nccl_unique_id(), sma.sma_nccl_unique_id()) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id, nccl_id_a = obj[0]

    w0 = sma_inputs.w0(d) if not learner else \
        np.random.default_rng(6).normal(0, 0.05 if args.config == "MLP" else 0.0, d).astype(np.float32)
    def make_handle(fl):
        hh = sma.Sma(d, k, alpha, gamma, mu, w0, rank=rank, world=world, device=local,
                     nccl_id=nccl_id, flags=fl)
        if (fl & sma.FLAG_P2P_ZSYNC) and world > 1:   # map every rank's buffers (CUDA IPC)
            handles = [None] * world
            dist.all_gather_object(handles, sma.sma_p2p_handle(hh.h))
            sma.sma_p2p_connect(hh.h, handles)
        return hh

    zsync = args.zsync if args.zsync != "auto" else ("p2p" if collective else "none")
    if args.zsync == "auto" and world > 1:
        # every rank must take the same path: agree on whether the peer mapping worked
        ok, h, err = 1, None, ""
        try:
            h = make_handle(flags)
        except Exception as e:  # noqa: BLE001 -- any setup failure selects NCCL
            ok, err = 0, str(e)
        flag_t = torch.tensor([ok], dtype=torch.int32, device=red_dev)
        dist.all_reduce(flag_t, op=dist.ReduceOp.MIN)
        if int(flag_t[0]) == 0:
            if h is not None:
                h.close()
            if rank == 0:
                print(f"p2p z-sync unavailable ({err or 'on another rank'}); using NCCL",
                      file=sys.stderr, flush=True)
            flags &= ~sma.FLAG_P2P_ZSYNC
            zsync = "nccl"
            h = make_handle(flags)
    else:
        h = make_handle(flags)
    r = h.local_count
    rank_info = None
    if collective:   # per-rank evidence: device identity and the peer mapping that ran
        pr = torch.cuda.get_device_properties(local)
        me = {"rank": rank, "local_rank": local, "device": pr.name,
              "uuid": str(getattr(pr, "uuid", "")),
              "pci_bus_id": getattr(pr, "pci_bus_id", None),
              "zsync": zsync, "p2p_peers_mapped": (world - 1) if zsync == "p2p" else 0,
              "can_access_peer": [bool(torch.cuda.can_device_access_peer(local, q))
                                  for q in range(torch.cuda.device_count()) if q != local]}
        rank_info = [None] * world
        if world > 1:
            dist.all_gather_object(rank_info, me)
        else:
            rank_info = [me]
    stream = torch.cuda.Stream()
    rnd = [0]
    if learner:   # MNIST-shaped synthetic blobs resident in HBM, learner in the loop
        X, y = sma_inputs.blobs(60_000, seed=4)
        Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
        sma.sma_learner_attach(h.h, 0 if args.config == "C1" else 1, 784,
                               256 if args.config == "MLP" else 0, 10, cfg["batch"], Xd, yd,
                               X.shape[0], 99)

        def run_steps(n):   # learner gradient + round, n rounds
            if args.rounds_per_call <= 1:
                for _ in range(n):
                    sma.sma_learner_step(h.h, rnd[0], stream)
                    rnd[0] += 1
                return
            while n > 0:
                c = min(n, args.rounds_per_call)
                sma.sma_learner_steps(h.h, rnd[0], c, stream)
                rnd[0] += c
                n -= c
    else:
        h.synth_grads(0, sma_inputs.SEED_G, stream)   # inputs resident in HBM before timing

        def run_steps(n):
            # tau = 1: every iteration is a full SMA round; tau > 1 / 0: the E11
            # analog with local-only iterations in between
            for _ in range(n):
                rnd[0] += 1
                if args.tau == 1 or (args.tau > 1 and rnd[0] % args.tau == 0):
                    h.step(stream)
                else:
                    h.step_local(stream)
    stream.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ------------------------------------------------- warm-up, clock sampling
    # The clock sampler (nvidia-smi) starts first and the W warm-up steps run
    # after its start-up pause, right before the timed region: an idle GPU
    # drops its clocks, and a short timed region (C1: ~10 ms) measured ~25 %
    # slower when it followed the pause directly.
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    run_steps(args.warmup)
    barrier()

    # ------------------------------------------------------------ timed region
    l0 = h.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    run_steps(args.steps)
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = h.launch_count() - l0
    clk = clocks.stop()
    # phase durations: replica kernel, reduce-scatter, shard update, all-gather,
    # fused z-sync
    one_kernel = mode == "fused" and not learner and args.tau == 1
    if one_kernel:   # K back-to-back launches of the one kernel of a round
        phase_avg = [ms / args.steps, 0.0, 0.0, 0.0, 0.0]
        timing_src = "timed window / K (each round is one kernel launched back to back)"
    else:
        h.set_timing(True)
        nt = max(20, args.steps // 5)
        for ph in range(5):
            h.kernel_time(reset=True, phase=ph)
        run_steps(nt)
        barrier()
        phase_avg = []
        for ph in range(5):
            pm, pn = h.kernel_time(reset=True, phase=ph)
            phase_avg.append(pm / pn if pn else 0.0)
        h.set_timing(False)
        timing_src = (f"CUDA events around each phase on its stream, in a separate pass of {nt} "
                      "steps after the timed region (events would slow the timed rounds)")

    t = torch.tensor([ms, *phase_avg, float(launches)], dtype=torch.float64, device=red_dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms_max, phase_avg = float(tmax[0]), [float(x) for x in tmax[1:6]]
        launches_total = int(tsum[6])
    else:
        ms_max, launches_total = ms, launches
    kern_avg = phase_avg[0]

    # ---------------------------------------------- clean NVLink measurement
    # In Mode B the collectives overlap the replica kernel, so their event
    # times include contention.  For N > 1 a second, Mode-A handle (same
    # workload) runs a short serial pass: its reduce-scatter / all-gather times
    # give the uncontended NVLink bus bandwidth (nccl-tests convention).
    serial = None
    link_counters = None
    if collective and mode == "B" and zsync in ("nccl", "p2p"):
        nccl_id_main, nccl_id = nccl_id, nccl_id_a   # the second handle's own communicator
        hA = make_handle((flags & ~sma.FLAG_OVERLAP) | sma.FLAG_TIMING)
        nccl_id = nccl_id_main
        hA.synth_grads(0, sma_inputs.SEED_G, stream)
        for _ in range(5):
            hA.step(stream)
        barrier()
        for ph in range(5):
            hA.kernel_time(reset=True, phase=ph)
        ns = max(10, args.steps // 4)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0 = nvlink_counters(local)
        e0.record(stream)
        for _ in range(ns):
            hA.step(stream)
        e1.record(stream)
        barrier()
        c1 = nvlink_counters(local)
        mine = None
        if c0 is not None and c1 is not None:
            mine = {"rank": rank, "tx_bytes_per_round": (c1[0] - c0[0]) / ns,
                    "rx_bytes_per_round": (c1[1] - c0[1]) / ns}
        allc = [None] * world
        if world > 1:
            dist.all_gather_object(allc, mine)   # every rank joins, counters or not
        else:
            allc = [mine]
        if any(x is not None for x in allc):
            link_counters = {"serial_mode_a_pass": allc,
                             "source": "nvidia-smi nvlink -gt d (cumulative data KiB over all "
                                       "links of each rank's GPU), delta over the serial "
                                       "Mode-A pass / its rounds"}
        pa = []
        for ph in range(5):
            pm, pn = hA.kernel_time(reset=True, phase=ph)
            pa.append(pm / pn if pn else 0.0)
        ta = torch.tensor([e0.elapsed_time(e1) / ns, *pa], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(ta, op=dist.ReduceOp.MAX)
        serial = [float(x) for x in ta]
        hA.close()

    # ------------------------------------------------------------------ e2e
    # Every step copies its inputs (all local learners' gradients) from pinned
    # host memory and reads z back, inside the timed wall-clock region, through
    # the public C ABI only.  Two variants: serial (sma_set_learner_grads_host,
    # sma_step, sma_get_central one after the other) and pipelined -- step s+1's
    # host-to-device copies into the other of libsma's two internal gradient
    # sets overlap step s's round and its read-back of z
    # (sma_stage_grads_host, sma_step, sma_get_central_async, and one
    # sma_synchronize at the end), the way a training loop would stream
    # batches.  The pipelined one is reported as `e2e`.
    e2e = None
    if not args.no_e2e and not learner:
        pinned = [torch.empty(d, dtype=torch.float32).pin_memory() for _ in range(r)]
        for s_ in range(r):
            pinned[s_].copy_(torch.from_numpy(sma_inputs.grad(0, h.local_first + s_, k, d)))
        zout = torch.empty(d, dtype=torch.float32).pin_memory()

        def e2e_step():
            for s_ in range(r):
                sma.sma_set_learner_grads_host(h.h, h.local_first + s_, pinned[s_], stream)
            h.step(stream)
            sma.sma_get_central(h.h, zout, False)

        def timed(fn, n):
            barrier()
            t0 = time.perf_counter()
            fn(n)
            barrier()
            t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=red_dev)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return n / float(t[0])

        e2e_step()
        e2e_serial = timed(lambda n: [e2e_step() for _ in range(n)], args.e2e_steps)

        zouts = [torch.empty(d, dtype=torch.float32).pin_memory() for _ in range(2)]

        def pipelined(n):
            for st in range(n):
                b = st & 1
                sma.sma_stage_grads_host(h.h, b, pinned)      # H2D into gradient set b
                h.step(stream)                                 # waits for set b's copies
                sma.sma_get_central_async(h.h, zouts[b])       # D2H of this round's z
            sma.sma_synchronize(h.h)

        pipelined(2)
        value = timed(pipelined, args.e2e_steps)
        e2e = {"value": value, "unit": UNIT,
               "h2d_bytes_per_step": 4 * d * k, "d2h_bytes_per_step": 4 * d * world,
               "serial_value": e2e_serial,
               "how": "per step, inside the wall-clock region, C ABI calls only: "
                      "sma_stage_grads_host (every local learner's gradient from pinned host "
                      "memory into one of libsma's two gradient sets), sma_step, "
                      "sma_get_central_async (z to pinned host memory); sma_synchronize at the "
                      "end -- step s+1's copies overlap step s's round and read-back.  "
                      "serial_value: sma_set_learner_grads_host / sma_step / sma_get_central "
                      "one after the other; max over ranks"}

    if rank == 0:
        d_pad = h.d_pad
        peak, peak_src = measured_peaks()
        kvar = "tma" if use_tma else "ldg"
        if mode == "fused":
            alg_bytes = 4 * d_pad * (3 * r + 3)
            kname = f"replica_step_{kvar}<kFused>"
        else:
            alg_bytes = 4 * d_pad * (3 * r + 2)
            kname = f"replica_step_{kvar}<kPartial{mode}>"
            if args.hier and mode == "B":   # rank 0 emits the pre-scaled partial (R20)
                kname = f"replica_step_{kvar}<kHierB0>"
        if args.matc:   # replica kernel: r x (read w, g; write w, c) + z; reduce: r x read c
            alg_bytes = 4 * d_pad * (5 * r + (4 if mode == "fused" else 2))
        if args.tau != 1 and not learner:   # mix of sync rounds and local-only iterations
            n_sync = (args.steps // args.tau) if args.tau > 1 else 0
            alg_bytes = (n_sync * alg_bytes + (args.steps - n_sync) * 4 * d_pad * 3 * r) / args.steps
            kname += " / replica_step_ldg<kLocal>"
        achieved = alg_bytes / (kern_avg * 1e-3) / 1e9 if kern_avg > 0 else 0.0
        traffic = None
        # the per-GPU replica kernel depends on (config, r, mode, kernel) only, so the
        # capture of r replicas on one GPU also serves N = k/r GPUs
        tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}_r{r}_{mode}_{kvar}.json")
        if os.path.exists(tpath) and not (args.matc or args.hier or args.tau != 1):
            try:
                traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        value = args.steps / (ms_max * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": arm_config(args, world, d, d_pad, k, alpha, gamma, mu, zsync=zsync,
                                 push=bool(flags & sma.FLAG_P2P_PUSH)),
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": kern_avg,
                         "peak_source": peak_src, "vs_8TBs_spec": achieved / 8000.0,
                         "timing": timing_src} if working_set(d_pad, r) > L2_BYTES else
                        {"bound": "l2", "kernel": kname, "achieved": achieved,
                         "peak": L2_PEAK_GBS, "unit": "GB/s", "frac": achieved / L2_PEAK_GBS,
                         "traffic": traffic, "alg_bytes_per_launch": alg_bytes,
                         "avg_launch_ms": kern_avg,
                         "peak_source": "derived: B300_MICROARCH.md L2 (LTS) throughput cap "
                                        "~6300 B/cycle x 1965 MHz; torch's L2-resident copy/add "
                                        "reach 8.2/9.2 TB/s here (profiles/r02_l2_bw.json)",
                         "vs_hbm_peak": achieved / peak, "timing": timing_src},
            "gpu_launches": launches_total,
            "clocks": clk,
        }
        if collective:
            line["nvlink"] = nvlink_block(zsync, mode, world, d_pad, phase_avg, serial,
                                          link_counters, rank_info)
        if shared:
            line["config"]["shared_gpu_test"] = ("all ranks time-share cuda:0 "
                                                 "(SMA_BENCH_SHARED_GPU): a code-path test, not a "
                                                 "multi-GPU measurement")
        if e2e:
            line["e2e"] = e2e
        if args.emulate_n:
            n_e = args.emulate_n
            line["config"]["emulated_n"] = n_e
            line["config"]["emulated_zsync_ctas"] = args.emulate_ctas or None
            line["config"]["note_emulation"] = (
                f"MEASUREMENT ONLY (not a bench value; the z it computes is wrong): one GPU runs "
                f"the replica kernel of r = k/{n_e} replicas over the full vector and, in Mode B "
                f"concurrently, a 1-rank z-sync that moves the HBM traffic one GPU of a "
                f"{n_e}-rank job sees: the whole partial read ({4 * d_pad} B), the whole z[1-cur] "
                f"written ({4 * d_pad} B), z and z_prev read on 1/{n_e} ({8 * d_pad // n_e} B); "
                f"its NVLink pacing is approximated by capping its grid (emulated_zsync_ctas)")
        if args.tau != 1:
            line["config"]["tau"] = args.tau
            line["config"]["note"] = ("E11 analog (P:1476-1503): iterations/s with "
                                      "synchronisation every tau iterations (0 = never)")
        if learner:
            line["config"]["learner"] = args.config
            line["config"]["batch"] = cfg["batch"]
            line["config"]["rounds_per_call"] = args.rounds_per_call
            line["config"]["l2"] = ("L2-resident working set (replicas, gradients, z and the "
                                    "dataset's batch rows): not flushed")
        if args.config in ("MLP", "C1") and mode == "fused":
            # the round is ONE kernel (learner gradient + fused update:
            # sma_learner_mlp_fused.cu, or the softmax cluster of
            # sma_learner_softmax_fused.cu) unless disabled: a FLOP roofline
            # against the FP32 FFMA peak
            bsz, hid, ind, ncls = cfg["batch"], 256, 784, 10
            if args.config == "MLP":
                flops = r * (4 * bsz * ind * hid + 6 * bsz * hid * ncls)
            else:   # logits + dW: r (2 b in_dim classes + 2 b in_dim classes)
                flops = r * 4 * bsz * ind * ncls
            fused = launches == args.steps
            multi = args.rounds_per_call > 1 and launches < args.steps
            ms_k = kern_avg if fused else ms_max / args.steps
            mhz = clk.get("sm_mhz") or 1965.0
            peak_tf = 148 * 4 * 32 / 2 * 2 * mhz * 1e6 / 1e12
            ach = flops / (ms_k * 1e-3) / 1e12
            kn = "mlp_round_kernel<TU, true>" if args.config == "MLP" else \
                f"softmax_cluster_kernel (one {r}-CTA cluster: {r} of 148 SMs)"
            line["roofline"] = {
                "bound": "alu", "kernel": kn if fused else
                (f"{kn}, {launches} launches for {args.steps} rounds "
                 "(the rounds of one epoch per launch); per-round time = window / K" if multi else
                 "per-round learner kernels + replica kernel (whole round)"),
                "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s", "frac": ach / peak_tf,
                "traffic": None, "flops_per_launch": flops, "avg_launch_ms": ms_k,
                "peak_source": "derived: 148 SMs x 4 SMSPs x 32 lanes / FFMA reciprocal "
                               "throughput 2 (B300_MICROARCH.md: 3-register FFMA rt_SMSP = 2) x 2 "
                               f"FLOP x {mhz:.0f} MHz (median SM clock under load)",
                "note": ("FLOPs = r (4 b in_dim hidden + 6 b hidden classes): layer 1, dW1, "
                         "logits, dW2, da1; the per-learner GEMMs are 16 x 784 x 256 -- a chain "
                         "of dependent phases, latency-bound, not FLOP-bound"
                         if args.config == "MLP" else
                         "FLOPs = r 4 b in_dim classes (logits, dW); one CTA per learner on "
                         "r SMs -- a chain of dependent phases (logits, softmax, z exchange, "
                         "dW, update) with two cluster barriers per round, latency-bound"),
                "timing": timing_src if fused else "timed window / K (CUDA events on the launching "
                                                   "stream around the K rounds)"}
        if not args.no_cpu_baseline and not learner and world == 1:   # rank 0 at N = 1 only
            line["cpu_baseline"] = cpu_baseline(d, k, alpha, gamma, mu)
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
