"""Variant sweep of the replica kernel on one GPU (CUDA-event timing).
python scripts/sweep.py  -> one JSON line per (k, flags) with rounds/s, kernel GB/s."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sma_inputs
from paper_1901_02244_b200 import sma

d = int(os.environ.get("SWEEP_D", sma_inputs.CONFIGS["C4"]["d"]))
steps = int(os.environ.get("SWEEP_STEPS", "300"))
w0 = sma_inputs.w0(d)
L, T = sma.FLAG_KERNEL_LDG, sma.FLAG_KERNEL_TMA
if os.environ.get("SWEEP_TMA_ONLY"):
    cases = [(16, T), (2, T), (8, T), (4, T), (2, T | sma.FLAG_FORCE_COLLECTIVE)]
elif os.environ.get("SWEEP_LDG_ONLY"):
    cases = [(16, L), (2, L), (8, L), (4, L), (2, L | sma.FLAG_FORCE_COLLECTIVE)]
else:
    cases = [(16, L), (16, T), (2, L), (2, T),
             (2, sma.FLAG_FORCE_COLLECTIVE), (2, sma.FLAG_FORCE_COLLECTIVE | T),
             (2, sma.FLAG_FORCE_COLLECTIVE | sma.FLAG_OVERLAP),
             (2, sma.FLAG_FORCE_COLLECTIVE | sma.FLAG_OVERLAP | T),
             (4, L), (4, T), (32, L), (32, T), (16, sma.FLAG_MATERIALIZE_C),
             (16, sma.FLAG_MATERIALIZE_C | L), (2, sma.FLAG_MATERIALIZE_C),
             (2, sma.FLAG_FORCE_COLLECTIVE | sma.FLAG_NVLS_ZSYNC),
             (2, sma.FLAG_FORCE_COLLECTIVE | sma.FLAG_NVLS_ZSYNC | sma.FLAG_OVERLAP)]
for k, flags in cases:
    try:
        h = sma.Sma(d, k, 1.0 / k, 0.1, 0.9, w0, flags=flags | sma.FLAG_TIMING)
    except sma.SmaError as e:
        print(json.dumps({"k": k, "flags": flags, "error": str(e)}), flush=True)
        continue
    s = torch.cuda.Stream()
    h.synth_grads(0, 2244, s)
    for _ in range(10):
        h.step(s)
    torch.cuda.synchronize()
    h.kernel_time(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        h.step(s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    kms, n = h.kernel_time(reset=True)
    kms /= max(n, 1)
    phases = [h.kernel_time(reset=True, phase=p) for p in range(1, 5)]
    coll = bool(flags & sma.FLAG_FORCE_COLLECTIVE)
    nbytes = 4 * h.d_pad * (3 * k + (2 if coll else 3))
    if flags & sma.FLAG_MATERIALIZE_C:
        nbytes = 4 * h.d_pad * (6 * k + 3)
    print(json.dumps({"k": k, "flags": flags, "tma_cfg": os.environ.get("SMA_TMA_CONFIG", "0"), "ms_per_round": ms, "rounds_s": 1000 / ms,
                      "kernel_ms": kms, "kernel_GBs": nbytes / kms / 1e6,
                      "frac": nbytes / kms / 1e6 / 6552.6,
                      "phase_ms": [pm / pn if pn else 0 for pm, pn in phases]}), flush=True)
    h.close()
