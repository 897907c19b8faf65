"""Per-round time of the fused n = 1 round vs model size, back to back on one
stream (the bench's small-round regime): where does the launch-to-launch floor
sit, and how much of a C2 / C3 round is bandwidth?  Prints one JSON line per
(d, k): us per round, per-round algorithmic bytes 4 d_pad (3r + 3) and the
effective rate.  Measurement only (scripts/README.md)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sma_inputs  # noqa: E402
from paper_1901_02244_b200 import sma  # noqa: E402

torch.cuda.set_device(0)
steps = int(os.environ.get("PROBE_STEPS", "5000"))
cases = [(512, 8), (4096, 8), (32768, 8), (131072, 8), (262144, 8), (431_080, 8),
         (464_154, 16), (431_080, 1), (1_000_003, 8)]
for d, k in cases:
    alpha = float(np.float32(1 / k))
    h = sma.Sma(d, k, alpha, 0.1, 0.9, sma_inputs.w0(d), device=0, flags=0)
    s = torch.cuda.Stream()
    h.synth_grads(0, sma_inputs.SEED_G, s)
    for _ in range(200):
        h.step(s)
    s.synchronize()
    best = None
    host_us = None
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        t0 = time.perf_counter()
        for _ in range(steps):
            h.step(s)
        th = (time.perf_counter() - t0) * 1e6 / steps   # host enqueue time per sma_step
        e1.record(s)
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / steps
        if best is None or us < best:
            best, host_us = us, th
    # the same rounds replayed from a CUDA graph of 100 captured sma_step calls
    # (no host work between rounds): is the floor the host or the GPU?
    graph_us = None
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cs = torch.cuda.current_stream()
            for _ in range(100):
                h.step(cs)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cs = torch.cuda.current_stream()
        e0.record(cs)
        for _ in range(steps // 100):
            g.replay()
        e1.record(cs)
        e1.synchronize()
        graph_us = e0.elapsed_time(e1) * 1e3 / (100 * (steps // 100))
    except Exception as ex:  # noqa: BLE001
        graph_us = f"capture failed: {ex}"[:200]
    dp = h.d_pad
    b = 4 * dp * (3 * k + 3)
    print(json.dumps({"d": d, "k": k, "d_pad": dp, "us_per_round": best, "host_enqueue_us": host_us, "graph100_us_per_round": graph_us, "bytes": b,
                      "eff_tbs": b / (best * 1e-6) / 1e12,
                      "env": {x: os.environ[x] for x in os.environ if x.startswith("SMA_")}}),
          flush=True)
    h.close()
