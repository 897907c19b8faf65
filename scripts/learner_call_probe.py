"""Host enqueue time of one sma_learner_step call vs the GPU time per round
(C1 softmax learner, k = 4, b = 16; MLP k = 4): is the one-call-per-round mode
host-bound?  Measurement only (scripts/README.md)."""
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
X, y = sma_inputs.blobs(60_000, seed=4)
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
for kind, hidden, d in ((0, 0, 7850), (1, 256, 256 * 785 + 10 * 256 + 10)):
    h = sma.Sma(d, 4, 0.25, 0.1, 0.9, np.random.default_rng(6).normal(0, 0.05 if kind else 0.0, d)
                .astype(np.float32), device=0)
    sma.sma_learner_attach(h.h, kind, 784, hidden, 10, 16, Xd, yd, X.shape[0], 99)
    s = torch.cuda.Stream()
    for i in range(100):
        sma.sma_learner_step(h.h, i, s)
    s.synchronize()
    n = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    for i in range(100, 100 + n):
        sma.sma_learner_step(h.h, i, s)
    th = (time.perf_counter() - t0) * 1e6 / n
    e1.record(s)
    e1.synchronize()
    print(json.dumps({"learner": "softmax" if kind == 0 else "mlp", "k": 4,
                      "host_enqueue_us_per_call": th, "gpu_us_per_round": e0.elapsed_time(e1) * 1e3 / n}),
          flush=True)
    h.close()
