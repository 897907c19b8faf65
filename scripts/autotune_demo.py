"""NEXT-4 end to end (the analog of the paper's fig:auto-tuning):
Alg. 2 (sma_autotune_step) driven by the measured learning throughput
(learner batches/s = k x rounds/s, "the rate at which learning tasks
complete") resizes the learners on the GPU between adaptation
periods (sma_set_local_replicas; added learners start from z, P:985-986;
alpha := 1/k).  Prints one JSON line per period."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sma_inputs  # noqa: E402
from paper_1901_02244_b200 import sma  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "C1"
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 2000.0
periods = int(sys.argv[3]) if len(sys.argv) > 3 else 24
rounds = 200
cfg = sma_inputs.CONFIGS[kind]
d, b = cfg["d"], cfg["batch"]
X, y = sma_inputs.blobs(60_000, seed=4)
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
w0 = np.random.default_rng(6).normal(0, 0.05 if kind == "MLP" else 0.0, d).astype(np.float32)
l, t_prev = np.array([1], np.int32), np.array([0.0])           # Alg. 2 lines 1-2
h = sma.Sma(d, 1, 1.0, 0.1, 0.9, w0)
sma.sma_learner_attach(h.h, 0 if kind == "C1" else 1, 784, 256 if kind == "MLP" else 0, 10, b,
                       Xd, yd, X.shape[0], 99)
s = torch.cuda.Stream()
rnd = 0
for period in range(periods):
    if l[0] < 1:
        l[0] = 1
    if l[0] != h.local_count:
        h.set_local_replicas(int(l[0]), s)
        h.set_hparams(1.0 / float(l[0]), 0.1, 0.9)
    for _ in range(20):  # warm-up of this configuration
        sma.sma_learner_step(h.h, rnd, s)
        rnd += 1
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(rounds):
        sma.sma_learner_step(h.h, rnd, s)
        rnd += 1
    e1.record(s)
    torch.cuda.synchronize()
    rps = rounds / (e0.elapsed_time(e1) * 1e-3)
    t = np.array([rps * h.local_count])                          # learner batches/s
    l_before = int(l[0])
    l, t_prev = sma.sma_autotune_step(tau, t, l, t_prev)        # Alg. 2 lines 4-9
    print(json.dumps({"learner": kind, "period": period, "learners": l_before,
                      "rounds_per_s": rps, "batches_per_s": float(t[0]), "tau": tau,
                      "next_learners": int(l[0])}), flush=True)
z = h.central()
acc = float(np.mean(np.argmax(X @ z[:7840].reshape(10, 784).T + z[7840:], 1) == y)) \
    if kind == "C1" else None
print(json.dumps({"learner": kind, "final_learners": h.local_count, "train_accuracy": acc}))
h.close()
