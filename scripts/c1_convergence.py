"""C1 end to end (SURVEY §8d "C1 ... report rounds/s and end-to-end convergence"):
SMA with the built-in softmax learner in the loop (k = 4, b = 16, alpha = 1/4,
gamma = 0.1, mu = 0.9, w0 = 0) on the MNIST-shaped synthetic blobs, the rounds
of one epoch through sma_learner_steps (the softmax cluster kernel), in chunks
of 25 rounds.  After each chunk, the central model z is read through the C ABI
and its mean cross-entropy and accuracy are evaluated on a held-out set drawn
from the same blobs (evaluation only, outside the timed chunks).  Prints one
JSON line per checkpoint and a summary line.  Measurement only (scripts/README.md)."""
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
k, b, chunk = 4, 16, 25
alpha, gamma, mu = float(np.float32(1 / k)), float(np.float32(0.1)), float(np.float32(0.9))
Xall, yall = sma_inputs.blobs(70_000, seed=4)
X, y = Xall[:60_000], yall[:60_000]
Xt, yt = torch.from_numpy(Xall[60_000:]).cuda(), torch.from_numpy(yall[60_000:]).cuda().long()
d = 10 * 785
h = sma.Sma(d, k, alpha, gamma, mu, np.zeros(d, np.float32), device=0)
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
sma.sma_learner_attach(h.h, 0, 784, 0, 10, b, Xd, yd, X.shape[0], 99)
E = X.shape[0] // (k * b)
s = torch.cuda.Stream()


def evaluate():
    z = torch.from_numpy(h.central()).cuda()
    logits = Xt @ z[:7840].view(10, 784).T + z[7840:]
    loss = torch.nn.functional.cross_entropy(logits, yt).item()
    acc = (logits.argmax(1) == yt).float().mean().item()
    return loss, acc


loss0, acc0 = evaluate()
print(json.dumps({"round": 0, "loss": loss0, "acc": acc0, "gpu_ms": 0.0}), flush=True)
gpu_ms, rnd, first99 = 0.0, 0, None
while rnd < E:
    n = min(chunk, E - rnd)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    sma.sma_learner_steps(h.h, rnd, n, s)
    e1.record(s)
    e1.synchronize()
    gpu_ms += e0.elapsed_time(e1)
    rnd += n
    loss, acc = evaluate()
    if first99 is None and acc >= 0.99:
        first99 = {"round": rnd, "gpu_ms": gpu_ms}
    print(json.dumps({"round": rnd, "loss": loss, "acc": acc, "gpu_ms": gpu_ms}), flush=True)
print(json.dumps({"summary": "C1 end to end, one epoch", "rounds": rnd, "gpu_ms": gpu_ms,
                  "rounds_per_s_incl_chunk_launches": rnd / (gpu_ms * 1e-3),
                  "first_heldout_acc_ge_0.99": first99, "final_loss": loss, "final_acc": acc,
                  "config": {"k": k, "b": b, "alpha": alpha, "gamma": gamma, "mu": mu,
                             "chunk": chunk, "train": 60_000, "heldout": 10_000}}), flush=True)
h.close()
