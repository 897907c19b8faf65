"""Subprocess worker for the MLP tensor-core tests (the SMA_MLP_TC policy is
read once per process): computes one learner-gradient round through libsma
and saves every replica's gradient (w0 - w', gamma = 1, alpha = mu = 0).
Usage: python mlp_grad_worker.py OUT.npy K B ROUND SEED"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import sma_inputs
    from paper_1901_02244_b200 import sma
    out, k, b, rnd, seed = sys.argv[1], *map(int, sys.argv[2:6])
    d = 256 * 784 + 256 + 10 * 256 + 10
    X, y = sma_inputs.blobs(2_000, seed=12)
    w0 = np.random.default_rng(seed).normal(0, 0.05, d).astype(np.float32)
    h = sma.Sma(d, k, 0.0, 1.0, 0.0, w0)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    sma.sma_learner_attach(h.h, 1, 784, 256, 10, b, Xd, yd, X.shape[0], 21)
    sma.sma_learner_grads(h.h, rnd, torch.cuda.current_stream())
    h.step()
    np.save(out, np.stack([w0.astype(np.float64) - h.replica(j) for j in range(k)]))
    h.close()


if __name__ == "__main__":
    main()
