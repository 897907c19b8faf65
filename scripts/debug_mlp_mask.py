"""Debug: after R rounds of the MLP bench configuration (k learners), recover
every learner's gradient of round R from the GPU (alpha = 0, gamma = 1, mu = 0
for that round: w' = w - g) and compare the W1 rows of the worst learner with a
numpy fp64 gradient computed with the oracle's mask and with single mask
entries flipped.  Usage: python scripts/debug_mlp_mask.py K R"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def np_grad(X, y, rows, p, mask_override=None):
    W1 = p[:256 * 784].reshape(256, 784); b1 = p[256 * 784:256 * 785]
    o = 256 * 785
    W2 = p[o:o + 2560].reshape(10, 256); b2 = p[o + 2560:o + 2570]
    x = X[rows].astype(np.float64)
    a1 = x @ W1.T + b1
    m = a1 > 0
    if mask_override is not None:
        for (t, u) in mask_override:
            m[t, u] = ~m[t, u]
    h = np.where(m, a1, 0.0)
    lg = h @ W2.T + b2
    lg -= lg.max(1, keepdims=True)
    P = np.exp(lg); P /= P.sum(1, keepdims=True)
    e = P.copy(); e[np.arange(len(rows)), y[rows]] -= 1
    b = len(rows)
    da = (e @ W2) * m
    return (da.T @ x) / b, a1


def main():
    import torch

    import oracle
    import sma_inputs
    from paper_1901_02244_b200 import sma
    k, R = int(sys.argv[1]), int(sys.argv[2])
    D = 256 * 784 + 256 + 10 * 256 + 10
    X, y = sma_inputs.blobs(60_000, seed=4)
    w0 = np.random.default_rng(6).normal(0, 0.05, D).astype(np.float32)
    F = lambda x: float(np.float32(x))  # noqa: E731
    a, g, m = F(1 / k), F(0.1), F(0.9)
    h = sma.Sma(D, k, a, g, m, w0)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    sma.sma_learner_attach(h.h, 1, 784, 256, 10, 16, Xd, yd, X.shape[0], 99)
    s = torch.cuda.Stream()
    for i in range(R):
        sma.sma_learner_step(h.h, i, s)
    s.synchronize()
    Wg = np.stack([h.replica(j) for j in range(k)]).astype(np.float64)
    sma.sma_set_hparams(h.h, 0.0, 1.0, 0.0)
    sma.sma_learner_step(h.h, R, s)
    s.synchronize()
    for j in range(k):
        gg = Wg[j] - h.replica(j).astype(np.float64)
        rows = oracle.batch_indices(60_000, k, 16, 99, R, j)
        G1, a1 = np_grad(X, y, rows, Wg[j])
        err = np.abs(gg[:256 * 784].reshape(256, 784) - G1)
        u = int(np.argmax(err.max(1)))
        if err.max() < 1e-6:
            continue
        print(f"learner {j}: worst W1 row {u}: max err {err[u].max():.3e}")
        near = np.argwhere(np.abs(a1) < 1e-3)
        print("   near-kink (t,u,a1):", [(int(t), int(uu), float(a1[t, uu])) for t, uu in near])
        for t, uu in near:
            Gf, _ = np_grad(X, y, rows, Wg[j], [(t, uu)])
            ef = np.abs(gg[:256 * 784].reshape(256, 784) - Gf).max()
            print(f"   flip ({t},{uu}) -> max err {ef:.3e}")
    h.close()


if __name__ == "__main__":
    main()
