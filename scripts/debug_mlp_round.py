"""Debug: run the MLP bench configuration (k learners) for R rounds through
sma_learner_step, then check round R against the oracle from the GPU's state
and report the worst gradient elements (which learner, which parameter block,
and for W1 / b1 the pre-activations of that unit on the learner's batch).
Usage: python scripts/debug_mlp_round.py K R"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


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
    z = h.central().astype(np.float64)
    sma.sma_learner_step(h.h, R, s)
    s.synchronize()
    W1 = 256 * 784
    worst = []
    for j in range(k):
        rows = oracle.batch_indices(60_000, k, 16, 99, R, j)
        _, G, mg = oracle.mlp_loss_grad(X, y, rows, Wg[j])
        wn = h.replica(j).astype(np.float64)
        gg = (Wg[j] - a * (Wg[j] - z) - wn) / g
        err = np.abs(gg - G)
        p = int(np.argmax(err))
        worst.append((err[p], j, p, gg[p], G[p], mg))
    worst.sort(reverse=True)
    for e, j, p, gv, gr, mg in worst[:4]:
        if p < W1:
            u, f = divmod(p, 784)
            where = f"W1[{u}][{f}]"
        elif p < W1 + 256:
            u = p - W1
            where = f"b1[{u}]"
        else:
            u = None
            where = f"head+{p - W1 - 256}"
        print(f"learner {j} err {e:.3e} at {where}: gpu {gv:.9g} oracle {gr:.9g} (oracle margin {mg:.3e})")
        if u is not None:
            rows = oracle.batch_indices(60_000, k, 16, 99, R, j)
            xr = X[rows].astype(np.float64)
            av = Wg[j][u * 784:(u + 1) * 784] @ xr.T + Wg[j][W1 + u]
            print("   a[t][u] =", " ".join(f"{v:.3e}" for v in av))
    h.close()


if __name__ == "__main__":
    main()
