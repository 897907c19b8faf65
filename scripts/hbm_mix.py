"""Achievable HBM bandwidth on this B200 for the replica kernel's traffic mix.

The roofline denominator (MEASURED_PEAKS.json hbm_gbs) is a 1:1 read:write copy.
The fused SMA round reads ~2 bytes per byte written (w, g, z, z_prev in; w, z'
out).  This measures torch's own streaming kernels on >L2-sized tensors:
copy (1:1), add a+b->c (2:1 triad), a.sum() (read only), fill (write only),
best of N with CUDA events.  Context for DESIGN.md, not a bench metric."""
import json
import torch

n = 1 << 28          # 256 Mi floats = 1 GiB per tensor
a = torch.rand(n, device="cuda")
b = torch.rand(n, device="cuda")
c = torch.empty(n, device="cuda")
def t(fn, nbytes, reps=10):
    best = 1e9
    for _ in range(3):
        fn()
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / (best * 1e-3) / 1e9
res = {
    "copy_1r1w_GBs": t(lambda: c.copy_(a), 8 * n),
    "triad_2r1w_GBs": t(lambda: torch.add(a, b, out=c), 12 * n),
    "read_only_GBs": t(lambda: a.sum(), 4 * n),
    "write_only_GBs": t(lambda: c.fill_(1.0), 4 * n),
}
print(json.dumps(res))
