"""Measured L2-resident streaming bandwidth on the GPU (the denominator of the
small configs' roofline, whose per-round working set fits the 126 MB L2):
torch's own copy (1 read : 1 write) and add (2 reads : 1 write) kernels over
buffers that stay L2-resident, timed with CUDA events over 500 back-to-back
launches after warm-up.  Prints one JSON object.  Usage: python scripts/l2_peak.py"""
import json

import torch


def bench(fn, nbytes, iters=500):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return nbytes / (ms * 1e-3) / 1e9, ms


def main():
    out = {"device": torch.cuda.get_device_name(0),
           "l2_bytes": torch.cuda.get_device_properties(0).L2_cache_size, "runs": []}
    for mb in (4, 8, 16, 24, 32):
        n = mb * (1 << 20) // 4
        a = torch.randn(n, device="cuda")
        b = torch.randn(n, device="cuda")
        c = torch.empty(n, device="cuda")
        gbs_copy, ms_copy = bench(lambda: c.copy_(a), 2 * 4 * n)
        gbs_add, ms_add = bench(lambda: torch.add(a, b, out=c), 3 * 4 * n)
        out["runs"].append({"mb_per_buffer": mb, "copy_gbs": gbs_copy, "copy_ms": ms_copy,
                            "add_gbs": gbs_add, "add_ms": ms_add})
    out["copy_gbs_max"] = max(r["copy_gbs"] for r in out["runs"])
    out["add_gbs_max"] = max(r["add_gbs"] for r in out["runs"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
