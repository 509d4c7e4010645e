#!/usr/bin/env python
"""Direction-split HBM bandwidth on this GPU (torch kernels, CUDA events, best of 10): write-only
(fill_), read-only (sum), copy (read + write).  Grounds the roofline of the write-dominated
reducers: the MEASURED_PEAKS copy figure counts read + write bytes."""
import json

import torch


def timed(fn, iters=10):
    best = 1e9
    for _ in range(iters + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    n = 278042880                       # one ERNIE-M-base cluster gradient, fp32 (1.11 GB)
    x = torch.empty(n, device="cuda")
    y = torch.empty(n, device="cuda")
    x.normal_()
    w = timed(lambda: y.fill_(0.5))
    r = timed(lambda: x.sum())
    c = timed(lambda: y.copy_(x))
    gb = 4.0 * n / 1e9
    print(json.dumps({"bytes": 4 * n, "write_only_gbs": round(gb / w * 1e3, 1), "read_only_gbs": round(gb / r * 1e3, 1),
                      "copy_rw_gbs": round(2 * gb / c * 1e3, 1), "ms": {"write": w, "read": r, "copy": c}}))


if __name__ == "__main__":
    main()
