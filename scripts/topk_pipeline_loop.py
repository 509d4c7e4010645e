#!/usr/bin/env python
"""Bench-like TOPK loop (no synchronisation between steps) at config-2 size; reports
whether the device faulted.  argv: rho steps pipeline(0/1)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2205_09470_b200 as nb
    from gradgen import fixed_buckets, model_gradient
    P = 2
    rho, steps, pipe = float(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    host = [model_gradient("ernie-m-base", cluster=c) for c in range(P)]
    n = host[0].size
    g = torch.empty(P * n, device="cuda")
    for c in range(P):
        g[c * n:(c + 1) * n].copy_(torch.from_numpy(host[c]))
    ctx = nb.SyncContext(fixed_buckets(n, 25 << 20), 3, topk_density=rho, num_clusters=P, transport=nb.LOOPBACK)
    ctx.set_option(nb.OPT_PIPELINE, pipe)
    out = torch.empty(n, device="cuda")
    try:
        for s in range(steps):
            ctx.step(nb.ALL_BUCKETS, g, out, s)
        ctx.check()
        torch.cuda.synchronize()
        print("LOOP OK", flush=True)
    except Exception as e:
        print("LOOP FAILED", repr(e)[:200], flush=True)


if __name__ == "__main__":
    main()
