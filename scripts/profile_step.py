#!/usr/bin/env python
"""Small driver for ncu captures: builds the bench workload (ERNIE-M-base, LOOPBACK P=2,
25 MiB buckets) and runs a few nebula_step(ALL) calls.  Exits 0 on success; run it plain
first, then under ncu (B200_PROFILING.md)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--method", default="int8", choices=["identity", "fp16", "int8", "topk", "fp8", "qsgd", "fp8e5m2"])
    ap.add_argument("--no-ef", action="store_true")
    ap.add_argument("--int8-kernel", default="auto")
    ap.add_argument("--values", default="f32", choices=["f32", "f16", "i8"])
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--workload", default="ernie-m-base")
    args = ap.parse_args()
    import torch
    import paper_2205_09470_b200 as nb
    from gradgen import fixed_buckets, model_gradient
    P = 2
    host = [model_gradient(args.workload, cluster=c) for c in range(P)]
    n = host[0].size
    g = torch.empty(P * n, device="cuda")
    for c in range(P):
        g[c * n:(c + 1) * n].copy_(torch.from_numpy(host[c]))
    out = torch.empty(n, device="cuda")
    m = {"identity": 0, "fp16": 1, "int8": 2, "topk": 3, "fp8": 4, "qsgd": 6, "fp8e5m2": 7}[args.method]
    ctx = nb.SyncContext(fixed_buckets(n, 25 << 20), m, topk_values={"f32": 0, "f16": 1, "i8": 2}[args.values],
                         topk_density=args.density, num_clusters=P, transport=nb.LOOPBACK,
                         error_feedback=not args.no_ef)
    if m == 2:
        ctx.set_int8_kernel(args.int8_kernel)
    for s in range(args.steps):
        ctx.step(nb.ALL_BUCKETS, g, out, s)
    ctx.check()
    torch.cuda.synchronize()
    ctx.destroy()
    print("profile_step OK")


if __name__ == "__main__":
    main()
