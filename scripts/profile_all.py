#!/usr/bin/env python
"""ncu driver: one nebula_step(ALL) of every default codec kernel at the bench workload
(ERNIE-M-base, 278,042,880 fp32 per cluster, 25 MiB buckets, LOOPBACK P = 2), plus the P2P
kernels through the SELF transport (pull reducer reading a peer's slots, the arrival-flag
kernel, the intra-cluster hop at G = 2) on a 25 MiB x 4 gradient.  Run it plain first, then
under `ncu --set full -k regex:...` (B200_PROFILING.md).  Prints PROFILE_ALL OK."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="", help="comma list of case names")
    args = ap.parse_args()
    import torch
    import paper_2205_09470_b200 as nb
    from gradgen import fixed_buckets, model_gradient

    P = 2
    # the bench's per-launch shape on a shorter gradient: 8 buckets of 25 MiB per cluster (ncu
    # replays each kernel ~40 times, saving and restoring its working set every time)
    n = 8 * ((25 << 20) // 4)
    host = [model_gradient("ernie-m-base", cluster=c)[:n].copy() for c in range(P)]
    g = torch.empty(P * n, device="cuda")
    for c in range(P):
        g[c * n:(c + 1) * n].copy_(torch.from_numpy(host[c]))
    del host
    out = torch.empty(n, device="cuda")
    sizes = fixed_buckets(n, 25 << 20)
    cases = {
        "fp16_step": (nb.FP16, {}, None),
        "fp16_staged": (nb.FP16, {}, "staged"),
        "identity": (nb.IDENTITY, {}, None),
        "fp8": (nb.FP8, {}, None),
        "e5m2": (nb.FP8_E5M2, {}, None),
        "qsgd": (nb.QSGD, {}, None),
        "int8_pull_split": (nb.INT8, {}, "pull-split"),
    }
    only = set(args.only.split(",")) if args.only else None
    for name, (m, kw, mode) in cases.items():
        if only and name not in only:
            continue
        ctx = nb.SyncContext(sizes, m, num_clusters=P, transport=nb.LOOPBACK, **kw)
        if mode == "staged":
            ctx.set_step_fusion(False)
        if mode == "pull-split":
            ctx.set_option(nb.OPT_STEP_FUSION, 2 + 4)
        for s in range(2):
            ctx.step(nb.ALL_BUCKETS, g, out, s)
        ctx.check()
        ctx.destroy()
    del g, out
    torch.cuda.empty_cache()
    if not only or "self" in only:
        m = 4 * (25 << 20) // 4
        for (PP, G, xch) in ((2, 1, "pull"), (1, 2, "auto")):
            grid = nb.self_group([m // 4 * G] * 4, num_clusters=PP, gpus_per_cluster=G, device=0, method=nb.INT8)
            gd = [[torch.randn(m * G, device="cuda") for _ in range(G)] for _ in range(PP)]
            od = [[torch.empty(m * G, device="cuda") for _ in range(G)] for _ in range(PP)]
            for row in grid:
                for ctx in row:
                    ctx.set_int8_kernel("two-pass")
                    if PP > 1:
                        ctx.set_exchange(xch)
            torch.cuda.synchronize()
            for s in range(2):
                for c in range(PP):
                    for l in range(G):
                        grid[c][l].compress(nb.ALL_BUCKETS, gd[c][l], s)
                for row in grid:
                    for ctx in row:
                        ctx.stream.synchronize()
                for c in range(PP):
                    for l in range(G):
                        grid[c][l].exchange(nb.ALL_BUCKETS)
                for c in range(PP):
                    for l in range(G):
                        grid[c][l].decompress_reduce(nb.ALL_BUCKETS, od[c][l])
                for row in grid:
                    for ctx in row:
                        ctx.stream.synchronize()
            for row in grid:
                for ctx in row:
                    ctx.check()
                    ctx.destroy()
    torch.cuda.synchronize()
    print("PROFILE_ALL OK", flush=True)


if __name__ == "__main__":
    main()
