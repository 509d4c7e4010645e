#!/usr/bin/env python
"""Small workload that launches every default kernel of the library once or twice, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck; one tool per run):

  LOOPBACK P = 2 and 3: INT8 / FP8 E4M3 / FP8 E5M2 / QSGD through the single-pass warp-specialised
  kernel (forced on small buckets), the fused step (TMA reduce role and the P2P-pull register
  reduce role), the two-pass kernels; FP16 (TMA ring and plain); IDENTITY; TOP-K f32 / f16 / i8
  (sample, bracket, stage, scan, move, resolve, merge, densify); the single-slot decode.
  SELF transport (every cross-GPU path on one GPU): P2P push and pull exchange with arrival
  flags (P = 2), the G = 2 intra-cluster hop (push reduce-scatter, fixed-order reduce, all-gather
  pull, exact-scale mailbox) and the exact cluster-wide top-k.

Checks every result against the oracle so a sanitizer-induced change would also show.  Exits 0
and prints SANITIZE WORKLOAD OK."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-self", action="store_true", help="skip the SELF-transport part (tools that serialise streams)")
    ap.add_argument("--small", action="store_true", help="smaller buckets (racecheck)")
    args = ap.parse_args()
    import torch
    import oracle as O
    import paper_2205_09470_b200 as nb
    from gradgen import seed_for, synthetic

    nb.load()
    sizes = [8192, 4100, 1028] if args.small else [40000, 16388, 4100]   # 16-B aligned: the single-pass paths run
    F = np.float32

    def loopback(method, P, vt=0, kern=None, fusion=None, fp16=None, steps=2, rho=0.05):
        ctx = nb.SyncContext(sizes, method, topk_values=vt, topk_density=rho, num_clusters=P, transport=nb.LOOPBACK)
        if kern:
            ctx.set_int8_kernel(kern)
        if fusion is not None:
            ctx.set_option(nb.OPT_STEP_FUSION, fusion)
        if fp16:
            ctx.set_fp16_kernel(fp16)
        codec = O.Codec(method=method, topk_values=vt, topk_density=rho)
        rs = [[np.zeros(n, F) for n in sizes] for _ in range(P)]
        for t in range(steps):
            gs = [[synthetic(n, seed_for(c, 0, t, salt=b), "model-like") for b, n in enumerate(sizes)] for c in range(P)]
            dev = torch.from_numpy(np.concatenate([np.concatenate(x) for x in gs])).cuda()
            out = torch.empty(sum(sizes), device="cuda")
            ctx.step(nb.ALL_BUCKETS, dev, out, t)
            ctx.check()
            got = out.cpu().numpy()
            off = 0
            for b, n in enumerate(sizes):
                exp, r_new, _, _ = O.oracle_step([gs[c][b] for c in range(P)], [rs[c][b] for c in range(P)], codec, t,
                                                 bucket=b)
                assert np.array_equal(got[off:off + n].view(np.uint32), exp.view(np.uint32)), (method, P, kern, b)
                for c in range(P):
                    rs[c][b] = r_new[c] if r_new[c] is not None else rs[c][b]
                off += n
        dec = torch.empty(sizes[0], device="cuda")
        ctx.compress(nb.ALL_BUCKETS, dev, steps)   # the staged calls and the single-slot decode
        ctx.exchange(nb.ALL_BUCKETS)
        ctx.decompress(0, 0, dec)
        ctx.decompress_reduce(nb.ALL_BUCKETS, out)
        ctx.check()
        ctx.destroy()

    for m in (O.INT8, O.FP8, O.FP8_E5M2, O.QSGD):
        loopback(m, 2, kern="single-pass", fusion=1)          # single-pass compress + dense reduce
        loopback(m, 2, kern="single-pass")                    # fused step, TMA reduce role
        loopback(m, 3, kern="single-pass", fusion=2 + 4)      # fused step, P2P-pull register reduce role
        loopback(m, 2, kern="two-pass")
    loopback(O.FP16, 2)
    loopback(O.FP16, 2, fp16="plain")
    loopback(O.IDENTITY, 2)
    for vt in (O.VAL_F32, O.VAL_F16, O.VAL_I8):
        loopback(O.TOPK, 2, vt=vt)

    # SELF transport: P2P exchange, flags, intra-cluster hop
    def self_run(method, P, G, exchange="auto", exact=False, exact_topk=False):
        grid = nb.self_group([s * G for s in sizes], num_clusters=P, gpus_per_cluster=G, device=0, method=method,
                             topk_density=0.05, exact_topk=exact_topk)
        for row in grid:
            for ctx in row:
                if method in (O.INT8, O.FP8, O.QSGD, O.FP8_E5M2):
                    ctx.set_int8_kernel("two-pass")
                if P > 1:
                    ctx.set_exchange(exchange)
                if exact:
                    ctx.set_exact_scale(True)
        n = sum(sizes) * G
        for t in range(2):
            gd = [[torch.from_numpy(synthetic(n, seed_for(c, l, t), "model-like")).cuda() for l in range(G)]
                  for c in range(P)]
            outs = [[torch.empty(n, device="cuda") for _ in range(G)] for _ in range(P)]
            torch.cuda.synchronize()
            for c in range(P):
                for l in range(G):
                    grid[c][l].compress(nb.ALL_BUCKETS, gd[c][l], t)
            for row in grid:
                for ctx in row:
                    ctx.stream.synchronize()
            for c in range(P):
                for l in range(G):
                    grid[c][l].exchange(nb.ALL_BUCKETS)
            for c in range(P):
                for l in range(G):
                    grid[c][l].decompress_reduce(nb.ALL_BUCKETS, outs[c][l])
            for row in grid:
                for ctx in row:
                    ctx.stream.synchronize()
                    ctx.check()
            ref = outs[0][0].cpu().numpy().view(np.uint32)
            for c in range(P):
                for l in range(G):
                    assert np.array_equal(outs[c][l].cpu().numpy().view(np.uint32), ref)
        for row in grid:
            for ctx in row:
                ctx.destroy()

    if args.no_self:
        torch.cuda.synchronize()
        print("SANITIZE WORKLOAD OK (no SELF)", flush=True)
        return
    self_run(O.INT8, 2, 1, "push")
    self_run(O.INT8, 2, 1, "pull")
    self_run(O.FP16, 2, 1, "push")
    self_run(O.TOPK, 2, 1, "pull")
    self_run(O.INT8, 2, 2, "pull")
    self_run(O.INT8, 1, 2, exact=True)
    self_run(O.TOPK, 2, 2, "pull", exact_topk=True)
    torch.cuda.synchronize()
    print("SANITIZE WORKLOAD OK", flush=True)


if __name__ == "__main__":
    main()
