#!/usr/bin/env python
"""Distributed parity check (run under torchrun, one process per GPU, NCCL transport).

Every rank is one GPU of cluster rank // G.  Each step every rank regenerates ALL ranks'
seeded gradients on the host (gradgen), runs the C-ABI step on its own, and checks:
  * its output is bit-identical to the oracle (flat P x 1: oracle_step; G > 1:
    hierarchical_step — on model-like (non-dyadic) inputs when the intra-cluster hop is the
    fixed-order P2P reduce-scatter, on dyadic inputs (mean exact in any order) for the NCCL
    ReduceScatter(avg) fallback, whose summation order is NCCL's),
  * its own payload slot and residual are bit-identical to the oracle's,
  * all ranks' outputs are bit-identical (all-gathered and compared on every rank).
Prints "DIST OK ..." on rank 0 and exits 0, else raises.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def dyadic(n, seed):
    rng = np.random.default_rng(seed)
    return (rng.integers(-4096, 4096, n).astype(np.float32) * np.float32(2.0 ** -14)).astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus-per-cluster", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import oracle as O
    import paper_2205_09470_b200 as nb
    from gradgen import seed_for, synthetic

    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    G = args.gpus_per_cluster
    P, cl, lr = nb.topology_for_rank(rank, world, G)
    sizes = [4096 * G, 12288 * G, 300004 * G, 8 * G]
    total = sum(sizes)
    # (method, top-k values, INT8 kernel, exact cluster-wide scale (NEXT-3, only meaningful for G > 1),
    #  intra-cluster hop for G > 1: "p2p" (auto) or "nccl")
    cases = [(O.INT8, 0, "two-pass", False, "p2p"), (O.INT8, 0, "fused-ws", False, "p2p"),
             (O.FP16, 0, None, False, "p2p"), (O.IDENTITY, 0, None, False, "p2p"), (O.FP8, 0, None, False, "p2p"),
             (O.QSGD, 0, None, False, "p2p"), (O.TOPK, O.VAL_F32, None, False, "p2p"),
             (O.TOPK, O.VAL_I8, None, False, "p2p"), (O.TOPK, O.VAL_F16, None, False, "p2p"),
             (O.FP8, 0, "fused-ws", False, "p2p"), (O.QSGD, 0, "fused-ws", False, "p2p")]   # fused step over P2P (G = 1)
    if G > 1:
        cases += [(O.TOPK, O.VAL_F32, None, "exact-topk", "p2p"), (O.TOPK, O.VAL_I8, None, "exact-topk", "nccl"),
                  (O.INT8, 0, None, True, "p2p"), (O.FP8, 0, None, True, "p2p"), (O.INT8, 0, None, False, "nccl"),
                  (O.TOPK, O.VAL_F32, None, False, "nccl"), (O.INT8, 0, None, True, "nccl"),
                  # the two-stream ALL-bucket step over the P2P intra hop (NEBULA_OPT_PIPELINE = 2)
                  (O.INT8, 0, "pipeline2", False, "p2p"), (O.TOPK, O.VAL_F32, "pipeline2", False, "p2p"),
                  (O.FP16, 0, "pipeline2", False, "p2p")]
    intra_seen = set()
    modes_seen = set()
    modes = ((False, "pull"), (True, "pull"), (False, "push"), (True, "push"), (False, "nccl"))
    for ci, (method, vt, kern, exact, intra) in enumerate(cases):
        # INT8 (the default codec) runs every (call shape, exchange) mode; the other cases rotate
        # through two modes each, so every mode is still met by several codecs at a fraction of
        # the oracle time (each rank recomputes every cluster's oracle step)
        sel_modes = modes if ci == 0 else (modes[ci % len(modes)], modes[(ci + 2) % len(modes)])
        for per_bucket, xch in sel_modes:
            xtopk = exact == "exact-topk"
            ctx = nb.init_process_group_context(sizes, gpus_per_cluster=G, device=local, method=method,
                                                topk_values=vt, topk_density=0.05, exact_topk=xtopk)
            exact = exact is True
            if kern == "pipeline2":
                ctx.set_option(nb.OPT_PIPELINE, 2)
            elif kern:
                ctx.set_int8_kernel(kern)
            if exact:
                ctx.set_exact_scale(True)
            if G > 1:
                ctx.set_intra(intra)
            exact_order = ctx.intra_mode() != "nccl"   # fixed-order P2P mean: any input is exact
            intra_seen.add(ctx.intra_mode())
            if P > 1:
                try:
                    ctx.set_exchange(xch)
                except nb.NebulaError:
                    assert xch in ("pull", "push")
                    ctx.set_exchange("nccl")
            modes_seen.add(ctx.exchange_mode())
            codec = O.Codec(method=method, topk_values=vt, topk_density=0.05)
            m = [s if xtopk else s // G for s in sizes]
            rs = [[[np.zeros(mb, np.float32) for mb in m] for _ in range(G)] for _ in range(P)]
            for t in range(args.steps):
                # gradient of (cluster c, gpu l, bucket b)
                def grad(c, l, b):
                    if G > 1 and not exact_order:
                        return dyadic(sizes[b], seed_for(c, l, t, salt=b))
                    return synthetic(sizes[b], seed_for(c, l, t, salt=b), "model-like")
                mine = np.concatenate([grad(cl, lr, b) for b in range(len(sizes))])
                g = torch.from_numpy(mine).cuda()
                out = torch.full((total,), float("nan"), device="cuda")
                if per_bucket:
                    off = 0
                    for b, n in enumerate(sizes):
                        ctx.step(b, g[off:off + n], out[off:off + n], t)
                        off += n
                else:
                    ctx.step(nb.ALL_BUCKETS, g, out, t)
                ctx.check()
                got = out.cpu().numpy()
                # cross-rank identity
                allo = [torch.empty_like(out) for _ in range(world)]
                dist.all_gather(allo, out)
                for o in allo:
                    assert torch.equal(o.view(torch.int32), out.view(torch.int32)), "ranks disagree"
                off = 0
                for b, n in enumerate(sizes):
                    if G == 1:
                        exp, r_new, payloads, _ = O.oracle_step([grad(c, 0, b) for c in range(P)],
                                                                [rs[c][0][b] for c in range(P)], codec, t, bucket=b)
                        myr, mypl = r_new[cl], payloads[cl]
                        for c in range(P):
                            rs[c][0][b] = r_new[c] if r_new[c] is not None else rs[c][0][b]
                    else:
                        exp, r_new, pls = O.hierarchical_step([[grad(c, l, b) for l in range(G)] for c in range(P)],
                                                              [[rs[c][l][b] for l in range(G)] for c in range(P)],
                                                              codec, t, exact_scale=exact, bucket=b,
                                                              exact_topk=xtopk)
                        myr, mypl = r_new[cl][lr], pls[cl][lr]
                        for c in range(P):
                            for l in range(G):
                                rs[c][l][b] = r_new[c][l] if r_new[c][l] is not None else rs[c][l][b]
                    assert np.array_equal(got[off:off + n].view(np.uint32), exp.view(np.uint32)), \
                        f"rank {rank} out mismatch method {method} vt {vt} bucket {b} step {t}"
                    assert ctx.payload_copy(b, cl) == mypl, f"rank {rank} payload mismatch b{b} t{t}"
                    if myr is not None:
                        rg = ctx.residual(b, cl).cpu().numpy()
                        assert np.array_equal(rg.view(np.uint32), myr.view(np.uint32)), \
                            f"rank {rank} residual mismatch b{b} t{t}"
                    # every slot (all clusters' payloads) after the exchange == oracle payloads
                    if G == 1:
                        for c in range(P):
                            assert ctx.payload_copy(b, c) == payloads[c], f"slot {c} mismatch b{b}"
                    off += n
            dist.barrier()          # nebula_sync_destroy is collective with peer mappings
            ctx.destroy()
    dist.barrier()
    if rank == 0:
        print(f"DIST OK world={world} P={P} G={G} cases={len(cases)} steps={args.steps} "
              f"exchange={sorted(modes_seen)} intra={sorted(intra_seen)}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
