#!/usr/bin/env python
"""Debug: TOPK 10 % at config-2 size — per-bucket stats of the one-stream step, then the
two-stream step (pipelined) on the same inputs; both must be bit-identical."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2205_09470_b200 as nb
    from gradgen import fixed_buckets, model_gradient
    P = 2
    rho = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
    host = [model_gradient("ernie-m-base", cluster=c) for c in range(P)]
    n = host[0].size
    g = torch.empty(P * n, device="cuda")
    for c in range(P):
        g[c * n:(c + 1) * n].copy_(torch.from_numpy(host[c]))
    sizes = fixed_buckets(n, 25 << 20)
    outs = {}
    for pipe in (0, 1):
        ctx = nb.SyncContext(sizes, 3, topk_density=rho, num_clusters=P, transport=nb.LOOPBACK)
        ctx.set_option(nb.OPT_PIPELINE, pipe)
        out = torch.empty(n, device="cuda")
        try:
            for s in range(int(os.environ.get("DBG_STEPS", "2"))):
                ctx.step(nb.ALL_BUCKETS, g, out, s)
                torch.cuda.synchronize()
                ctx.check()
                print("pipe", pipe, "step", s, "ok", flush=True)
        except Exception as e:
            print("pipe", pipe, "FAILED", repr(e), flush=True)
            return
        if pipe == 0:
            for b in range(len(sizes)):
                for c in range(P):
                    st = ctx.topk_stats(b, c)
                    print("bucket", b, "half", 1 if b < len(sizes) // 2 else 2, "cluster", c, st, flush=True)
        outs[pipe] = out.clone()
        ctx.destroy()
    d = (outs[0] != outs[1]).nonzero()
    print("mismatches", d.numel(), d[:10].flatten().tolist(), flush=True)


if __name__ == "__main__":
    main()
