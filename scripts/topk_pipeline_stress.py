#!/usr/bin/env python
"""Three TOPK contexts on the same inputs in lock-step — A and B one-stream, C two-stream;
after every step compare the outputs (A vs B: nondeterminism of the serial path; A vs C: of the
two-stream path) and, on a difference, which buckets' payloads differ."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2205_09470_b200 as nb
    from gradgen import fixed_buckets, model_gradient
    P = 2
    rho = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    host = [model_gradient("ernie-m-base", cluster=c) for c in range(P)]
    n = host[0].size
    sizes = fixed_buckets(n, 25 << 20)
    offs = np.cumsum([0] + list(sizes))
    g = torch.empty(P * n, device="cuda")
    for c in range(P):
        g[c * n:(c + 1) * n].copy_(torch.from_numpy(host[c]))
    ctxs, outs = [], []
    for pipe in (0, 0, 1):
        ctx = nb.SyncContext(sizes, 3, topk_density=rho, num_clusters=P, transport=nb.LOOPBACK)
        ctx.set_option(nb.OPT_PIPELINE, pipe)
        ctxs.append(ctx)
        outs.append(torch.empty(n, device="cuda"))
    for s in range(steps):
        for ctx, out in zip(ctxs, outs):
            ctx.step(nb.ALL_BUCKETS, g, out, s)
        torch.cuda.synchronize()
        for ctx in ctxs:
            ctx.check()
        for name, j in (("A-B", 1), ("A-C", 2)):
            d = (outs[0].view(torch.int32) != outs[j].view(torch.int32)).nonzero().flatten()
            if d.numel():
                e = d[:5].tolist()
                bks = sorted(set(int(np.searchsorted(offs, x, side="right") - 1) for x in d[:2000].tolist()))
                pl = []
                for b in bks[:4]:
                    for c in range(P):
                        if ctxs[0].payload_copy(b, c) != ctxs[j].payload_copy(b, c):
                            pl.append((b, c))
                print(f"step {s} {name}: {d.numel()} outputs differ, first {e}, buckets {bks[:8]}, payload diffs {pl}",
                      flush=True)
                # resynchronise the diverged context's state is not possible: report and stop
                return
        print(f"step {s} ok", flush=True)


if __name__ == "__main__":
    main()
