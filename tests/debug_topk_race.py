#!/usr/bin/env python
"""Debug: which of the one-stream / two-stream TOPK 10 % steps at config-2 size diverges from
the oracle, on the bucket holding element E, step by step (payload, residual, output)."""
import hashlib
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))   # run from the repo root: python tests/debug_topk_race.py


def h(b):
    return hashlib.sha1(b).hexdigest()[:12]


def main():
    import numpy as np
    import torch
    import paper_2205_09470_b200 as nb
    import oracle as O
    from gradgen import fixed_buckets, model_gradient
    P = 2
    rho = 0.1
    E = int(sys.argv[1]) if len(sys.argv) > 1 else 109432384
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    host = [model_gradient("ernie-m-base", cluster=c) for c in range(P)]
    n = host[0].size
    sizes = fixed_buckets(n, 25 << 20)
    offs = np.cumsum([0] + list(sizes))
    b = int(np.searchsorted(offs, E, side="right") - 1)
    o0, nb_ = int(offs[b]), int(sizes[b])
    print("bucket", b, "offset", o0, "n", nb_, "half", 1 if b < len(sizes) // 2 else 2, flush=True)
    g = torch.empty(P * n, device="cuda")
    for c in range(P):
        g[c * n:(c + 1) * n].copy_(torch.from_numpy(host[c]))
    rec = {}
    for pipe in (0, 1):
        ctx = nb.SyncContext(sizes, 3, topk_density=rho, num_clusters=P, transport=nb.LOOPBACK)
        ctx.set_option(nb.OPT_PIPELINE, pipe)
        out = torch.empty(n, device="cuda")
        rec[pipe] = []
        for s in range(steps):
            ctx.step(nb.ALL_BUCKETS, g, out, s)
            ctx.check()
            pl = [ctx.payload_copy(b, c) for c in range(P)]
            rr = [ctx.residual(b, c).cpu().numpy().tobytes() for c in range(P)]
            oo = out[o0:o0 + nb_].cpu().numpy().tobytes()
            st = [ctx.topk_stats(b, c) for c in range(P)]
            rec[pipe].append((pl, rr, oo, st))
        ctx.destroy()
    codec = O.Codec(method=O.TOPK, topk_density=rho)
    gs = [host[c][o0:o0 + nb_] for c in range(P)]
    rs = [np.zeros(nb_, np.float32) for _ in range(P)]
    for s in range(steps):
        exp_out, r_new, payloads, stats = O.oracle_step(gs, rs, codec, s, bucket=b)
        line = [f"step {s}"]
        for pipe in (0, 1):
            pl, rr, oo, st = rec[pipe][s]
            okp = all(pl[c] == payloads[c] for c in range(P))
            okr = all(rr[c] == r_new[c].tobytes() for c in range(P))
            oko = oo == exp_out.astype(np.float32).tobytes()
            line.append(f"pipe{pipe}: payload {'OK' if okp else 'BAD'} resid {'OK' if okr else 'BAD'} out {'OK' if oko else 'BAD'} "
                        f"T={[x.threshold for x in st]} above={[x.count_above for x in st]} cand={[x.candidates for x in st]} path={[x.path for x in st]}")
            if not oko:
                go = np.frombuffer(oo, np.float32)
                bad = np.flatnonzero(go.view(np.uint32) != exp_out.astype(np.float32).view(np.uint32))
                line.append(f"  out bad at {bad[:6].tolist()} (+{o0}) count {bad.size}")
        line.append(f"oracle T={[x['threshold'] for x in stats]} above={[x['count_above'] for x in stats]}")
        print(" | ".join(line), flush=True)
        rs = r_new


if __name__ == "__main__":
    main()
