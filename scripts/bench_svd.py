#!/usr/bin/env python
"""FP16(SVD(rho)) compressor timing (NEXT-1) at the paper's Scenario-II activation shape
(H^E = 128 x 64 tokens x 768) for Table 5's rho column.

Prints one JSON line per rho: compress / decompress ms (CUDA events on the handle's stream,
median of --iters after --warmup), payload ratio, fp32 bytes of A per second, and the
GEMM-equivalent flop rate of the three contractions (Gram 2 L k^2 / 2, projection 2 L k r,
reconstruction 2 m n r).  Synthetic input: low-rank (decay 0.995) + 1e-3 noise, seeded."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=128 * 64)
    ap.add_argument("--n", type=int, default=768)
    ap.add_argument("--rhos", default="0.9,0.8,0.7,0.6,0.5,0.4,0.3,0.2")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--eig", default="syevd", choices=["syevd", "syevj"])
    ap.add_argument("--gram", default="dmma", choices=["dmma", "simt"])
    args = ap.parse_args()
    import torch
    import paper_2205_09470_b200 as nb
    from paper_2205_09470_b200 import build
    build.build()
    m, n = args.m, args.n
    k, L = min(m, n), max(m, n)
    rng = np.random.default_rng(7)
    Q1, _ = np.linalg.qr(rng.standard_normal((m, k)))
    Q2, _ = np.linalg.qr(rng.standard_normal((n, k)))
    A = ((Q1 * (20.0 * 0.995 ** np.arange(k))[None, :]) @ Q2.T + 1e-3 * rng.standard_normal((m, n))).astype(np.float32)
    dA = torch.from_numpy(A).cuda()
    out = torch.empty(m, n, device="cuda")
    for rho in [float(x) for x in args.rhos.split(",")]:
        h = nb.SvdCodec(m, n, rho=rho)
        h.set_eigensolver(args.eig, args.gram)
        r = h.r
        pl = torch.empty(h.payload_bytes(), dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream()
        tc, td = [], []
        for it in range(args.warmup + args.iters):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(st)
            h.compress(dA, pl)
            e1.record(st)
            h.decompress(pl, out)
            e2.record(st)
            torch.cuda.synchronize()
            if it >= args.warmup:
                tc.append(e0.elapsed_time(e1))
                td.append(e1.elapsed_time(e2))
        h.check()
        err = float(torch.linalg.norm(out - dA) / torch.linalg.norm(dA))
        c, d = float(np.median(tc)), float(np.median(td))
        flops_c = L * k * k + 2.0 * L * k * r
        flops_d = 2.0 * m * n * r
        print(json.dumps({"workload": f"svd-fp16 m={m} n={n}", "eigensolver": args.eig, "gram": args.gram, "rho": rho, "r": r,
                          "payload_ratio": round((h.payload_bytes() - 16) / (4.0 * m * n), 4),
                          "compress_ms": round(c, 4), "decompress_ms": round(d, 4),
                          "compress_gbs_fp32": round(4.0 * m * n / c / 1e6, 2),
                          "decompress_gbs_fp32": round(4.0 * m * n / d / 1e6, 2),
                          "contraction_tflops_compress": round(flops_c / c / 1e9, 2),
                          "contraction_tflops_decompress": round(flops_d / d / 1e9, 2),
                          "rel_reconstruction_error": round(err, 6)}), flush=True)
        h.destroy()


if __name__ == "__main__":
    main()
