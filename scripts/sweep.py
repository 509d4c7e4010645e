#!/usr/bin/env python
"""BASELINE.json configs 1 and 5 as JSONL (one line per point).

  config 1: one 1M-float (2^20) bucket, P = 2 clusters x 1 GPU: step latency in us for
            INT8+EF (primary), FP16+EF, TOPK 1 % / 10 % (the CPU oracle is timed only by
            bench.py's cpu_baseline / reference arm: no script outside tests/ runs it).  N = 1: LOOPBACK (both clusters on one GPU); N = 2 (torchrun):
            the real 2-GPU exchange over NVLink.
  config 5: bucket 1 MiB .. 1 GiB (2^18 .. 2^28 elements) x {INT8+EF, FP16+EF, TOPK rho in
            {1, 5, 10, 25, 50} % x values {f32, f16, i8}}: GB/s fp32 synced per GPU and the step's
            fraction of the HBM roofline (algorithmic bytes / time / measured copy peak); at
            N > 1 also the NVLink bytes per direction and their fraction of the in-run
            all-gather bus bandwidth.

Every point: a fresh single-bucket context, 3 warm-up steps, then per-step CUDA events on the
context's stream around each step with a 256 MiB L2 flush between steps (outside the events);
the median step time (max over ranks).  Inputs: the first n elements of the ERNIE-M-base
synthetic gradient (gradgen recipe) of each cluster.

  python scripts/sweep.py --config 5 --out profiles/r02/config5_n1.jsonl
  torchrun --nproc-per-node 2 scripts/sweep.py --config 1 --out profiles/r02/config1_n2.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VB = {0: 4, 1: 2, 2: 1}


def specs(config):
    if config == 1:
        return [("int8", 2, 0, 0.0), ("fp16", 1, 0, 0.0), ("topk", 3, 0, 0.01), ("topk", 3, 0, 0.10)]
    out = [("int8", 2, 0, 0.0), ("fp16", 1, 0, 0.0)]
    for rho in (0.01, 0.05, 0.10, 0.25, 0.50):
        for vt in (0, 1, 2):
            out.append(("topk", 3, vt, rho))
    return out


def hbm_bytes(method, vt, P_here, P, n, k):
    """Algorithmic HBM bytes of one step on one GPU: compress of the clusters
    hosted here (+ EF), the exchange's local writes / reads, the average."""
    if method == 2:
        comp = 13 * n
        red = (P + 4) * n
    elif method == 1:
        comp = 14 * n
        red = (2 * P + 4) * n
    else:
        comp = 12 * n + k * (4 + VB[vt]) + 4 * k
        red = P * k * (4 + VB[vt]) + 4 * n
    return P_here * comp + red


def payload(method, vt, n, k):
    if method == 2:
        return 16 + -(-n // 16) * 16
    if method == 1:
        return 16 + -(-2 * n // 16) * 16
    return 16 + -(-4 * k // 16) * 16 + -(-VB[vt] * k // 16) * 16


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, choices=[1, 5], default=5)
    ap.add_argument("--out", required=True)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--sizes", default="18,20,22,24,26,28", help="log2 bucket elements")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_2205_09470_b200 as nb
    from gradgen import model_gradient

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nb.load()
    P = 2 if world == 1 else world
    P_here = P if world == 1 else 1
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    busbw = None
    if world > 1:   # in-run NVLink roofline: 1 GiB all-gather bus bandwidth
        x = torch.empty((1 << 30) // world // 4, device="cuda")
        y = torch.empty(x.numel() * world, device="cuda")
        for _ in range(3):
            dist.all_gather_into_tensor(y, x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            dist.all_gather_into_tensor(y, x)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10 * 1e-3
        busbw = (world - 1) / world * y.numel() * 4 / t / 1e9
        tt = torch.tensor([busbw], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MIN)
        busbw = float(tt.item())
        del x, y
    sizes = [1 << 20] if args.config == 1 else [1 << int(s) for s in args.sizes.split(",")]
    nmax = max(sizes)
    if world == 1:
        src = [torch.from_numpy(model_gradient("ernie-m-base", cluster=c)[:nmax].copy()) for c in range(P)]
    else:
        src = [torch.from_numpy(model_gradient("ernie-m-base", cluster=rank)[:nmax].copy())]
    flush = torch.empty(64 << 20, device="cuda")
    out_f = open(args.out, "a") if rank == 0 else None
    for n in sizes:
        g = torch.cat([s[:n] for s in src]).cuda()
        out = torch.empty(n, device="cuda")
        for name, method, vt, rho in specs(args.config):
            kw = dict(topk_values=vt, topk_density=rho if rho else 0.01)
            if world == 1:
                ctx = nb.SyncContext([n], method, num_clusters=P, transport=nb.LOOPBACK, device=local, **kw)
            else:
                ctx = nb.init_process_group_context([n], device=local, method=method, **kw)
            st = torch.cuda.current_stream()
            for s in range(3):
                ctx.step(nb.ALL_BUCKETS, g, out, s)
            ctx.check()
            times = []
            for s in range(args.steps):
                flush.fill_(float(s))
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                ctx.step(nb.ALL_BUCKETS, g, out, 3 + s)
                b.record(st)
                b.synchronize()
                times.append(a.elapsed_time(b))
            ctx.check()
            # per-phase breakdown in a separate pass (the timers' events would add to the latency)
            ctx.timing_enable(True)
            ctx.timing_read()
            for s in range(args.steps):
                ctx.step(nb.ALL_BUCKETS, g, out, 3 + args.steps + s)
            torch.cuda.synchronize()
            phases = ctx.timing_read()
            ctx.timing_enable(False)
            ctx.check()
            ms = float(np.median(times))
            if world > 1:
                tt = torch.tensor([ms], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                ms = float(tt.item())
            k = max(1, min(n, int(np.floor(rho * n + 0.5)))) if method == 3 else 0
            byt = hbm_bytes(method, vt, P_here, P, n, k)
            rec = {"config": args.config, "n_gpus": world, "clusters": P,
                   "transport": "loopback" if world == 1 else ctx.exchange_mode(),
                   "bucket_mib": n * 4 / 2 ** 20, "elements": n, "method": name + ("+ef"),
                   "values": {0: "f32", 1: "f16", 2: "i8"}[vt] if method == 3 else None,
                   "rho": rho if method == 3 else None, "k": k or None,
                   "us_per_step": round(ms * 1e3, 2),
                   "gbs_fp32_synced_per_gpu": round(P_here * n * 4 / (ms * 1e-3) / 1e9, 2),
                   "hbm_algorithmic_bytes": byt, "hbm_frac": round(byt / (ms * 1e-3) / 1e9 / peak, 4),
                   "payload_bytes": payload(method, vt, n, k),
                   "phase_ms_per_step": {kk: round(v[1] / args.steps, 4) for kk, v in phases.items()}}
            if world > 1:
                nv = (P - 1) * payload(method, vt, n, k)      # bytes into this GPU per step
                rec["nvlink_bytes_in"] = nv
                rec["nvlink_busbw_gbs"] = round(busbw, 1)
                rec["nvlink_frac"] = round(nv / (ms * 1e-3) / 1e9 / busbw, 4)
                rec["bound"] = "nvlink" if nv / busbw > byt / peak else "hbm"
            if out_f:
                out_f.write(json.dumps(rec) + "\n")
                out_f.flush()
                print(json.dumps(rec), flush=True)
            if world > 1:
                dist.barrier()
            ctx.destroy()
        del g, out
        torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
