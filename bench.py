#!/usr/bin/env python
"""bench.py — compressed gradient sync throughput (BASELINE.json metric:
"GB/s fp32 gradient synced per GPU (1/2/4/8 B200); % HBM roofline").

A step is one pass of the whole hot path (EF-accumulate, compress+pack,
exchange, decompress+average, residual update) over every bucket of one synthetic gradient.

  N = 1 : BASELINE config 2 — ERNIE-M-base-shaped gradient (278,042,880 fp32), P = 2
          simulated clusters on one B200 (LOOPBACK transport), fixed 25 MiB buckets.
  N > 1 : (torchrun) one cluster per GPU, P = N, NCCL over NVLink, same gradient shape per
          GPU (weak scaling: every GPU syncs its full replica gradient).

value = fp32 gradient GB/s synced PER GPU (the BASELINE metric's unit): the fp32 bytes of the
gradient(s) one GPU synchronises / device time of K steps (max over ranks) — at N = 1 the GPU
hosts both simulated clusters (2 n elements), at N > 1 its own replica (n elements);
value_aggregate = the same summed over the N GPUs.  At N > 1 the roofline is the larger of the
HBM time and the NVLink time, the latter against an in-run 1 GiB all-gather bus bandwidth.  e2e = the same through nebula_step_host (pinned host buffers, H2D + D2H inside the
timed region).  cpu_baseline = the CPU oracle on a bounded sample (rank 0, N = 1 only).
`--impl reference` runs the oracle as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METHODS = {"identity": 0, "fp16": 1, "int8": 2, "topk": 3, "fp8": 4, "qsgd": 6, "fp8e5m2": 7}
VALUES = {"f32": 0, "f16": 1, "i8": 2}
VB = {0: 4, 1: 2, 2: 1}
METRIC = "GB/s fp32 gradient synced per GPU (1/2/4/8 B200); % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="nebula", choices=["nebula", "reference"])
    ap.add_argument("--method", default="int8", choices=list(METHODS))
    ap.add_argument("--values", default="f32", choices=list(VALUES))
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--workload", default="ernie-m-base",
                    choices=["ernie-m-base", "ernie-m-large", "ernie-m-large-adapters", "transformer-big"])
    ap.add_argument("--bucket-mib", type=float, default=25.0)
    ap.add_argument("--clusters", type=int, default=2, help="simulated clusters at N=1 (LOOPBACK)")
    ap.add_argument("--gpus-per-cluster", type=int, default=1,
                    help="G > 1: hierarchical topology (P = N / G clusters; BASELINE config 3 is 2 x 4)")
    ap.add_argument("--no-ef", action="store_true")
    ap.add_argument("--exact-scale", action="store_true",
                    help="G > 1: cluster-wide INT8/FP8 scale (NEBULA_OPT_EXACT_SCALE, NEXT-3)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "nccl", "push", "pull"])
    ap.add_argument("--intra", default="auto", choices=["auto", "p2p", "nccl"],
                    help="G > 1: intra-cluster hop (NEBULA_OPT_INTRA)")
    ap.add_argument("--fp16-kernel", default="tma", choices=["tma", "plain"])
    ap.add_argument("--no-step-fusion", action="store_true",
                    help="run compress / exchange / reduce as separate launches (NEBULA_OPT_STEP_FUSION=1)")
    ap.add_argument("--step-config", type=int, default=None, help="fused-step warp split 0..10 (tuning)")
    ap.add_argument("--int8-kernel", default="auto", choices=["auto", "two-pass", "single-pass", "fused-ws"])
    ap.add_argument("--no-pipeline", action="store_true",
                    help="one stream per step (no two-half pipelining of ALL-bucket steps)")
    ap.add_argument("--topk-stage", default="tma", choices=["tma", "plain"],
                    help="top-k stage pass: TMA ring (default) or plain vector loads")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def load_traffic(workload_name, method_name, bucket_mib, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture of the same workload
    (profiles/*/traffic.json), else None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "traffic.json")), reverse=True):
        try:
            with open(path) as f:
                d = json.load(f)
            if d["workload"] == workload_name and d["method"] == method_name and float(d["bucket_mib"]) == bucket_mib:
                v = d["per_launch_dram_bytes"].get(kernel)
                if v:
                    return int(v)
        except Exception:
            continue
    return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------------------- accounting
def kernel_bytes(phase, method, vt, P, ef, n_elems, k_total):
    """Algorithmic HBM bytes of one launch of `phase` over `n_elems` coded elements
    (all items of the launch) — DESIGN.md "Roofline" table."""
    e = 4 if ef else 0
    if phase == "int8_ef_absmax":
        return (4 + e) * n_elems
    if phase == "int8_ef_quant_pack":
        return (4 + e + e + 1) * n_elems
    if phase == "qsgd_ef_quant_pack":
        return (4 + e + e + 1) * n_elems
    if phase == "fp8_ef_quant_pack":
        return (4 + e + e + 1) * n_elems
    if phase == "fp16_ef_pack":
        return (4 + e + e + 2) * n_elems
    if phase == "identity_pack":
        return 8 * n_elems
    if phase == "topk_ef_sample":
        return (4 + e + e) * n_elems
    if phase == "topk_classify":
        return 4 * n_elems
    if phase == "int8_fused_ef_quant_pack":
        return (4 + e + e + 1) * n_elems
    return None


def reduce_bytes(method, vt, P, n_out, k_per_cluster):
    if method == 3:
        return P * k_per_cluster * (4 + VB[vt]) + 4 * n_out
    b = {0: 4, 1: 2, 2: 1, 4: 1, 6: 1, 7: 1}[method]
    return P * b * n_out + 4 * n_out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled (every 20 ms) during the timed region.
    The sampler is started (and its first row awaited) before the region; only rows stamped
    inside [start, stop] are summarised (the nearest row if the region is shorter)."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def __enter__(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown," \
            "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
            "clocks_event_reasons.sw_power_cap,power.draw"
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "20", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            deadline = time.time() + 5
            while not self.rows and time.time() < deadline:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for t, r in self.rows if self.t0 is not None and self.t0 <= t <= (self.t1 or t) + 0.02]
        if not rows and self.rows and self.t0 is not None:
            rows = [min(self.rows, key=lambda tr: abs(tr[0] - self.t0))[1]]
        sm, mx, reasons, pw = [], None, set(), []
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for i, nm in enumerate(self.NAMES):
                    if r[2 + i].lower().startswith("active"):
                        reasons.add(nm)
                pw.append(float(r[6]))
            except Exception:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ----------------------------------------------------------------------------- oracle (CPU) legs
def oracle_sample(method, vt, density, ef, P, bucket_elems, budget_s, gs, max_buckets=None):
    """Time the oracle (as it stands) on a bounded sample: P clusters x successive buckets of
    the same synthetic gradient gs[c], until ~budget_s of CPU work (at least one bucket)."""
    import oracle as O
    codec = O.Codec(method=method, topk_values=vt, topk_density=density, error_feedback=ef)
    elems, t_used, nb = 0, 0.0, 0
    off = 0
    while (nb == 0 or t_used < budget_s) and off < gs[0].size and (max_buckets is None or nb < max_buckets):
        n = min(bucket_elems, gs[0].size - off)
        parts = [g[off:off + n] for g in gs]
        t0 = time.perf_counter()
        O.oracle_step(parts, [np.zeros(n, np.float32) for _ in range(P)], codec, 1)
        t_used += time.perf_counter() - t0
        elems += n
        nb += 1
        off += n
    return elems, t_used, nb


def cpu_desc():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    method, vt, ef = METHODS[args.method], VALUES[args.values], not args.no_ef
    from gradgen import fixed_buckets, model_numel
    n = model_numel(args.workload)
    per = fixed_buckets(n, int(args.bucket_mib * 2 ** 20))[0]
    G = args.gpus_per_cluster if args.gpus > 1 else 1
    P = args.clusters if args.gpus == 1 else args.gpus // G
    budget = max(1.0, 120.0 / max(1, args.steps + args.warmup))
    from gradgen import model_gradient
    gs = [model_gradient(args.workload, cluster=c) for c in range(P)]
    for _ in range(args.warmup):
        oracle_sample(method, vt, args.density, ef, P, per, 0.0, gs, max_buckets=1)
    elems = t = 0.0
    for _ in range(args.steps):
        e, tt, _ = oracle_sample(method, vt, args.density, ef, P, per, budget, gs)
        elems += e
        t += tt
    value = (P if args.gpus == 1 else 1) * elems * 4 / t / 1e9   # per GPU, as the repo arm
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": workload_config(args, n, P, G),
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"per step: P={P} clusters x 25 MiB buckets of the {args.workload} gradient "
                                       f"until ~{budget:.1f}s; single-threaded NumPy on '{cpu_desc()}' "
                                       f"({os.cpu_count()} host cores)"},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, n, P, G=1):
    mname = {0: "identity", 1: "fp16+ef", 2: "int8+ef", 3: f"topk{args.density:g}-{args.values}+ef",
             4: "fp8e4m3+ef", 6: "qsgd-int8-sr+ef", 7: "fp8e5m2+ef"}[METHODS[args.method]]
    if args.exact_scale and G > 1:
        mname += "+exact-cluster-scale"
    if args.no_ef:
        mname = mname.replace("+ef", "")
    return {"workload": f"{args.workload}-" + (f"loopback-P{P}" if args.gpus == 1 else f"P{P}xG{G}"),
            "elements_per_cluster": n, "clusters": P, "gpus_per_cluster": G, "method": mname,
            "bucketing": f"fixed {args.bucket_mib:g} MiB slices of the flat gradient",
            "transport": "loopback" if args.gpus == 1 else "nvlink",
            "l2": (f"per-GPU working set (gradient + residual + output, {3 * 4 * n / 1e6:.0f} MB) exceeds "
                   "the 126 MB L2; no flush needed"),
            "pipeline": "off" if args.no_pipeline else "auto"}


# ----------------------------------------------------------------------------- main arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    import paper_2205_09470_b200 as nb
    from paper_2205_09470_b200 import build
    from gradgen import fixed_buckets, model_gradient

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if rank == 0:
        build.build()
    torch.cuda.set_device(local)
    busbw = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        busbw = nvlink_busbw(world)
    if rank != 0:
        build.build()   # up to date after rank 0's build + barrier: loads only
    method, vt, ef = METHODS[args.method], VALUES[args.values], not args.no_ef
    n = None
    G = args.gpus_per_cluster if world > 1 else 1
    if world % G:
        raise SystemExit("--gpus must be a multiple of --gpus-per-cluster")
    P = args.clusters if world == 1 else world // G
    stream = torch.cuda.current_stream()

    # ---- inputs (seeded synthetic, gradgen recipe), resident in HBM before timing
    if world == 1:
        host = [model_gradient(args.workload, cluster=c) for c in range(P)]
        n = host[0].size
        g = torch.empty(P * n, dtype=torch.float32, device="cuda")
        for c in range(P):
            g[c * n:(c + 1) * n].copy_(torch.from_numpy(host[c]))
        del host
    else:
        h = model_gradient(args.workload, cluster=rank // G, local_rank=rank % G)
        n = h.size
        g = torch.from_numpy(h).cuda()
        del h
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    sizes = fixed_buckets(n, int(args.bucket_mib * 2 ** 20), multiple=4 * G)
    if any(sz % G for sz in sizes):
        raise SystemExit(f"{args.workload}: {n} elements cannot be split into shards of {G}")
    common = dict(topk_values=vt, topk_density=args.density, error_feedback=ef)
    if world == 1:
        ctx = nb.SyncContext(sizes, method, num_clusters=P, transport=nb.LOOPBACK, device=local, **common)
    else:
        ctx = nb.init_process_group_context(sizes, gpus_per_cluster=G, device=local, method=method, **common)
    if method == 2:
        ctx.set_int8_kernel(args.int8_kernel)
    if method == 1:
        ctx.set_fp16_kernel(args.fp16_kernel)
    if args.exact_scale and G > 1:
        ctx.set_exact_scale(True)
    if args.no_step_fusion:
        ctx.set_step_fusion(False)
    if args.step_config is not None:
        ctx.set_option(nb.OPT_STEP_FUSION, 2 + args.step_config)
    if args.no_pipeline:
        ctx.set_option(nb.OPT_PIPELINE, 0)
    if method == 3 and args.topk_stage == "plain":
        ctx.set_option(nb.OPT_TOPK_STAGE, 0)
    if world > 1 and args.exchange != "auto":
        ctx.set_exchange(args.exchange)
    if G > 1 and args.intra != "auto":
        ctx.set_intra(args.intra)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    step = 0
    for _ in range(args.warmup):
        ctx.step(nb.ALL_BUCKETS, g, out, step)
        step += 1
    ctx.check()
    ctx.timing_enable(True)
    ctx.timing_read()
    barrier()
    l0 = ctx.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        clk.start()
        e0.record(stream)
        for _ in range(args.steps):
            ctx.step(nb.ALL_BUCKETS, g, out, step)
            step += 1
        e1.record(stream)
        barrier()
        clk.stop()
    launches = ctx.kernel_launches() - l0
    ms = e0.elapsed_time(e1)
    phases = ctx.timing_read()
    ctx.timing_enable(False)
    ctx.check()
    t_max = ms
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    ms_step = t_max / args.steps
    gpu_bytes = P * n * 4 if world == 1 else n * 4      # fp32 bytes this GPU synchronises per step
    synced_bytes = gpu_bytes * world                     # all GPUs
    value = gpu_bytes / (ms_step * 1e-3) / 1e9
    value_aggregate = synced_bytes / (ms_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel
    peak, peak_src = load_peaks()
    n_local = (P if world == 1 else 1) * n // G          # coded elements on this GPU (a shard when G > 1)
    k_per_cluster = sum(min(s // G, max(1, int(np.floor(args.density * (s // G) + 0.5)))) for s in sizes) \
        if method == 3 else 0
    kern = {}
    for name, (cnt, tot) in phases.items():
        kern[name] = {"launches_per_step": cnt / args.steps, "ms_per_step": tot / args.steps,
                      "share": (tot / args.steps) / ms_step if ms_step else None}
    dom = max((k for k in phases if not k.startswith("nccl") and k != "memset"), key=lambda k: phases[k][1],
              default=None)
    roof = None
    if dom:
        cnt, tot = phases[dom]
        if dom in ("dense_decompress_reduce", "sparse_decompress_reduce"):
            byt = reduce_bytes(method, vt, P, n // G, k_per_cluster)
        elif dom == "int8_fused_step":   # compress of the local clusters + the average (one kernel)
            byt = kernel_bytes("int8_fused_ef_quant_pack", method, vt, P, ef, n_local, 0) + \
                reduce_bytes(method, vt, P, n // G, 0)
        elif dom == "fp16_fused_step":
            byt = kernel_bytes("fp16_ef_pack", method, vt, P, ef, n_local, 0) + reduce_bytes(method, vt, P, n // G, 0)
        else:
            byt = kernel_bytes(dom, method, vt, P, ef, n_local, k_per_cluster * (P if world == 1 else 1))
        if byt:
            # byt covers every element the phase processes in a step; with several launches per
            # step (e.g. the two halves of the pipelined top-k step) each launch moves its share
            byt = byt / max(1.0, cnt / args.steps)
            per_launch_s = tot / cnt * 1e-3
            ach = byt / per_launch_s / 1e9
            wc = workload_config(args, n, P, G)
            roof = {"kernel": dom, "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4),
                    "traffic": load_traffic(wc["workload"], wc["method"], args.bucket_mib, dom),
                    "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": int(byt), "ms_per_launch": round(tot / cnt, 4)}
            if method == 3 and cnt > args.steps:
                roof["note"] = ("two-stream top-k step: the two halves' launches of this kernel run "
                                "concurrently and share HBM, so each launch's duration includes the "
                                "other's traffic; serialized (--no-pipeline, or ncu) the kernel runs "
                                "at ~0.86-0.90 of the peak; step_roofline is the whole-step figure")
    step_bytes = step_algorithmic_bytes(method, vt, P, ef, n, k_per_cluster, world)
    if world > 1 and (busbw or 0) > 0:
        # NVLink bound: bytes INTO this GPU per step (P - 1 peers' payloads of its shard, plus
        # the G > 1 intra-cluster fp32 hop: (G - 1) / G of the bucket in each of RS and AG)
        pb = payload_elems_bytes(method, vt, n // G, k_per_cluster)
        nv = (P - 1) * pb + (2 * (G - 1) * (n // G) * 4 if G > 1 else 0)
        t_hbm, t_nv = step_bytes / peak, nv / busbw
        if t_nv > t_hbm:
            roof = {"kernel": "whole step (exchange)", "bound": "nvlink",
                    "achieved": round(nv / (ms_step * 1e-3) / 1e9, 1), "peak": round(busbw, 1), "unit": "GB/s",
                    "frac": round(nv / (ms_step * 1e-3) / 1e9 / busbw, 4), "traffic": None,
                    "peak_source": "in-run ncclAllGather bus bandwidth, 1 GiB, min over ranks",
                    "nvlink_bytes_in_per_step": int(nv), "hbm_kernel_roofline": roof}
    step_roof = {"algorithmic_bytes_per_step": int(step_bytes),
                 "achieved_gbs": round(step_bytes / (ms_step * 1e-3) / 1e9, 1),
                 "frac_of_hbm_peak": round(step_bytes / (ms_step * 1e-3) / 1e9 / peak, 4)}

    # ---- e2e through the host-buffer C-ABI call
    e2e = None
    if not args.no_e2e:
        gelems = (P if world == 1 else 1) * n
        hg = torch.empty(gelems, dtype=torch.float32, pin_memory=True)
        ho = torch.empty(n, dtype=torch.float32, pin_memory=True)
        hg.copy_(g.cpu())
        ke = max(2, min(args.steps, 10))
        ctx.step_host(hg, ho, step)
        step += 1
        barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            ctx.step_host(hg, ho, step)
            step += 1
        barrier()
        te = (time.perf_counter() - t0) / ke
        if world > 1:
            tt = torch.tensor([te], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": round(synced_bytes / te / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(gelems * 4),
               "d2h_bytes_per_step": int(n * 4), "steps": ke,
               "note": "wall clock around nebula_step_host (H2D of every cluster's gradient from pinned memory, "
                       "step, D2H of the averaged gradient, stream sync)"}
        del hg, ho

    # ---- CPU oracle baseline (rank 0, N = 1)
    cpu = None
    if world == 1 and not args.no_cpu:
        from gradgen import model_gradient as _mg
        gs_cpu = [_mg(args.workload, cluster=c) for c in range(P)]
        elems, t_used, nbk = oracle_sample(method, vt, args.density, ef, P, sizes[0], args.cpu_seconds, gs_cpu)
        del gs_cpu
        cpu = {"value": round(P * elems * 4 / t_used / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"{nbk} x {sizes[0]}-element buckets x P={P} clusters of the same {args.workload} "
                         f"gradient ({elems} elements per cluster, {t_used:.1f} s), single-threaded NumPy on "
                         f"'{cpu_desc()}' ({os.cpu_count()} host cores)"}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "value_aggregate": round(value_aggregate, 2), "exchange": ctx.exchange_mode(),
                "intra": ctx.intra_mode(), "nvlink_busbw_gbs": round(busbw, 1) if busbw else None,
                "config": workload_config(args, n, P, G), "roofline": roof, "step_roofline": step_roof,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "kernels": kern,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    ctx.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


def payload_elems_bytes(method, vt, n, k):
    """Payload bytes of one cluster's bucket(s) of n coded elements (k = top-k entries)."""
    if method == 3:
        return k * (4 + VB[vt])
    return n * {0: 4, 1: 2, 2: 1, 4: 1, 6: 1, 7: 1}[method]


def nvlink_busbw(world):
    """In-run NVLink roofline: ncclAllGather bus bandwidth over 1 GiB (min over ranks)."""
    import torch
    import torch.distributed as dist
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
    bw = (world - 1) / world * y.numel() * 4 / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e9
    t = torch.tensor([bw], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    del x, y
    torch.cuda.empty_cache()
    return float(t.item())


def step_algorithmic_bytes(method, vt, P, ef, n, k_per_cluster, world):
    """Minimum HBM bytes of one step on one GPU."""
    e = 4 if ef else 0
    clusters_here = P if world == 1 else 1
    if method in (2, 4, 6, 7):   # single pass (warp-specialised kernel / fused step) for INT8, FP8, QSGD
        comp = (4 + e + e + 1) * n
    elif method == 1:
        comp = (4 + e + e + 2) * n
    elif method == 0:
        comp = 8 * n
    else:
        comp = (4 + e + e) * n + k_per_cluster * (4 + VB[vt]) + (4 * k_per_cluster if ef else 0)
    exch = 0 if world == 1 else 2 * (P - 1) * (n * {0: 4, 1: 2, 2: 1, 4: 1, 6: 1, 7: 1}.get(method, 0) + (k_per_cluster * (4 + VB[vt]) if method == 3 else 0))
    red = reduce_bytes(method, vt, P, n, k_per_cluster)
    return clusters_here * comp + exch + red


if __name__ == "__main__":
    sys.exit(main())
