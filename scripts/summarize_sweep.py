#!/usr/bin/env python
"""Markdown summary of a config-5 / config-1 sweep JSONL (scripts/sweep.py): one row per
(bucket, codec), us per step, GB/s per GPU, HBM / NVLink fractions."""
import json
import sys


def main(path):
    rows = [json.loads(l) for l in open(path) if l.strip()]
    print("| bucket MiB | codec | µs / step | GB/s per GPU | HBM frac | NVLink frac |")
    print("|---|---|---|---|---|---|")
    for d in rows:
        codec = d["method"] + (f" ρ={d['rho']:g} {d['values']}" if d.get("rho") else "")
        print(f"| {d['bucket_mib']:g} | {codec} | {d['us_per_step']:.1f} | {d['gbs_fp32_synced_per_gpu']:.1f} | "
              f"{d['hbm_frac']:.3f} | {d.get('nvlink_frac', '—')} |")


if __name__ == "__main__":
    main(sys.argv[1])
