#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
T="timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k topk"
for i in 1 2; do NEBULA_EXPERIMENT_WIDE_MIN=8192 $T > gpurun_out/dbg2_w8192_$i.log 2>&1; echo "rc $?" >> gpurun_out/dbg2_w8192_$i.log; done
for i in 1 2; do $T > gpurun_out/dbg2_default_$i.log 2>&1; echo "rc $?" >> gpurun_out/dbg2_default_$i.log; done
NEBULA_EXPERIMENT_STAGE_PLAIN=1 NEBULA_EXPERIMENT_WIDE_MIN=8192 $T > gpurun_out/dbg2_w8192_plain.log 2>&1; echo "rc $?" >> gpurun_out/dbg2_w8192_plain.log
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 10 --method topk --density 0.1"
NEBULA_EXPERIMENT_WIDE_MIN=32768 $B > gpurun_out/dbg2_b10_w32768.log 2>&1
NEBULA_EXPERIMENT_STAGE_PLAIN=1 NEBULA_EXPERIMENT_WIDE_MIN=32768 $B > gpurun_out/dbg2_b10_w32768_plain.log 2>&1
timeout 600 python -m pytest tests/test_gpu_division.py tests/test_gpu_parity.py -q -x -k "qsgd or division" > gpurun_out/dbg2_qsgd.log 2>&1; echo "rc $?" >> gpurun_out/dbg2_qsgd.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 30 --method qsgd > gpurun_out/dbg2_bench_qsgd.log 2>&1
timeout 300 python bench.py --no-cpu --no-e2e --steps 30 --method qsgd --no-ef > gpurun_out/dbg2_bench_qsgd_noef.log 2>&1
