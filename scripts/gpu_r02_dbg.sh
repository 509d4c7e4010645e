#!/bin/bash
# 1 GPU: the pipelined top-k step with the multi-CTA resolve kernels launched (low threshold):
# serialized launches vs concurrent, and repeated default-threshold runs (flakiness).
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
T="timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k two_stream_pipeline"
NEBULA_EXPERIMENT_WIDE_MIN=8192 CUDA_LAUNCH_BLOCKING=1 $T > gpurun_out/dbg_w8192_blocking.log 2>&1; echo "rc $?" >> gpurun_out/dbg_w8192_blocking.log
NEBULA_EXPERIMENT_WIDE_MIN=8192 $T > gpurun_out/dbg_w8192.log 2>&1; echo "rc $?" >> gpurun_out/dbg_w8192.log
NEBULA_EXPERIMENT_WIDE_MIN=1000000000 $T > gpurun_out/dbg_wbig.log 2>&1; echo "rc $?" >> gpurun_out/dbg_wbig.log
for i in 1 2 3; do $T > gpurun_out/dbg_default_$i.log 2>&1; echo "rc $?" >> gpurun_out/dbg_default_$i.log; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "topk_wide_resolve" > gpurun_out/dbg_wide.log 2>&1; echo "rc $?" >> gpurun_out/dbg_wide.log
timeout 300 python scripts/dbg_topk_pipe.py > gpurun_out/dbg_pipe_py.log 2>&1; echo "rc $?" >> gpurun_out/dbg_pipe_py.log
