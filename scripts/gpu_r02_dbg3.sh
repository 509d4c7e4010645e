#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
NEBULA_EXPERIMENT_WIDE_MIN=32768 timeout 300 python scripts/dbg_topk_pipe.py 0.1 > gpurun_out/dbg3_w32768.log 2>&1
NEBULA_EXPERIMENT_WIDE_MIN=32768 CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/dbg_topk_pipe.py 0.1 > gpurun_out/dbg3_w32768_blocking.log 2>&1
timeout 300 python scripts/dbg_topk_pipe.py 0.1 > gpurun_out/dbg3_default.log 2>&1
NEBULA_EXPERIMENT_WIDE_MIN=32768 timeout 300 python scripts/dbg_topk_pipe.py 0.05 > gpurun_out/dbg3_w32768_5.log 2>&1
