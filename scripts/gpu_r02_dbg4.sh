#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
DBG_STEPS=6 NEBULA_EXPERIMENT_WIDE_MIN=32768 timeout 300 python scripts/dbg_topk_pipe.py 0.1 > gpurun_out/dbg4_w32768.log 2>&1
DBG_STEPS=6 timeout 300 python scripts/dbg_topk_pipe.py 0.1 > gpurun_out/dbg4_default.log 2>&1
DBG_STEPS=6 NEBULA_EXPERIMENT_WIDE_MIN=32768 CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/dbg_topk_pipe.py 0.1 > gpurun_out/dbg4_w32768_blocking.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_division.py -q -x -k "int8 or fp8 or qsgd or e5m2 or division or dense or pull_reducer" > gpurun_out/dbg4_int8_tests.log 2>&1; echo "rc $?" >> gpurun_out/dbg4_int8_tests.log
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 30"
$B --method int8 > gpurun_out/dbg4_int8.log 2>&1
$B --method int8 --no-ef > gpurun_out/dbg4_int8_noef.log 2>&1
$B --method qsgd > gpurun_out/dbg4_qsgd.log 2>&1
