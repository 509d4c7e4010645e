#!/bin/bash
# 1 GPU: winners' residuals stored by the top-k stage pass — parity + bench.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_self.py tests/test_gpu_fullsize.py tests/test_gpu_topk_pipeline.py -q -x -k "topk or nonfinite or overflow or fallback or fullsize or two_stream" > gpurun_out/wis_tests.log 2>&1
echo "rc $?" >> gpurun_out/wis_tests.log
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 30 --method topk"
$B > gpurun_out/wis_topk1.log 2>&1
$B --density 0.1 > gpurun_out/wis_topk10.log 2>&1
$B --values f16 > gpurun_out/wis_topk1_f16.log 2>&1
$B --density 0.1 --values f16 > gpurun_out/wis_topk10_f16.log 2>&1
$B --density 0.1 --no-pipeline > gpurun_out/wis_topk10_nopipe.log 2>&1
