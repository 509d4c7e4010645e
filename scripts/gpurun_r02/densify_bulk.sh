#!/bin/bash
# 1 GPU: the sparse densify with one TMA bulk store per sub-tile — parity + bench.
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "topk" > gpurun_out/db_tests.log 2>&1
echo "rc $?" >> gpurun_out/db_tests.log
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 30 --method topk"
$B > gpurun_out/db_topk1.log 2>&1
$B --no-pipeline > gpurun_out/db_topk1_nopipe.log 2>&1
$B --density 0.001 > gpurun_out/db_topk01.log 2>&1
