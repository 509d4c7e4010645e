#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --deselect tests/test_multigpu.py > gpurun_out/gpu_tests_i.log 2>&1
echo "suite rc $?" >> gpurun_out/gpu_tests_i.log
for m in int8 qsgd fp8 fp8e5m2 fp16 identity; do
  timeout 300 python bench.py --method $m --no-cpu --no-e2e --steps 100 > gpurun_out/bench_i_$m.log 2>&1
done
timeout 300 python bench.py --method int8 --no-ef --no-cpu --no-e2e --steps 100 > gpurun_out/bench_i_int8_noef.log 2>&1
