#!/bin/bash
# compute-sanitizer --tool memcheck over every default kernel (one tool per gpurun call)
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
python tests/sanitize_workload.py  > gpurun_out/san_plain_memcheck.log 2>&1 && \
timeout 2400 compute-sanitizer --tool memcheck --print-limit 50 python tests/sanitize_workload.py  > gpurun_out/san_memcheck.log 2>&1
echo "sanitizer rc $?" >> gpurun_out/san_memcheck.log
