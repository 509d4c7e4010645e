#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
B="timeout 300 python bench.py --no-cpu --no-e2e --steps 30 --no-ef"
for L in 2 3 4 6; do NEBULA_DEBUG_NOEF_LEAD=$L $B > gpurun_out/lead_noef_$L.log 2>&1; done
for L in 3 4; do NEBULA_DEBUG_NOEF_LEAD=$L $B --method fp8 > gpurun_out/lead_noef_fp8_$L.log 2>&1; done
