#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
CMD="python scripts/profile_step.py --method topk --density 0.1 --steps 2"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_topk_(merge|move|resolve|densify|stage|scan|write|splits|sample|bracket)" -s 10 -c 12 -o gpurun_out/topk10 $CMD > gpurun_out/ncu_topk10.log 2>&1
