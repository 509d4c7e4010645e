#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
CMD="python scripts/profile_all.py"
$CMD > gpurun_out/plain_all.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fp16_step|k_fp16_tma|k_identity|k_int8_ws|k_reduce_dense|k_exchange_flags|k_rs_push|k_rs_reduce|k_ag_pull" -c 40 -o gpurun_out/all_kernels $CMD > gpurun_out/ncu_all.log 2>&1
