#!/bin/bash
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
N="ncu --set full --clock-control none --import-source on"
python scripts/profile_all.py > gpurun_out/plain_all.log 2>&1 && \
$N -k regex:"k_fp16_step|k_fp16_tma|k_identity|k_reduce_dense" -c 8 -o gpurun_out/ncu_a \
   python scripts/profile_all.py --only fp16_step,fp16_staged,identity > gpurun_out/ncu_a.log 2>&1 ; \
$N -k regex:"k_int8_ws" -c 8 -o gpurun_out/ncu_b \
   python scripts/profile_all.py --only fp8,e5m2,qsgd,int8_pull_split > gpurun_out/ncu_b.log 2>&1 ; \
$N -k regex:"k_exchange_flags|k_rs_push|k_rs_reduce|k_ag_pull|k_reduce_dense" -c 12 -o gpurun_out/ncu_c \
   python scripts/profile_all.py --only self > gpurun_out/ncu_c.log 2>&1
