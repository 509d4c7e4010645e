#!/bin/bash
# ncu of the default dense-codec kernels (not the SELF P2P cases: ncu serialises kernels, and a
# member's flag kernel would wait for a peer's that cannot run meanwhile).  Summaries only are
# kept (the .ncu-rep files stay on the box: gpurun_out must stay under 64 MiB).
python -m paper_2205_09470_b200.build > gpurun_out/build.log 2>&1
N="ncu --set full --clock-control none --import-source on"
python scripts/profile_all.py --only fp16_step,fp16_staged,identity,fp8,e5m2,qsgd,int8_pull_split > gpurun_out/plain_all.log 2>&1 && \
timeout 1200 $N -k regex:"k_fp16_step|k_fp16_tma|k_identity|k_reduce_dense" -c 6 -o /tmp/ncu_a \
   python scripts/profile_all.py --only fp16_step,fp16_staged,identity > gpurun_out/ncu_a.log 2>&1 ; \
timeout 1200 $N -k regex:"k_int8_ws" -c 8 -o /tmp/ncu_b \
   python scripts/profile_all.py --only fp8,e5m2,qsgd,int8_pull_split > gpurun_out/ncu_b.log 2>&1 ; \
python scripts/ncu_summary.py /tmp/ncu_a.ncu-rep > gpurun_out/ncu_a_summary.txt 2>&1
python scripts/ncu_summary.py /tmp/ncu_b.ncu-rep > gpurun_out/ncu_b_summary.txt 2>&1
