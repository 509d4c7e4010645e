#!/bin/bash
# SASS evidence (no GPU needed): the default warp-specialised kernels issue TMA bulk copies
# (UBLKCP = cp.async.bulk) completing on shared-memory mbarriers (SYNCS.* = mbarrier ops).
# Usage: bash scripts/sass_evidence.sh > profiles/r02/sass_tma_mbarrier.txt
O=paper_2205_09470_b200/build
echo "# cuobjdump -sass of the in-tree objects (nvcc -gencode arch=compute_100a,code=sm_100a): per kernel, count of"
echo "# TMA bulk-copy (UBLKCP) and mbarrier (SYNCS.*) instructions, then excerpts."
for f in kernels_ws.o; do
  cuobjdump -sass $O/$f | awk '/Function : /{fn=$3} /UBLKCP|SYNCS/{split($0,a,";"); n=split(a[1],w," "); op=""; for(i=1;i<=n;i++) if (w[i] ~ /^(UBLKCP|SYNCS)/) op=w[i]; c[fn" "op]++} END{for(k in c) print c[k], k}' | sort -k2 | grep -E "k_int8_wsILb1ELi8ELi19ELi4ELi1ELi0ELb0E|k_int8_wsILb1ELi8ELi23ELi0ELi0ELi0ELb0E|k_fp16_tmaILb1E|k_fp16_stepILb1ELi23ELi8E|k_int8_wsILb1ELi4ELi16ELi11ELi2ELi0ELb0E"
done
echo
echo "# excerpt: k_int8_ws<EF=1, AW=8, BW=19, CW=4, CM=1> (the default INT8 fused step, LOOPBACK)"
cuobjdump -sass -fun '_ZN2nb9k_int8_wsILb1ELi8ELi19ELi4ELi1ELi0ELb0EEEvPKNS_4ItemEiPKfPfNS_5DestsEPjS8_S8_NS_8StepArgsE' $O/kernels_ws.o | grep -E "UBLKCP|TRYWAIT|ARRIVE" | head -16
echo
echo "# excerpt: k_fp16_tma<EF=1> (the default FP16 compressor)"
cuobjdump -sass -fun '_ZN2nb10k_fp16_tmaILb1EEEvPKNS_4ItemEimPKfPfNS_5DestsEPj' $O/kernels_ws.o | grep -E "UBLKCP|TRYWAIT|ARRIVE" | head -10
echo
echo "# k_topk_stage<EF=1, VEC=1, TMA=1> (the default top-k stage pass, round 2): counts, then excerpt"
cuobjdump -sass $O/kernels_topk.o | awk '/Function : /{fn=$3} /UBLKCP|SYNCS/{split($0,a,";"); n=split(a[1],w," "); op=""; for(i=1;i<=n;i++) if (w[i] ~ /^(UBLKCP|SYNCS)/) op=w[i]; c[fn" "op]++} END{for(k in c) print c[k], k}' | sort -k2 | grep -E "k_topk_stageILb1ELb1ELb1E"
cuobjdump -sass -fun '_ZN2nb12k_topk_stageILb1ELb1ELb1EEEvPKNS_4ItemEPKNS_8TopkItemEPNS_9TopkStateEimPKfPfPySC_P5uint2m' $O/kernels_topk.o | grep -E "UBLKCP|TRYWAIT|ARRIVE" | head -8
