#!/bin/bash
# ncu --set full of the backward (config 2) and the fused multi-branch kernel (LongNet set, B = 64), one launch each.
TAG=${1:-r02k}
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dfa_bwd_sm100_kernel -s 2 -c 1 -f -o gpurun_out/ncu_bwd_$TAG python scripts/micro/bwd_once.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dfa_mb_sm100_kernel -s 2 -c 1 -f -o gpurun_out/ncu_mb_$TAG python scripts/micro/mb_once.py > /dev/null 2>&1
ls -la gpurun_out/ncu_*_$TAG.ncu-rep
