#!/bin/bash
# ncu captures of the fused multi-branch kernel (LongNet set) per variant lib.
mkdir -p gpurun_out
for L in scripts/variants/libdfa_*.so; do n=$(basename $L .so)
DFA_LIB_VARIANT=$PWD/$L timeout 300 ncu --set full --clock-control none --import-source on -k regex:dfa_mb -s 2 -c 1 -o gpurun_out/prof_mb_$n -f python scripts/micro/mb_once.py > gpurun_out/prof_mb_$n.log 2>&1
done
DFA_LIB_VARIANT=$PWD/scripts/variants/libdfa_ord0.so timeout 300 ncu --set full --clock-control none -k regex:dfa_sm100 -s 4 -c 1 -o gpurun_out/prof_mb_single512 -f python scripts/micro/mb_once.py > /dev/null 2>&1
ls gpurun_out | grep prof_mb
