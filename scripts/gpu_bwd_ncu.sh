#!/bin/bash
# Stall-reason captures of the backward kernel for several library builds.
mkdir -p gpurun_out
for lib in "$@"; do
  n=$(basename $lib .so)
  DFA_LIB_VARIANT=$PWD/$lib timeout 600 ncu -k regex:dfa_bwd_sm100_kernel -s 2 -c 1 --clock-control none --import-source on \
    --section SourceCounters --section WarpStateStats --section SchedulerStats --section InstructionStats \
    -f -o gpurun_out/bwd_$n python scripts/micro/bwd_once.py > gpurun_out/bwd_$n.log 2>&1
  python scripts/ncu_stalls.py gpurun_out/bwd_$n.ncu-rep 12 > gpurun_out/bwd_${n}_stalls.txt 2>&1
  ncu -i gpurun_out/bwd_$n.ncu-rep --page raw --csv > gpurun_out/bwd_${n}_raw.csv 2>&1
done
