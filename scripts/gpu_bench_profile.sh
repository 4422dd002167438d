#!/bin/bash
# Runs on the GPU box (via gpurun): bench line, launch list, one ncu --set full
# capture of the attention kernel.  Outputs under gpurun_out/ (tag = $1).
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt
python bench.py --steps 50 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_$TAG.json 2>> $OUT/bench_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 10 --warmup 3 --quick > $OUT/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dfa_sm100 -s 5 -c 1 -o $OUT/prof_$TAG -f \
    python bench.py --steps 3 --warmup 3 --quick > $OUT/ncu_full_$TAG.log 2>&1
ls -la $OUT
