#!/bin/bash
# Round-2 profile refresh: per-branch ncu metrics over the config-4 grid, the
# fused multi-branch kernel (LongNet set), launch list of the default bench.
OUT=gpurun_out; mkdir -p $OUT
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none -k regex:dfa_sm100 --csv --log-file $OUT/r02_ncu_sweep.csv python scripts/sweeps.py --ncu > $OUT/r02_ncu_sweep.log 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:"dfa_mb|dfa_sm100" --csv --log-file $OUT/r02_ncu_mb.csv python scripts/micro/mb_once.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dfa_mb -s 2 -c 1 -o $OUT/r02_prof_mb -f python scripts/micro/mb_once.py > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/r02_launches.csv python bench.py --steps 10 --warmup 3 --quick > /dev/null 2>&1
ls -la $OUT | grep r02
