#!/bin/bash
# On the GPU box: all gpu tests, bench (+ reference arm), sweeps, launch list,
# ncu full capture of the attention kernel, ncu per-branch metrics.  Tag $1.
TAG=${1:-rx}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > $OUT/tests_$TAG.log 2>&1
echo "tests rc=$?" >> $OUT/tests_$TAG.log; tail -3 $OUT/tests_$TAG.log
timeout 300 python bench.py --steps 50 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_$TAG.json 2>> $OUT/bench_$TAG.err
timeout 600 python scripts/sweeps.py --out $OUT/sweeps_$TAG.json > $OUT/sweeps_$TAG.txt 2>&1; tail -40 $OUT/sweeps_$TAG.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 10 --warmup 3 --quick > $OUT/ncu_launch_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dfa_sm100 -s 5 -c 1 -o $OUT/prof_$TAG -f \
    python bench.py --steps 3 --warmup 3 --quick > $OUT/ncu_full_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:dfa_sm100 --csv --log-file $OUT/ncu_sweep_$TAG.csv python scripts/sweeps.py --ncu > $OUT/ncu_sweep_$TAG.log 2>&1
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print('ms', d['roofline']['kernel_ms'], 'GB/s', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'],3), 'TF', round(d['tflops']), d['clocks'])"
ls $OUT | tail -20
timeout 300 python scripts/measure_next.py --out $OUT/next_$TAG.json > $OUT/next_$TAG.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/bwd_launches_$TAG.csv python scripts/measure_next.py --only backward > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dfa_bwd_sm100 -s 2 -c 1 -o $OUT/prof_bwd_$TAG -f python scripts/measure_next.py --only backward > $OUT/ncu_bwd_$TAG.log 2>&1
python -c "import json; d=json.load(open('$OUT/next_$TAG.json')); print({k: (round(v['ms'],3) if isinstance(v, dict) else v) for k, v in d.items()})"
