#!/bin/bash
# On the GPU box: gpu tests (-x), timeline traces, bench line (no ncu), config-4 sweep.  Tag $1.
TAG=${1:-rx}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 300 > gpurun_out/tests_$TAG.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$TAG.log
tail -4 gpurun_out/tests_$TAG.log
timeout 300 python scripts/trace_timeline.py run --w 512 --r 2 2>&1 | head -9
timeout 300 python scripts/trace_timeline.py run --w 2048 --r 1 2>&1 | head -9
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('ms', d['roofline']['kernel_ms'], 'GB/s', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'],3), 'TF', round(d['tflops']), d['clocks'])"
timeout 600 python scripts/sweeps.py --only config4 --out gpurun_out/sweeps_$TAG.json 2>&1 | tail -22
