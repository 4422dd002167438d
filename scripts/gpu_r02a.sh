#!/bin/bash
# Round-2 first pass on the GPU box: GPU tests, bench (both arms), MUFU / XU
# micro-benchmarks, launch list, ncu full capture of the forward.  Tag $1.
TAG=${1:-r02a}
OUT=gpurun_out
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_bench scripts/micro/mufu_bench.cu && /tmp/mufu_bench > $OUT/mufu_$TAG.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/xu_bench scripts/micro/xu_bench.cu && /tmp/xu_bench > $OUT/xu_$TAG.txt 2>&1
cat $OUT/mufu_$TAG.txt $OUT/xu_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > $OUT/tests_$TAG.log 2>&1
echo "tests rc=$?" >> $OUT/tests_$TAG.log; tail -5 $OUT/tests_$TAG.log
timeout 600 bash scripts/gpu_bench_profile.sh $TAG > /dev/null 2>&1
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print('ms', d['roofline']['kernel_ms'], 'frac', round(d['roofline']['frac'],3), 'e2e', d['e2e']['value'], d['clocks']); print(json.dumps(d.get('extras',{}))[:3000])"
head -c 600 $OUT/bench_ref_$TAG.json
