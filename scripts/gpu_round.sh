#!/bin/bash
# On the GPU box: gpu tests, then bench + launch list + ncu full capture (tag $1).
TAG=${1:-rx}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 300 > gpurun_out/tests_$TAG.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests_$TAG.log
tail -5 gpurun_out/tests_$TAG.log
timeout 600 bash scripts/gpu_bench_profile.sh $TAG
cat gpurun_out/bench_$TAG.json
