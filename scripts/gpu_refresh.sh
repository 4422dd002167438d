#!/bin/bash
# On the GPU box: the full round refresh under one tag -- gpu tests, bench (+
# reference arm), sweeps (configs 1/3/4 + backward grid), launch list + ncu
# captures of the forward and backward kernels, §8(f) rows, config 5, and the
# per-kernel-family ncu table.  Tag $1.
TAG=${1:-rx}
OUT=gpurun_out
bash scripts/gpu_full.sh $TAG
timeout 400 python scripts/sweeps.py --only config4bwd --out $OUT/bwd_sweep_$TAG.json > $OUT/bwd_sweep_$TAG.txt 2>&1
timeout 400 python bench.py --workload config5 --steps 30 --warmup 3 > $OUT/config5_$TAG.json 2> $OUT/config5_$TAG.err
# (the all-kernels ncu capture is ~57 MB: run it in a separate call, gpurun returns <= 64 MiB)
echo refresh done
