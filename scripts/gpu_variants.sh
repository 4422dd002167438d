#!/bin/bash
# A/B timing of variant builds (scripts/variants/*.so), interleaved 3 times.
CASES=${CASES:-512:2,512:1,1024:2,2048:1,4096:4,256:8}
V=$(ls scripts/variants/libdfa_*.so)
for rep in 1 2 3; do timeout 600 python scripts/variants.py $V --cases $CASES; done
