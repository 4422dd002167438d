#!/bin/bash
# Fused multi-branch kernel: parity tests + timing of the LongNet set.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multibranch_fused.py tests/test_full_batch_parity.py -k "multibranch or fused" -x -q -p no:cacheprovider --timeout 300 2>&1 | tail -25
timeout 300 python scripts/micro/mb_once.py 2>&1 | tail -20
timeout 300 python scripts/micro/mb_time.py 2>&1 | tail -8
