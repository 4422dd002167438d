#!/bin/bash
# Build a profiling variant of libdfa.so with extra -D knobs:
#   scripts/build_variant.sh NAME "-DDFA_POLY_MASK=0xA5A5u ..." [SOURCE.cu, default dfa_sm100.cu]
# -> scripts/variants/libdfa_NAME.so (same sources; timed by scripts/variants.py)
set -e
NAME=$1; DEFS=$2; SRC=${3:-dfa_sm100.cu}
HERE=$(cd $(dirname $0)/.. && pwd)
C=$HERE/paper_2403_09195_b200/csrc
OUT=$HERE/scripts/variants
mkdir -p $OUT/build_$NAME
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr $DEFS"
nvcc $FL -c $C/$SRC -o $OUT/build_$NAME/variant.o
OTHERS=$(ls $C/build/*.o | grep -v "/$SRC.o")
nvcc $ARCH -shared -o $OUT/libdfa_$NAME.so $OTHERS $OUT/build_$NAME/variant.o -lcudart_static -lrt -ldl -lpthread
echo built $OUT/libdfa_$NAME.so
