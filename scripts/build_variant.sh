#!/bin/bash
# Build an A/B variant of libbq.so with extra nvcc defines:
#   scripts/build_variant.sh NAME "-DFOO -DBAR"   ->  _variants/libbq_NAME.so  (load with BQ_LIB=...)
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_1402_4073_b200/csrc
B=$CS/_build_$NAME
mkdir -p $B $ROOT/_variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in $(cd $CS && ls *.cu | sed "s/\.cu$//"); do
  /usr/local/cuda/bin/nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fvisibility=hidden -cudart static \
    --expt-relaxed-constexpr $DEFS -c $CS/$f.cu -o $B/$f.o 2> $B/$f.log &
done
wait
/usr/local/cuda/bin/nvcc $ARCH -shared -cudart static -o $ROOT/_variants/libbq_$NAME.so $B/*.o -ldl
echo $ROOT/_variants/libbq_$NAME.so
