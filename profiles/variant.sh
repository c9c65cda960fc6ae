#!/bin/bash
# Build the working tree's library with extra nvcc defines into ab/lib_<name>.so
# (A/B runs through TM_LIB):  profiles/variant.sh <name> "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/.."
name=${1:?name}; defs=${2:-}
B=ab/build_$name; mkdir -p $B
NVCC=/usr/local/cuda/bin/nvcc
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $defs"
objs=""
for f in paper_2204_09236_b200/csrc/*.cu; do
  o=$B/$(basename ${f%.cu}).o; objs="$objs $o"
  $NVCC $FLAGS -c -o $o $f &
done
wait
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o ab/lib_$name.so $objs -lcudart -lpthread
echo ab/lib_$name.so
