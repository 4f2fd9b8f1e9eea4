#!/bin/bash
# Build libmoe_b200.so variants of rng.cu (MOE_RNG_* switches) under build/variants/<name>/.
set -e
cd "$(dirname "$0")/../paper_2109_10465_b200/csrc"
OBJ=../../build/obj
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  d=../../build/variants/$name; mkdir -p $d
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $defs -c rng.cu -o $d/rng.o
  objs=$(ls $OBJ/*.o | grep -v '/rng.o$')
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libmoe_b200.so $objs $d/rng.o -lnccl -lcuda
done
