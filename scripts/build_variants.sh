#!/bin/bash
# Build libmoe_b200.so variants of one source file with extra -D switches:
#   build_variants.sh <file.cu> name:"-DX=1 -DY=2" ...   -> build/variants/<name>/libmoe_b200.so
set -e
src=$1; shift
cd "$(dirname "$0")/../paper_2109_10465_b200/csrc"
OBJ=../../build/obj
base=$(basename $src .cu)
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  d=../../build/variants/$name; mkdir -p $d
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $defs -c $src -o $d/$base.o
  objs=$(ls $OBJ/*.o | grep -v "/$base.o\$")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libmoe_b200.so $objs $d/$base.o -lnccl -lcuda
done
