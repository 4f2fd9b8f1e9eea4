#!/bin/bash
# C5-shape fused gate span: in-tree lib vs build/variants/<name> (eval, E=16, d=1024).
cd $GRAFT_REPO_ROOT
for v in cur "$@"; do
  if [ $v = cur ]; then unset MOE_B200_LIB; else export MOE_B200_LIB=$PWD/build/variants/$v/libmoe_b200.so; fi
  for T in 16384 65536 262144; do
    echo "$v T=$T: $(timeout 120 python scripts/micro/gate_stamps_c5.py 16 $T 1024 0 2>&1 | grep 'main loop\|span' | tr '\n' ' ')"
  done
done
