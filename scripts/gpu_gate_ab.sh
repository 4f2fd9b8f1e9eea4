#!/bin/bash
# Fused-gate main-loop A/B: gate_stamps_c5 for the in-tree lib and build/variants/<name>.
cd $GRAFT_REPO_ROOT
for v in cur "$@"; do
  if [ $v = cur ]; then unset MOE_B200_LIB; else export MOE_B200_LIB=$PWD/build/variants/$v/libmoe_b200.so; fi
  for a in "64 8192 2048 1" "64 8192 2048 0" "16 65536 1024 0"; do
    echo "== $v $a: $(timeout 120 python scripts/micro/gate_stamps_c5.py $a 2>&1 | grep 'main loop\|span' | tr '\n' ' ')"
  done
done
