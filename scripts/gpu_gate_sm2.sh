#!/bin/bash
# C5-shape fused gate (eval, E=16 / 8): two-CTAs-per-SM instance vs one CTA per SM.
cd $GRAFT_REPO_ROOT
for T in 4096 16384 65536 262144; do for v in 1 0; do
  echo "SM2=$v T=$T: $(MOE_B200_GATE_SM2=$v timeout 120 python scripts/micro/gate_stamps_c5.py 16 $T 1024 0 2>&1 | grep 'main loop\|span' | tr '\n' ' ')"
done; done
