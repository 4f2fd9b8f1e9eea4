#!/bin/bash
# gate dW on the side stream next to gate dx (MOE_B200_GATE_DW_SIDE) A/B, one GPU.
cd $GRAFT_REPO_ROOT
AB_VAR=MOE_B200_GATE_DW_SIDE PYTEST_K="bf16" bash scripts/gpu_ab.sh
