#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_kernel -s 2 -c 1 \
  -o gpurun_out/ag_d64 python scripts/one_call.py 2048 64 1 shift 1 3 > gpurun_out/ag_d64.log 2>&1
