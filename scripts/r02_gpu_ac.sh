#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for cfg in "512 128 shift" "2048 128 shift" "4096 128 shift" "8192 128 descending" "16384 128 descending"; do
  set -- $cfg
  timeout 300 python scripts/trace_pipeline.py --seqlen $1 --head-dim $2 --schedule $3 \
    --out gpurun_out/ac_trace_$1_$2_$3.json --npz gpurun_out/ac_trace_$1_$2_$3.npz > /dev/null 2>&1
done
