#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for cfg in "512 128 shift" "2048 128 shift"; do
  set -- $cfg
  timeout 300 python scripts/trace_pipeline.py --seqlen $1 --head-dim $2 --schedule $3 \
    --npz gpurun_out/s_trace_$1_$2_$3.npz > /dev/null 2> gpurun_out/s_trace_$1_$2_$3.err
done
