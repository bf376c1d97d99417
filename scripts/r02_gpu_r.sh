#!/bin/bash
# round 2: pipeline traces (raw stamps) for job-boundary and d=64 softmax analysis
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for cfg in "512 128 shift" "2048 128 shift" "16384 128 descending" "2048 64 shift" "16384 64 descending"; do
  set -- $cfg
  timeout 300 python scripts/trace_pipeline.py --seqlen $1 --head-dim $2 --schedule $3 \
    --out gpurun_out/r_trace_$1_$2_$3.json --npz gpurun_out/r_trace_$1_$2_$3.npz > /dev/null 2> gpurun_out/r_trace_$1_$2_$3.err
done
