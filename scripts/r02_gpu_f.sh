#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --npz gpurun_out/f_pair.npz > gpurun_out/f_trace_pair.json 2>&1
DASH_TILE=128 timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --npz gpurun_out/f_1cta.npz > gpurun_out/f_trace_1cta.json 2>&1
