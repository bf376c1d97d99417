#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --atomic --npz gpurun_out/g_pair.npz > gpurun_out/g_trace.json 2>&1
