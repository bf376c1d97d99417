#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 120 python scripts/trace_pipeline.py --seqlen 16384 --schedule descending --npz gpurun_out/k_desc16k.npz > gpurun_out/k_desc16k.json 2>&1
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --npz gpurun_out/k_shift2k.npz > gpurun_out/k_shift2k.json 2>&1
