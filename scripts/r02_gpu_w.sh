#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
DASH_FORCE_PREFETCH=2 timeout 300 python scripts/trace_pipeline.py --seqlen 512 --head-dim 128 --schedule shift --npz gpurun_out/w_trace_512_pf2.npz > /dev/null 2>&1
