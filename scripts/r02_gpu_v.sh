#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
DASH_FORCE_PREFETCH=2 timeout 300 python scripts/trace_pipeline.py --seqlen 512 --head-dim 128 --schedule shift --npz gpurun_out/v_trace_512_pf2.npz > /dev/null 2>&1
DASH_FORCE_PREFETCH=0 timeout 300 python scripts/trace_pipeline.py --seqlen 512 --head-dim 128 --schedule descending --npz gpurun_out/v_trace_512_desc.npz > /dev/null 2>&1
DASH_FORCE_PREFETCH=1 timeout 300 python scripts/trace_pipeline.py --seqlen 512 --head-dim 128 --schedule descending --npz gpurun_out/v_trace_512_desc_pf1.npz > /dev/null 2>&1
