#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for X in 0 1 2 3 4 7; do
DASH_XDBG=$X timeout 120 python scripts/trace_pipeline.py --seqlen 16384 --schedule descending --atomic > gpurun_out/n_x$X.json 2>&1
done
