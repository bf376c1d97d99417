#!/bin/bash
# early claim without the CAS loop: A/B all schedules, both kernels, d=128 and d=64
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for v in 0 1; do
DASH_FORCE_PREFETCH=$v timeout 900 python scripts/ab_points.py pf$v --scheds shift,descending,naive --masks causal,full >> gpurun_out/x_ab.txt 2>&1
DASH_FORCE_PREFETCH=$v timeout 900 python scripts/ab_points.py pf${v}_d64 --d 64 --scheds shift,descending,naive --masks causal,full >> gpurun_out/x_ab.txt 2>&1
done
DASH_FORCE_PREFETCH=1 timeout 300 python scripts/trace_pipeline.py --seqlen 512 --head-dim 128 --schedule shift --npz gpurun_out/x_trace_512_pf1.npz > /dev/null 2>&1
