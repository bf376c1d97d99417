#!/bin/bash
# early-claim point A/B: 0 = all MMAs of the job complete, 1 = K/V free (pair), 2 = loads issued
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for rep in 1 2; do
for v in 0 1 2; do
DASH_CLAIM_AT=$v timeout 900 python scripts/ab_points.py claim$v --scheds auto,shift,descending --masks causal,full >> gpurun_out/am_ab.txt 2>&1
DASH_CLAIM_AT=$v timeout 900 python scripts/ab_points.py claim${v}_d64 --d 64 --scheds shift,descending --masks causal,full --seqlens 1024,4096,16384 >> gpurun_out/am_ab.txt 2>&1
done
done
