#!/bin/bash
# fused dQ finalise v3 (16384-element tasks, mode policy): tests + A/B against K4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused_dq.py tests/test_gpu_chunk.py -x -q > gpurun_out/at_fused_tests.txt 2>&1 || exit 1
timeout 900 python scripts/ab_points.py fz --fused 2,0 --total --rounds 3 --scheds auto --d 64 > gpurun_out/at_points_c64.json 2>&1
timeout 900 python scripts/ab_points.py fz --fused 2,0 --total --rounds 3 --scheds auto --d 64 --masks full > gpurun_out/at_points_f64.json 2>&1
timeout 900 python scripts/ab_points.py fz --fused 2,0 --total --rounds 3 --scheds auto > gpurun_out/at_points_c128.json 2>&1
for rep in 1 2 3; do
FUSED=0 timeout 600 python scripts/ab_split.py k4 >> gpurun_out/at_split.txt 2>&1
FUSED=1 timeout 600 python scripts/ab_split.py policy >> gpurun_out/at_split.txt 2>&1
FUSED=2 timeout 600 python scripts/ab_split.py fused >> gpurun_out/at_split.txt 2>&1
done
