#!/bin/bash
# K1 rows per thread: 2 vs 4 (all loads in flight)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
DASH_K1_ROWS=4 timeout 1200 python -m pytest tests/test_gpu_bwd.py -x -q -k "matches_oracle" > gpurun_out/ay_tests.txt 2>&1 || exit 1
for rep in 1 2 3; do
DASH_K1_ROWS=2 FUSED=0 timeout 600 python scripts/ab_split.py k1r2 >> gpurun_out/ay_split.txt 2>&1
DASH_K1_ROWS=4 FUSED=0 timeout 600 python scripts/ab_split.py k1r4 >> gpurun_out/ay_split.txt 2>&1
done
