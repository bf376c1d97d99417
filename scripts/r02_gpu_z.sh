#!/bin/bash
# single-CTA kernel TMA-store epilogue: GPU tests + d64 per-point timings
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/z_tests.txt 2>&1
timeout 900 python scripts/ab_points.py epi_d64 --d 64 --scheds shift,descending,naive --masks causal,full >> gpurun_out/z_ab.txt 2>&1
DASH_TILE=128 timeout 900 python scripts/ab_points.py epi_d128_tile128 --scheds shift,descending --masks causal >> gpurun_out/z_ab.txt 2>&1
