#!/bin/bash
# W (interleaved accumulators) re-measured on the current kernels, whole call (K1 + K2 + K4)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python scripts/ab_points.py W_causal --scheds descending,shift --masks causal --seqlens 4096,8192,16384 --splits 1,2,4,8 --rounds 3 --total > gpurun_out/aj_ab.txt 2>&1
timeout 1800 python scripts/ab_points.py W_full --scheds naive,shift --masks full --seqlens 4096,8192,16384 --splits 1,2,4,8 --rounds 3 --total >> gpurun_out/aj_ab.txt 2>&1
timeout 1800 python scripts/ab_points.py W_causal_short --scheds shift --masks causal,full --seqlens 512,1024,2048 --splits 1,2,4 --rounds 3 --total >> gpurun_out/aj_ab.txt 2>&1
