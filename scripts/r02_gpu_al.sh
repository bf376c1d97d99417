#!/bin/bash
# segment ends from a table (no chained task scan in the producer / MMA warps)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py tests/test_gpu_chunk.py -x -q > gpurun_out/al_tests.txt 2>&1
timeout 900 python scripts/ab_points.py segend --scheds auto,shift,descending --masks causal,full >> gpurun_out/al_ab.txt 2>&1
timeout 900 python scripts/ab_points.py segend_d64 --d 64 --scheds shift --masks causal,full >> gpurun_out/al_ab.txt 2>&1
timeout 300 python scripts/trace_pipeline.py --seqlen 4096 --head-dim 128 --schedule shift --npz gpurun_out/al_trace_4096.npz > /dev/null 2>&1
