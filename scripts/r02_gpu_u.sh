#!/bin/bash
# pair kernel: TMA-store dK/dV epilogue -> parity, per-point A/B, trace
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_bwd.py tests/test_gpu_chunk.py -x -q > gpurun_out/u_tests.txt 2>&1
for v in 0 2; do
DASH_FORCE_PREFETCH=$v timeout 600 python scripts/ab_points.py epi_pf$v --scheds auto,shift,descending --masks causal,full >> gpurun_out/u_ab.txt 2>&1
done
timeout 300 python scripts/trace_pipeline.py --seqlen 512 --head-dim 128 --schedule shift --npz gpurun_out/u_trace_512.npz > /dev/null 2>&1
