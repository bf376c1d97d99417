#!/bin/bash
# d = 64: four softmax warpgroups that also drain dQ (640 threads)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -x -q > gpurun_out/ai_tests.txt 2>&1
timeout 900 python scripts/ab_points.py smx4wg_d64 --d 64 --scheds shift,descending,naive --masks causal,full >> gpurun_out/ai_ab.txt 2>&1
timeout 300 python scripts/trace_pipeline.py --seqlen 2048 --head-dim 64 --schedule shift --out gpurun_out/ai_trace_2048_64.json > /dev/null 2>&1
