#!/bin/bash
# single-CTA softmax: 16-column chunks, TMEM loads pipelined one chunk ahead
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -x -q > gpurun_out/af_tests.txt 2>&1
timeout 900 python scripts/ab_points.py smx16_d64 --d 64 --scheds shift,descending --masks causal,full >> gpurun_out/af_ab.txt 2>&1
timeout 900 python scripts/ab_points.py smx16_d128single --scheds shift,descending --masks causal,full --tiles 128 --seqlens 512,1024,2048,4096 >> gpurun_out/af_ab.txt 2>&1
timeout 300 python scripts/trace_pipeline.py --seqlen 2048 --head-dim 64 --schedule shift --out gpurun_out/af_trace_2048_64.json > /dev/null 2>&1
