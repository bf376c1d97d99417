#!/bin/bash
# K1 / K4 with FastDiv index maps vs the previous commit's library (64-bit divisions)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
V=paper_2601_21824_b200/variants/libdash_head.so
timeout 1200 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_fused_dq.py tests/test_gpu_chunk.py -x -q > gpurun_out/ax_tests.txt 2>&1 || exit 1
for rep in 1 2 3; do
DASH_LIB_PATH=$V FUSED=0 timeout 600 python scripts/ab_split.py head_k4 >> gpurun_out/ax_split.txt 2>&1
FUSED=0 timeout 600 python scripts/ab_split.py fastdiv_k4 >> gpurun_out/ax_split.txt 2>&1
done
