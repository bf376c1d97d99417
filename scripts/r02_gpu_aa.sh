#!/bin/bash
# tile 128 (single-CTA) vs 256 (pair) at d = 128, interleaved rounds
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python scripts/ab_points.py tiles --scheds shift,descending,naive --masks causal,full --tiles 256,128 --rounds 3 > gpurun_out/aa_ab.txt 2>&1
