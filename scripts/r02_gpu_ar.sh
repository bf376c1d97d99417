#!/bin/bash
# packed-fp32 (FFMA2/FADD2/FMUL2) softmax: GPU tests + A/B against the previous commit's library
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
V=paper_2601_21824_b200/variants/libdash_head.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/au_tests.txt 2>&1 || exit 1
for rep in 1 2; do
for lib in new head; do
  if [ $lib = head ]; then export DASH_LIB_PATH=$V; else unset DASH_LIB_PATH; fi
  timeout 900 python scripts/ab_points.py $lib --rounds 1 --reps 20 --d 64 --masks causal,full >> gpurun_out/au_points_d64.txt 2>&1
  timeout 900 python scripts/ab_points.py $lib --rounds 1 --reps 20 --masks causal,full >> gpurun_out/au_points_d128.txt 2>&1
  timeout 600 python scripts/ab_split.py $lib >> gpurun_out/au_split.txt 2>&1
done
done
unset DASH_LIB_PATH
