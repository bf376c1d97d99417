#!/bin/bash
# A/B of the working tree's libdash.so against paper_2601_21824_b200/variants/libdash_head.so
# (python scripts/build_variant.py head --rev HEAD): selected GPU tests, then interleaved per-point and
# whole-step timings.   gpurun -- 'bash scripts/gpu_ab.sh TAG "pytest -k args"'
T=${1:-ab}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
V=paper_2601_21824_b200/variants/libdash_head.so
if [ -n "$2" ]; then timeout 1500 python -m pytest tests -m gpu -x -q $2 > gpurun_out/${T}_tests.txt 2>&1 || exit 1; fi
for rep in 1 2; do
for lib in new head; do
  if [ $lib = head ]; then export DASH_LIB_PATH=$V; else unset DASH_LIB_PATH; fi
  timeout 900 python scripts/ab_points.py $lib --rounds 1 --reps 20 --masks causal,full >> gpurun_out/${T}_points_d128.txt 2>&1
  timeout 600 python scripts/ab_split.py $lib >> gpurun_out/${T}_split.txt 2>&1
done
done
unset DASH_LIB_PATH
