#!/bin/bash
# poly-exp2 A/B: fraction of softmax exponentials on the FMA pipe
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
V=paper_2601_21824_b200/variants
DASH_LIB_PATH=$V/libdash_p3.so timeout 900 python -m pytest tests/test_gpu_bwd.py -x -q -k "backward_matches_oracle or peaky" > gpurun_out/ah_tests_p3.txt 2>&1
for rep in 1 2; do
for v in base p4 p3 p2; do
  if [ $v = base ]; then L=""; else L="$V/libdash_$v.so"; fi
  DASH_LIB_PATH=$L timeout 900 python scripts/ab_points.py $v --d 64 --scheds shift --masks causal,full --seqlens 1024,4096,16384 >> gpurun_out/ah_ab.txt 2>&1
  DASH_LIB_PATH=$L timeout 900 python scripts/ab_points.py ${v}_d128 --scheds auto --masks causal --seqlens 1024,4096,16384 >> gpurun_out/ah_ab.txt 2>&1
done
done
