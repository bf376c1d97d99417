#!/bin/bash
# Experiment: W = 4 vs W = 8 interleaved dQ accumulators at long context and N = 16k.
set -x
for W in 4 8; do
  DASH_ACC_SPLIT=$W timeout 600 python scripts/long_context.py --reps 2 > gpurun_out/w8_lc_W$W.json 2>&1
done
for W in 4 8; do
  DASH_ACC_SPLIT=$W timeout 300 python -m pytest tests/test_gpu_bwd.py -x -q -k "replay or determin" > gpurun_out/w8_tests_W$W.log 2>&1
done
for W in 4 8; do
  timeout 300 python bench.py --acc-split $W --seqlens 8192,16384 --no-cpu --no-e2e --steps 5 > gpurun_out/w8_bench_W$W.json 2>gpurun_out/w8_bench_W$W.err
done
