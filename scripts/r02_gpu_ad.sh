#!/bin/bash
# K1 / K4 rewritten (one-wave grid-stride, streaming loads, W-templated convert): tests, per-kernel split, ncu times, traces
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/ad_tests.txt 2>&1
timeout 600 python scripts/ab_split.py k1k4 > gpurun_out/ad_split.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dash_(pre|dq)" -c 12 --csv \
  --log-file gpurun_out/ad_k1k4.csv python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu --no-e2e --no-gate > gpurun_out/ad_k1k4.log 2>&1
for cfg in "512 128 shift" "2048 128 shift" "4096 128 shift" "8192 128 descending" "16384 128 descending"; do
  set -- $cfg
  timeout 300 python scripts/trace_pipeline.py --seqlen $1 --head-dim $2 --schedule $3 \
    --out gpurun_out/ac_trace_$1_$2_$3.json --npz gpurun_out/ac_trace_$1_$2_$3.npz > /dev/null 2>&1
done
