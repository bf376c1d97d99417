#!/bin/bash
# compute-sanitizer on the final kernels (TMA-store epilogue, segment-end table, early claim)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 900 compute-sanitizer --tool $tool $extra python scripts/one_call.py 256 64 1 shift 1 1 1 1 > gpurun_out/ap_${tool}_d64.txt 2>&1
  DASH_TILE=128 timeout 900 compute-sanitizer --tool $tool $extra python scripts/one_call.py 512 128 1 shift 1 1 1 2 > gpurun_out/ap_${tool}_single128.txt 2>&1
  DASH_TILE=256 timeout 900 compute-sanitizer --tool $tool $extra python scripts/one_call.py 512 128 1 shift 1 1 1 2 > gpurun_out/ap_${tool}_pair.txt 2>&1
done
