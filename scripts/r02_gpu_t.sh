#!/bin/bash
# A/B: early claim for SHIFT (all / single-job heads) on the hd128 causal + full sweeps
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for rep in 1 2; do
for v in 0 1 2; do
  DASH_FORCE_PREFETCH=$v timeout 600 python scripts/ab_points.py pf$v --scheds shift,descending --masks causal,full >> gpurun_out/t_ab.txt 2>&1
done
done
