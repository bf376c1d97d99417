#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for W in 1 2 4 8; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-gate --acc-split $W > gpurun_out/j_bench_w$W.json 2> gpurun_out/j_bench_w$W.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-gate --full --acc-split $W > gpurun_out/j_bench_full_w$W.json 2> gpurun_out/j_bench_full_w$W.err
done
