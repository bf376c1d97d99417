#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/d_bench_pair.json 2> gpurun_out/d_bench_pair.err
DASH_TILE=128 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-gate > gpurun_out/d_bench_tile128.json 2> gpurun_out/d_bench_tile128.err
tail -2 gpurun_out/d_bench_pair.err
