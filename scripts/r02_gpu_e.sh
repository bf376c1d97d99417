#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 240 python scripts/pair_smoke.py > gpurun_out/e_pair_smoke.txt 2>&1
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift > gpurun_out/e_trace_pair.json 2>&1
DASH_PAIR_VARIANT=1 timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift > gpurun_out/e_trace_pair_v1.json 2>&1
timeout 120 python scripts/trace_pipeline.py --seqlen 2048 --schedule shift --atomic > gpurun_out/e_trace_pair_atomic.json 2>&1
timeout 200 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-gate > gpurun_out/e_bench_v0.json 2>&1
