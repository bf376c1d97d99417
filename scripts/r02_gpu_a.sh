#!/bin/bash
# round 2, call A: microbenchmarks (TMEM ld/st, MUFU vs poly exp2) + baseline bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 300 python scripts/tmem_rate.py > gpurun_out/a_tmem_rate.txt 2>&1
timeout 300 python scripts/mma_rate.py > gpurun_out/a_mma_rate.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
tail -3 gpurun_out/a_tmem_rate.txt
