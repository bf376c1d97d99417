#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_bwd.py -x -q -k watchdog > gpurun_out/i_watchdog.txt 2>&1
echo "watchdog rc=$?" >> gpurun_out/i_watchdog.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-gate > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err
tail -2 gpurun_out/i_watchdog.txt
