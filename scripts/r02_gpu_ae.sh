#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_replay.py -x -q > gpurun_out/ae_tests.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"dash_(pre|dq)" -c 12 --csv \
  --log-file gpurun_out/ae_k1k4.csv python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu --no-e2e --no-gate > gpurun_out/ae_k1k4.log 2>&1
