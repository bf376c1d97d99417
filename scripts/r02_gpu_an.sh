#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/an_tests.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/an_bench.json 2> gpurun_out/an_bench.err
