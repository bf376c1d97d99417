#!/bin/bash
# TMA-store epilogue + early-claim policy: GPU tests, bench (hd128 causal headline + gates)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/y_tests.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/y_bench.json 2> gpurun_out/y_bench.err
