#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_bwd.py -x -q -k watchdog > gpurun_out/h_watchdog.txt 2>&1
echo "watchdog rc=$?" >> gpurun_out/h_watchdog.txt
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/h_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/h_pytest.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
tail -3 gpurun_out/h_watchdog.txt gpurun_out/h_pytest.txt
