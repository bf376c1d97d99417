#!/bin/bash
# round 2, call B: validate the cleaned-up library (watchdog first, bounded), GPU tests, bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_bwd.py -x -q -k watchdog > gpurun_out/b_watchdog.txt 2>&1
echo "watchdog rc=$?" >> gpurun_out/b_watchdog.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/b_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/b_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
tail -3 gpurun_out/b_watchdog.txt gpurun_out/b_pytest.txt
