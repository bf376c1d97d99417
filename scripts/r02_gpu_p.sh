#!/bin/bash
# round 2: per-thread L/D release in the pair kernel -> racecheck, DRAM bytes over the
# bench sweep (-s 0), GPU tests, full bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu --no-e2e --no-gate"
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all python scripts/one_call.py 512 128 1 shift 1 1 1 2 > gpurun_out/p_racecheck_pair.txt 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dash_bwd -s 0 -c 6 --csv \
  --log-file gpurun_out/p_dram.csv $B > gpurun_out/p_dram.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p_tests.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
