#!/bin/bash
# round-2 evidence at HEAD: GPU tests, bench, ncu launch list, DRAM per main-kernel launch, ncu --set full of both kernels
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/ak_tests.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/ak_bench.json 2> gpurun_out/ak_bench.err
B="python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu --no-e2e --no-gate"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/ak_launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --no-gate > gpurun_out/ak_launches.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dash_bwd -s 0 -c 6 --csv \
  --log-file gpurun_out/ak_dram.csv $B > gpurun_out/ak_dram.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_pair -s 2 -c 1 \
  -o gpurun_out/ak_pair16k python scripts/one_call.py 16384 128 1 descending 1 3 > gpurun_out/ak_pair16k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_kernel -s 2 -c 1 \
  -o gpurun_out/ak_single2k python scripts/one_call.py 2048 128 1 shift 1 3 > gpurun_out/ak_single2k.log 2>&1
