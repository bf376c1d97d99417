#!/bin/bash
# round 2: ncu launch list of the bench step, ncu --set full of the pair kernel
# (N = 16384 causal DESCENDING, the sweep's dominant point; N = 2048 SHIFT),
# compute-sanitizer racecheck / synccheck on small problems.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/l_launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --no-gate > gpurun_out/l_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_pair -s 2 -c 1 \
  -o gpurun_out/l_pair16k python scripts/one_call.py 16384 128 1 descending 1 3 > gpurun_out/l_pair16k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_pair -s 2 -c 1 \
  -o gpurun_out/l_pair2k python scripts/one_call.py 2048 128 1 shift 1 3 > gpurun_out/l_pair2k.log 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all python scripts/one_call.py 256 64 1 shift 1 1 1 1 > gpurun_out/l_racecheck_d64.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python scripts/one_call.py 256 64 1 shift 1 1 1 1 > gpurun_out/l_synccheck_d64.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all python scripts/one_call.py 512 128 1 shift 1 1 1 2 > gpurun_out/l_racecheck_pair.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python scripts/one_call.py 512 128 1 shift 1 1 1 2 > gpurun_out/l_synccheck_pair.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python scripts/one_call.py 512 128 1 shift 1 1 1 2 > gpurun_out/l_memcheck_pair.txt 2>&1
ls -la gpurun_out/ | grep " l_"
