#!/bin/bash
# round 2 evidence at HEAD: launch list, per-launch DRAM bytes of the main kernel
# over the bench sweep, ncu --set full of the pair kernel, pair-MMA rates, sanitizers
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu --no-e2e --no-gate"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/o_launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --no-gate > gpurun_out/o_launches.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:dash_bwd -s 6 -c 6 --csv \
  --log-file gpurun_out/o_dram.csv $B > gpurun_out/o_dram.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_pair -s 2 -c 1 \
  -o gpurun_out/o_pair16k python scripts/one_call.py 16384 128 1 descending 1 3 > gpurun_out/o_pair16k.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_pair -s 2 -c 1 \
  -o gpurun_out/o_pair2k python scripts/one_call.py 2048 128 1 shift 1 3 > gpurun_out/o_pair2k.log 2>&1
timeout 300 python scripts/pair_mma_rate.py > gpurun_out/o_pair_mma_rate.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all python scripts/one_call.py 512 128 1 shift 1 1 1 2 > gpurun_out/o_racecheck_pair.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python scripts/one_call.py 512 128 1 shift 1 1 1 2 > gpurun_out/o_synccheck_pair.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python scripts/one_call.py 512 128 1 shift 1 1 1 2 > gpurun_out/o_memcheck_pair.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all python scripts/one_call.py 256 64 1 shift 1 1 1 1 > gpurun_out/o_racecheck_d64.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python scripts/one_call.py 256 64 1 shift 1 1 1 1 > gpurun_out/o_synccheck_d64.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python scripts/one_call.py 256 64 1 shift 1 1 1 1 > gpurun_out/o_memcheck_d64.txt 2>&1
