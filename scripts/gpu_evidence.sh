#!/bin/bash
# Evidence at HEAD on one B200 (run under gpurun): GPU tests, smoke, bench line, reference arm,
# ncu launch list, DRAM bytes per main-kernel launch, ncu --set full of both main kernels.
#   gpurun --timeout 3000 -- 'bash scripts/gpu_evidence.sh TAG'   -> gpurun_out/TAG_*
T=${1:-ev}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
B="python bench.py --steps 1 --warmup 0 --no-sweep --no-cpu --no-e2e --no-gate"
# each ncu command line runs once without ncu first (it must exit 0)
timeout 600 python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --no-gate > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --no-gate > gpurun_out/${T}_launches.log 2>&1
timeout 600 $B > /dev/null 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dash_bwd -s 0 -c 6 --csv \
  --log-file gpurun_out/${T}_dram.csv $B > gpurun_out/${T}_dram.log 2>&1
timeout 300 python scripts/one_call.py 16384 128 1 descending 1 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_pair -s 2 -c 1 \
  -o gpurun_out/${T}_pair16k python scripts/one_call.py 16384 128 1 descending 1 3 > gpurun_out/${T}_pair16k.log 2>&1
timeout 300 python scripts/one_call.py 2048 128 1 shift 1 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dash_bwd_kernel -s 2 -c 1 \
  -o gpurun_out/${T}_single2k python scripts/one_call.py 2048 128 1 shift 1 3 > gpurun_out/${T}_single2k.log 2>&1
echo done > gpurun_out/${T}_done.txt
