#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 240 python scripts/pair_smoke.py > gpurun_out/e_pair_smoke.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_replay.py -x -q -k "pair or every_plane" > gpurun_out/m_replay.txt 2>&1
bash scripts/r02_gpu_k.sh
for V in 0 1; do DASH_PAIR_VARIANT=$V timeout 200 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-gate > gpurun_out/m_bench_v$V.json 2>&1; done
