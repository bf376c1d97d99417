#!/bin/bash
# A/B on one box: HEAD~ (claim after KV_EMPTY) vs working tree (claim after the last load), bench sweep twice each
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for rep in 1 2; do
DASH_LIB_PATH=paper_2601_21824_b200/variants/libdash_prev.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-gate --no-sweep > gpurun_out/ao_prev_$rep.json 2>/dev/null
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-gate --no-sweep > gpurun_out/ao_new_$rep.json 2>/dev/null
done
