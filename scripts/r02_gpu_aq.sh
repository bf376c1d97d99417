#!/bin/bash
# programmatic dependent launch K1 -> K2 -> K4 (and across calls): tests + A/B bench on one box
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/aq_tests.txt 2>&1
for rep in 1 2; do
DASH_PDL=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-gate --no-sweep > gpurun_out/aq_off_$rep.json 2>/dev/null
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-gate --no-sweep > gpurun_out/aq_on_$rep.json 2>/dev/null
done
DASH_PDL=0 timeout 600 python scripts/ab_split.py pdl_off > gpurun_out/aq_split.txt 2>&1
timeout 600 python scripts/ab_split.py pdl_on >> gpurun_out/aq_split.txt 2>&1
