#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 240 python scripts/pair_smoke.py > gpurun_out/c_pair_smoke.txt 2>&1
echo "rc=$?" >> gpurun_out/c_pair_smoke.txt
tail -30 gpurun_out/c_pair_smoke.txt
