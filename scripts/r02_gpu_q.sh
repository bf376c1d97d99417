#!/bin/bash
# round 2: dQ-plane budget (head chunks) -> chunk tests, config-4 parity and timing,
# clocked model check and block e2e
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_chunk.py -x -q > gpurun_out/q_chunk.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bwd.py -x -q -k "long_context or profile or watchdog" > gpurun_out/q_bwd.txt 2>&1
timeout 900 python scripts/long_context.py --out gpurun_out/q_long_context.json > gpurun_out/q_long_context.log 2>&1
timeout 900 python scripts/model_check.py --out gpurun_out/q_model_check.json > gpurun_out/q_model_check.log 2>&1
timeout 900 python scripts/block_e2e.py --out gpurun_out/q_block_e2e.json > gpurun_out/q_block_e2e.log 2>&1
