# v9: 2-CTA pair kernel -- correctness first, then pair vs single timing
set -x
timeout 600 python -m pytest tests/test_gpu_replay.py -m gpu -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
for pr in 1 0; do
  DASH_PAIR=$pr timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 causal
  DASH_PAIR=$pr timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 full
  DASH_PAIR=$pr timeout 300 python scripts/exp_reduce_path.py 2048,16384 64 causal
done 2>&1 | grep -E "DEBUG|PAIR" | tee gpurun_out/exp_v9b.txt
timeout 120 python scripts/grid_probe.py 2>&1 | tail -3
