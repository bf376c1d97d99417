# v12: W = 4 vs 2 (+ replay for every W)
set -x
timeout 900 python -m pytest tests/test_gpu_replay.py -m gpu -x -q 2>&1 | tail -3
DASH_ACC_SPLIT=4 timeout 900 python -m pytest tests/test_gpu_bwd.py -m gpu -x -q 2>&1 | tail -3
for w in 2 4; do
  DASH_ACC_SPLIT=$w timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 causal
  DASH_ACC_SPLIT=$w timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 128 full
  DASH_ACC_SPLIT=$w timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 64 causal
  DASH_ACC_SPLIT=$w timeout 300 python scripts/exp_reduce_path.py 512,2048,16384 64 full
done 2>&1 | grep -E "DEBUG" | tee gpurun_out/exp_v12.txt
